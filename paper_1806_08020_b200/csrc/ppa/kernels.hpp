#pragma once
// Host-side launchers for the sm_100a kernels (csrc/kernels/*.cu).
// Every launcher is asynchronous on the given stream; none synchronises.

#include <cuda_runtime.h>

#include <vector>

#include "ppa/device.hpp"

namespace ppa {
namespace kern {

/// Device copy of a CsrMatrix plus the row-block partition used by the
/// streaming SpMV.  Pointers are device pointers.
struct CsrDevice {
  int n = 0;
  long long nnz = 0;
  const int* row_ptr = nullptr;  // [n+1]
  const int* col_idx = nullptr;  // [nnz (+pad)]
  const double* values = nullptr;
  const int* blk_row = nullptr;  // [nblocks+1] first row of each row block
  int nblocks = 0;
  // Sliced ELL (SELL-32) copy: slice s holds rows 32s..32s+31; entry k of
  // lane l sits at slice_ptr[s] + 32k + l; padding has col = -1.  Used when
  // the padding overhead is small (regular rows); nullptr otherwise.
  const long long* slice_ptr = nullptr;  // [nslices+1]
  const int* sell_col = nullptr;
  const double* sell_val = nullptr;
  const int* sell_perm = nullptr;  // slice row -> matrix row (nullptr: identity)
  int nslices = 0;
  int sell_sigma = 1;
  long long sell_entries = 0;
  int bandwidth = -1;  // max |col - row| over the entries (-1: unknown)
  // Packed SELL-32 (spmv_packed.cu): same slices and row order as SELL-32,
  // widths rounded up to kPackChunk; column stored as an int16 offset from
  // the row (kPackPad marks padding), value as a uint8 code into `pk_dict`
  // (pk_ndict <= 256 distinct values) or, without a dictionary, as fp64.
  // Entry k of lane l of slice s: pk_ptr[s] + 32*kPackChunk*(k/kPackChunk)
  // + kPackChunk*l + k%kPackChunk.  nullptr when it would not save bytes.
  const long long* pk_ptr = nullptr;  // [nslices+1]
  const short* pk_col = nullptr;
  const unsigned char* pk_code = nullptr;
  const double* pk_val = nullptr;
  const double* pk_dict = nullptr;
  int pk_ndict = 0;  // 0: values stored in pk_val
  long long pk_entries = 0;
  // Diagonal-coded layout (spmv_dia.cu): row r's codes at
  // dia_code[r*dia_stride + j] for diagonal j (offset dia_off[j], increasing);
  // a code indexes dia_dict, kDiaAbsent marks no entry.  nullptr: not used.
  const unsigned char* dia_code = nullptr;
  const double* dia_dict = nullptr;
  int dia_ndict = 0;
  int dia_ndiag = 0;
  int dia_stride = 0;  // 4, 8, 16 or 32 bytes per row
  int dia_off[32] = {};
  // Regular-row form (spmv_dia.cu k_spmv_diar): a row is regular when every
  // diagonal is present with its default value dia_dflt[j]; regular rows
  // stream no codes (bit r%32 of dia_mask[r/32] set).  The irregular rows
  // are listed in dia_irr_rows with their codes at dia_irr_codes[k*stride].
  // nullptr: every row streams its codes.
  const unsigned* dia_mask = nullptr;
  const int* dia_irr_rows = nullptr;
  const unsigned char* dia_irr_codes = nullptr;
  long long dia_nirr = 0;
  double dia_dflt[32] = {};
  // Presence form (spmv_dia2.cu): bit j of dia_pres[r] set when row r has an
  // entry on diagonal j; only built when at most 8 diagonals and every
  // present entry carries its diagonal's default value.  nullptr otherwise.
  // Rows [-5D - 64, n + 5D + 64) are readable (zero outside the matrix);
  // dia_pres is 16-byte aligned.
  const unsigned char* dia_pres = nullptr;
  long long dia_pres_pad = 0;
  // Box-grid stencil (spmv_grid2.cu): the presence form is exactly a 7-point
  // stencil on a grid_nx x grid_ny x grid_nz box (offsets -nx ny, -nx, -1, 0,
  // 1, nx, nx ny) or a 5-point one on grid_nx x grid_nz (grid_ny = 1), cut at
  // the box faces.  grid_nx = 0 otherwise.
  int grid_nx = 0, grid_ny = 0, grid_nz = 0;
};

constexpr int kDiaMaxDiag = 32;
constexpr int kDiaMaxDict = 255;
constexpr unsigned kDiaAbsent = 0xffu;
/// Largest (diagonals x n) / nnz accepted for the diagonal layout.
constexpr double kDiaMaxFill = 1.5;

/// Largest diagonal count of the regular-row kernel.
constexpr int kDiaRegularMaxDiag = 16;
/// Entries per lane per packed load group and the padding marker.
constexpr int kPackChunk = 4;
constexpr short kPackPad = -32768;
constexpr int kPackMaxDict = 256;

/// Host-side packed SELL-32 construction over an existing SELL-32 row order
/// (`perm` empty: identity).  Returns false when a column offset does not
/// fit int16 or the packed stream would not be smaller than SELL-32's.
bool build_sell32_packed(const int* row_ptr, const int* col_idx, const double* values, int n,
                         const std::vector<int>& perm, long long sell_entries,
                         std::vector<long long>& pk_ptr, std::vector<short>& cols,
                         std::vector<unsigned char>& codes, std::vector<double>& vals,
                         std::vector<double>& dict);
/// Bytes the packed stream occupies (cols + codes/values) per entry.
inline double packed_entry_bytes(int ndict) { return 2.0 + (ndict > 0 ? 1.0 : 8.0); }

/// Two polynomial factors applied in one temporally blocked pass
/// (spmv_dia2.cu, spmv_grid2.cu):
///   pair = false: y1 = x + a0 (A x),  y2 = y1 + b0 (A y1)   (two real roots)
///   pair = true : t = A x,            y2 = (x + a1 t) + a0 (A t)  (conjugate pair)
/// Only y2 is stored.
struct Mp2Pass {
  bool pair = false;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0;
  bool one = false;  // box-grid slab pass only: a single real factor y = x + a0 (A x)
};

/// True when two factors can run as one temporally blocked pass over the
/// diagonal layout (spmv_dia2.cu): presence form, outer diagonals +-D, even n
/// and D, in-plane offsets small against D.  PPA_DISABLE_DIA2=1 turns it off.
bool dia2_supported(const CsrDevice& a);
/// True when the box-grid form of the two-factor pass applies (spmv_grid2.cu:
/// grid_nx > 0 and a launch plan exists).  PPA_DISABLE_GRID2=1 turns it off.
bool grid2_supported(const CsrDevice& a);
/// The per-device zero page the box-grid pass copies for planes outside the
/// box (allocated on first use; layout_build.cu touches it so that a capture
/// never allocates).
const double* grid2_zeros();
/// Row evaluations of one box-grid pass: level 1 (the widened tiles and
/// the chunks' extra planes) and level 2 (= n); 0 when the form does not run.
void grid2_row_evals(const CsrDevice& a, long long* l1, long long* l2);
/// The box-grid two-factor pass (same contract as spmv_dia2).
void spmv_grid2(const CsrDevice& a, const Mp2Pass& p, const double* x, double* y,
                const double* base, cudaStream_t st);
/// The box-grid pass over one rank's z-slab (planes [zo0, zo1) of an
/// nx x ny x nz box; ny = 1 for the 2-D 5-point form), the halo planes read
/// by the kernel straight from the neighbours' buffers xl (local plane 0 =
/// global plane zl0) and xr (local plane 0 = global plane zo1) after their
/// 64-bit epoch flags fl / fr reach `epoch` (dist.py ShardedGridPoly).
/// x and y hold the owned planes only.  *err is set if a flag never arrives.
/// own (this rank's flag, 2 words: flag, ticket counter) non-null: the
/// pass's last CTA publishes epoch + 1 into it (system-scope release).
/// Argument checks of spmv_grid2_slab (std::invalid_argument), no device work.
void spmv_grid2_slab_check(int nd, int nx, int ny, int nz, int zo0, int zo1, const double* xl,
                           int zl0, const long long* fl, const double* xr, const long long* fr);
void spmv_grid2_slab(int nd, int nx, int ny, int nz, const double* vals, int zo0, int zo1,
                     const Mp2Pass& p, const double* x, double* y, const double* xl, int zl0,
                     const long long* fl, const double* xr, const long long* fr,
                     long long epoch, int* err, long long* own, cudaStream_t st);
/// One two-factor pass (Mp2Pass semantics, y2 only; t / y1 never stored).
/// x and y distinct and 16-byte aligned; `base` folds the complement.
void spmv_dia2(const CsrDevice& a, const Mp2Pass& p, const double* x, double* y,
               const double* base, cudaStream_t st);

/// Halo of the row-sharded pi(A)v pulled from a peer's memory (peer_halo.cu;
/// dist.py PeerHalo): x_ext[dst_offset + i] = src[src_index[i]], i < count,
/// once *flag >= the exchange's epoch.  src and flag are CUDA-IPC pointers
/// into the owner's HBM; src_index lives on the reader.
struct PeerHaloDesc {
  const double* src;
  const long long* src_index;
  long long count;
  long long dst_offset;
  const long long* flag;
};
/// *flag = epoch (system-scope release) after the stream's earlier work.
void publish(long long* flag, long long epoch, cudaStream_t st);
/// Waits for every peer's flag (bounded: *error = 1 on timeout) and gathers.
void halo_pull(const PeerHaloDesc* peers_dev, int npeers, long long max_count, double* x_ext,
               long long epoch, int* error, cudaStream_t st);

/// SELL-32 is used when its padded entry count is at most this factor of nnz.
constexpr double kSellMaxPadding = 1.15;

/// Sorting window used when unsorted SELL-32 pads too much (irregular rows).
constexpr int kSellSigma = 16384;

/// Device-built SELL-32 (layout_build.cu): owns the arrays CsrDevice points to.
struct DevSell {
  DBuffer<long long> slice_ptr;  // [nslices+1]
  DBuffer<int> cols;             // [total+32], padding -1
  DBuffer<double> vals;          // [total+32], padding 0
  DBuffer<int> perm;             // empty when sigma == 1
  long long total = 0;
  int nslices = 0;
};
/// SELL-32 from the device CSR; sigma > 1 stably sorts rows by decreasing
/// length inside sigma-row windows (same order as a host stable sort).
/// False (nothing kept) when the padding exceeds kSellMaxPadding.
bool build_sell32_device(const int* row_ptr, const int* col_idx, const double* values, int n,
                         long long nnz, int sigma, DevSell& out, cudaStream_t st);

/// Device-built diagonal-coded layout and, when `regular`, its regular-row form.
struct DevDia {
  std::vector<int> offsets;  // increasing
  std::vector<double> dict;  // ascending bit patterns
  int ndiag = 0;
  int stride = 0;
  DBuffer<unsigned char> codes;  // [round32(n) * stride]
  bool regular = false;
  std::vector<double> defaults;  // per diagonal
  DBuffer<unsigned> mask;
  DBuffer<int> irr_rows;
  DBuffer<unsigned char> irr_codes;
  long long nirr = 0;
  DBuffer<unsigned char> pres;  // presence form, pres_pad zero rows each side; may be empty
  long long pres_pad = 0;
  int grid[3] = {0, 0, 0};  // box-grid stencil nx, ny, nz (0: not one; spmv_grid2.cu)
};
/// Diagonal-coded layout from the device CSR; false when the matrix has more
/// than kDiaMaxDiag diagonals, more than kDiaMaxDict distinct values or a
/// fill above kDiaMaxFill.  The regular-row form is added when `want_regular`,
/// ndiag <= kDiaRegularMaxDiag and at least half the rows are regular.
bool build_dia_device(const int* row_ptr, const int* col_idx, const double* values, int n,
                      long long nnz, bool want_regular, DevDia& out, cudaStream_t st);

/// Row-block capacities of the streaming SpMV (must match spmv.cu).
constexpr int kSpmvThreads = 256;
constexpr int kSpmvMaxRows = 256;
constexpr int kSpmvMaxNnz = 2048;
/// Elements of padding after col_idx/values so vector loads never run off
/// the allocation.
constexpr int kSpmvPad = 8;

/// Fused epilogues of the SpMV (s = (A x)[i]).  Each reproduces the
/// reference's operation order (src/gmres_poly.cpp:129-143) without FMA
/// contraction so the result is bit-identical to the scalar CPU loop:
///   plain : y = s
///   real  : y = x[i] + (c0 * s)                 real root, c0 = -1/theta
///   pair  : y = (o[i] + (c1 * x[i])) + (c0 * s) conjugate pair, second
///           product; x = t1, c1 = -2Re(theta)/|theta|^2, c0 = 1/|theta|^2
/// Optionally, complement: y = base[i] - z (tau = I - pi, src/gmres_poly.cpp:306-308).
enum class Epi : int { plain = 0, real = 1, pair = 2 };

struct EpiArgs {
  Epi mode = Epi::plain;
  double c0 = 0.0;
  double c1 = 0.0;
  const double* o = nullptr;     // pair: running product (may alias y)
  const double* base = nullptr;  // complement base (nullptr: no complement)
  // outer factor of a nested polynomial folded after the complement
  // (spmv_epilogue.cuh); only with base != nullptr.  oo may alias y.
  int outer = 0;  // 0 none, 1 real, 2 pair
  double oc0 = 0.0, oc1 = 0.0;
  const double* oo = nullptr;
};

void spmv(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep, cudaStream_t st);
/// The packed-SELL path of spmv() (requires a.pk_ptr).
void spmv_packed(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                 cudaStream_t st);
/// The diagonal-coded paths of spmv() / spmm() (require a.dia_code).
void spmv_dia(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
              cudaStream_t st);
void spmm_dia(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY,
              long long ldo, cudaStream_t st);
/// The packed-SELL path of spmm() (requires a.pk_ptr).
void spmm_packed(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY,
                 long long ldo, cudaStream_t st);

/// AY[:,j] = A Y[:,j] for j < p (column-major, leading dims ldy / ldo):
/// one matrix read per 8 columns with SELL-32, per-column SpMV otherwise.
/// Every column is bit-identical to spmv() of that column.
void spmm(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY, long long ldo,
          cudaStream_t st);

/// Builds the row-block partition on the host from row_ptr.
/// Returns the first row of each block (size nblocks+1).
void build_row_blocks(const int* row_ptr_host, int n, int max_rows, int max_nnz,
                      std::vector<int>& blk_row);

// ---------------------------------------------------------------- blas1 ---
void copy(const double* x, double* y, long long n, cudaStream_t st);
void axpy(double a, const double* x, double* y, long long n, cudaStream_t st);  // y += a*x
void scale(double* x, double a, long long n, cudaStream_t st);                  // x *= a
void div_scale(double* x, const double* dev_a, long long n, cudaStream_t st);   // x /= *dev_a
void div_value(double* x, double a, long long n, cudaStream_t st);               // x /= a
void sub(const double* x, const double* w, double* y, long long n, cudaStream_t st);  // y = x - w
void fill(double* x, double v, long long n, cudaStream_t st);

/// out[0] = x . y  (deterministic two-stage reduction; device result)
void dot(const double* x, const double* y, long long n, double* out, ReduceWorkspace& ws,
         int sm_count, cudaStream_t st);
/// out[0] = ||x||_2
void nrm2(const double* x, long long n, double* out, ReduceWorkspace& ws, int sm_count,
          cudaStream_t st);

// ---------------------------------------------------------- tall-skinny ---
/// out[j] = sum_i V[i,j] * w[i], j < c.  V column-major with leading dim ld.
void ts_dot(const double* V, long long ld, int n, int c, const double* w, double* out,
            ReduceWorkspace& ws, int sm_count, cudaStream_t st);

/// One CGS2 orthogonalisation step of w against V[:,0:c] (three sweeps):
///   h1 = V^T w;  w -= V h1;  h2 = V^T w, s = ||w||^2 (fused);
///   hsub = sqrt(s - ||h2||^2);  V[:,c] = (w - V h2) / hsub (fused).
/// Hcol[0..c] receives (h1 + h2, hsub) and *flag the breakdown test
/// hsub <= 1e-14 * ||Hcol|| (src/arnoldi.cpp:140-148); on breakdown
/// Hcol[c] = 0 and V[:,c] is not written.  All outputs stay on device.
void cgs2_step(double* V, long long ld, int n, int c, double* w, double* Hcol, int* flag,
               ReduceWorkspace& ws, int sm_count, cudaStream_t st);

/// Delayed CGS2 (arnoldi.cpp "DCGS2"), sweep 1: with the pending vector u in
/// column c-1 of V, out[0..c) = V[:,0:c]^T z and out[c..2c) = V[:,0:c]^T u in
/// one read of V.
void dcgs2_dot(const double* V, long long ld, int n, int c, const double* z, double* out,
               ReduceWorkspace& ws, int sm_count, cudaStream_t st);
/// Delayed CGS2, sweep 2: coef = [s (c-1), d (c-1), e, rho];
/// V[:,c-1] = (u - V[:,0:c-1] s) / rho  and, in place,
/// z = (z / rho - V[:,0:c-1] d) - e u  (the next pending vector).
void dcgs2_update(double* V, long long ld, int n, int c, double* z, const double* coef,
                  ReduceWorkspace& ws, int sm_count, cudaStream_t st);

/// One classical Gram-Schmidt pass: c = V^T v; v -= V c; out_norm = ||v||.
/// corr (device, c) receives the coefficients.
/// Row-sharded CGS2 (dist.py): sweep 2 with rank-local sums out = [V^T w',
/// ||w'||^2] (c + 1) after w' = w - V h, and sweep 3 V[:,c] = (w - V h2) / *hsub.
void cgs_update_dot_local(const double* V, long long ld, int n, int c, double* w,
                          const double* h, double* out, ReduceWorkspace& ws, int sm_count,
                          cudaStream_t st);
void cgs_store_local(double* V, long long ld, int n, int c, const double* w, const double* h2,
                     const double* hsub, ReduceWorkspace& ws, int sm_count, cudaStream_t st);
void cgs1_pass(const double* V, long long ld, int n, int c, double* v, double* corr,
               double* out_norm, ReduceWorkspace& ws, int sm_count, cudaStream_t st);

/// Out[:,0:p] = V[:,0:d] * G, G column-major d x p on device.  In place
/// (Out == V, same ld) is allowed when p <= d: every row block is staged in
/// shared memory before it is overwritten.
/// TMA-fed form of ts_combine (cgs.cu k_combine_tma), same bits; false when
/// it does not apply (p > 32, d > 96, misaligned V, PPA_COMBINE_TMA=0).
bool ts_combine_tma(const double* V, long long ldv, int n, int d, const double* G, int p,
                    double* Out, long long ldo, int sm_count, cudaStream_t st);
void ts_combine(const double* V, long long ldv, int n, int d, const double* G, int p,
                double* Out, long long ldo, cudaStream_t st);

/// out[j] = sum_i Y[i,j]^2 for j < p.
void col_sumsq(const double* Y, long long ld, int n, int p, double* out, ReduceWorkspace& ws,
               int sm_count, cudaStream_t st);

/// Ritz-pair checks against A (solver convergence test).
/// real:  out[0] = mu = y.Ay ; out[1] = ||Ay - mu y||
void ritz_check_real(const double* y, const double* Ay, long long n, double* out,
                     ReduceWorkspace& ws, int sm_count, cudaStream_t st);
/// complex y = yr + i yi:  out[0..1] = mu (re, im), out[2] = ||Ay - mu y||
void ritz_check_complex(const double* yr, const double* yi, const double* Ayr,
                        const double* Ayi, long long n, double* out, ReduceWorkspace& ws,
                        int sm_count, cudaStream_t st);

/// Ensures the reduction workspace can host `blocks` partial rows of
/// `width` values.
void ensure_workspace(ReduceWorkspace& ws, int blocks, int width);

}  // namespace kern
}  // namespace ppa
