"""ctypes bindings of libppa_b200.so (include/ppa_b200.h).

Names follow the reference's API (proj/include/ppa/*.hpp); C status codes
map back onto the reference's exception types:
    PPA_INVALID_ARGUMENT -> ValueError   (std::invalid_argument)
    PPA_RUNTIME_ERROR    -> RuntimeError (std::runtime_error)
    PPA_LOGIC_ERROR      -> LogicError   (std::logic_error)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libppa_b200.so")

STREAM_NORM, STREAM_POLY, STREAM_ARNOLDI, STREAM_POLY2, STREAM_MATRIX = 1, 2, 3, 4, 5
SMALLEST_MAGNITUDE, LARGEST_MAGNITUDE, TARGET_ONE = 0, 1, 2
# int (*)(void* ctx, const double* x_dev, double* y_dev, void* cuda_stream)
_APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)

KINDS = ["csr", "diagonal", "shifted", "block2", "poly", "composite", "external"]


class PPAError(RuntimeError):
    pass


class LogicError(RuntimeError):
    """std::logic_error (e.g. a complex root without adjacent conjugate)."""


class CostRecord(C.Structure):
    """inc/cost.hpp:17-23"""

    _fields_ = [("mvps", C.c_longlong), ("dots", C.c_longlong), ("vops", C.c_longlong),
                ("nnzr", C.c_double), ("wall_seconds", C.c_double)]

    def as_dict(self):
        return {"mvps": self.mvps, "dots": self.dots, "vops": self.vops, "nnzr": self.nnzr}

    def __repr__(self):
        return f"CostRecord(mvps={self.mvps}, dots={self.dots}, vops={self.vops}, nnzr={self.nnzr})"


class _SolveConfigC(C.Structure):
    _fields_ = [("m", C.c_int), ("k", C.c_int), ("nev", C.c_int), ("degree", C.c_int),
                ("rtol_multiplier", C.c_double), ("rtol_absolute", C.c_double),
                ("variant", C.c_int), ("stability", C.c_int), ("double_d1", C.c_int),
                ("double_d2", C.c_int), ("use_double", C.c_int), ("max_cycles", C.c_int),
                ("seed", C.c_ulonglong), ("allow_nev_above_k", C.c_int),
                ("damping", C.c_int), ("damping_alpha", C.c_double), ("damping_power", C.c_int),
                ("check_mid_cycle", C.c_int), ("mid_cycle_stride", C.c_int),
                ("stagnation_stop", C.c_int), ("stagnation_window", C.c_int),
                ("stagnation_rtol", C.c_double), ("want_eigenvectors", C.c_int),
                ("orthogonalization", C.c_int)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class _SolveResultC(C.Structure):
    _fields_ = [("cap_nev", C.c_int), ("cap_roots", C.c_int), ("cap_cycles", C.c_int),
                ("eig_re", _dp), ("eig_im", _dp), ("residuals", _dp), ("converged_flags", _ip),
                ("poly_re", _dp), ("poly_im", _dp), ("inner_re", _dp), ("inner_im", _dp),
                ("cycle_max_residual", _dp),
                ("n_eig", C.c_int), ("n_poly", C.c_int), ("n_inner", C.c_int),
                ("n_cycles", C.c_int), ("converged", C.c_int), ("cycles", C.c_int),
                ("composite_degree", C.c_int), ("poly_base_degree", C.c_int),
                ("discarded_probes", C.c_int),
                ("rtol", C.c_double), ("max_err", C.c_double), ("norm_estimate", C.c_double),
                ("cost", CostRecord),
                ("t_total", C.c_double), ("t_setup", C.c_double), ("t_extend", C.c_double),
                ("t_check", C.c_double), ("t_restart", C.c_double),
                ("evec_re", _dp), ("evec_im", _dp), ("evec_ld", C.c_longlong)]


_lib = None


def lib():
    """The loaded C-ABI library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run __graft_entry__.build() "
                              "(there is no CPU fallback for the CUDA path)")
        L = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        L.ppa_last_error.restype = C.c_char_p
        sigs = {
            "ppa_abi_version": [],
            "ppa_device_info": [_ip, _dp],
            "ppa_set_stream": [vp],
            "ppa_synchronize": [],
            "ppa_host_csr_create": [C.c_int, C.c_longlong, vp, vp, vp, C.POINTER(vp)],
            "ppa_host_csr_from_triplets": [C.c_int, C.c_longlong, vp, vp, vp, C.POINTER(vp)],
            "ppa_gen_convdiff_ref": [C.c_int, C.POINTER(vp)],
            "ppa_gen_config": [C.c_int, C.POINTER(vp)],
            "ppa_gen_bidiagonal": [C.c_int, C.POINTER(vp)],
            "ppa_gen_convdiff_const": [C.c_int, C.c_double, C.POINTER(vp)],
            "ppa_gen_laplacian_3d": [C.c_int, C.POINTER(vp)],
            "ppa_gen_random_poisson": [C.c_int, C.c_double, C.c_ulonglong, C.POINTER(vp)],
            "ppa_host_csr_info": [vp, _ip, C.POINTER(C.c_longlong), C.POINTER(C.c_ulonglong)],
            "ppa_host_csr_arrays": [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
            "ppa_normal_vector": [C.c_longlong, C.c_ulonglong, C.c_ulonglong, vp],
            "ppa_csr_operator": [vp, C.POINTER(vp)],
            "ppa_diagonal_operator": [C.c_int, vp, C.POINTER(vp)],
            "ppa_poly_operator": [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)],
            "ppa_op_info": [vp, _ip, _ip, _dp, _ip],
            "ppa_op_apply": [vp, vp, vp, C.POINTER(CostRecord)],
            "ppa_op_apply_host": [vp, vp, vp, C.POINTER(CostRecord)],
            "ppa_op_apply_host_batch": [vp, C.c_int, vp, vp, C.POINTER(CostRecord)],
            "ppa_csr_model_bytes": [vp, _dp, C.POINTER(C.c_longlong)],
            "ppa_csr_layout": [vp, _ip, _dp, _ip, _ip],
            "ppa_spmv_factor": [vp, vp, vp, C.c_int, C.c_double, C.c_double, vp, vp],
            "ppa_factor_plan": [vp, vp, C.c_int, _ip, vp, vp, _ip],
            "ppa_host_csr_multiply": [vp, vp, vp],
            "ppa_csr_operator_layout": [vp, C.c_int, C.POINTER(vp)],
            "ppa_csr_two_factor_pass": [vp, _ip],
            "ppa_csr_grid_work": [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)],
            "ppa_csr_grid_form": [vp, _ip, _ip, _ip, _ip],
            "ppa_arnoldi_set_orthogonalization": [vp, C.c_int],
            "ppa_apply_poly": [vp, vp, C.c_int, vp, vp, vp, C.POINTER(CostRecord)],
            "ppa_build_gmres_poly": [vp, vp, C.c_int, vp, vp, _ip, _ip, C.POINTER(CostRecord)],
            "ppa_build_gmres_poly_ortho": [vp, vp, C.c_int, C.c_int, vp, vp, _ip, _ip,
                                           C.POINTER(CostRecord)],
            "ppa_solve_config_default": [vp],
            "ppa_cgs_dot_local": [vp, C.c_longlong, C.c_int, C.c_int, vp, vp],
            "ppa_cgs_update_dot_local": [vp, C.c_longlong, C.c_int, C.c_int, vp, vp, vp],
            "ppa_cgs_store_local": [vp, C.c_longlong, C.c_int, C.c_int, vp, vp, vp],
            "ppa_dot_local": [vp, vp, C.c_longlong, vp],
            "ppa_dev_alloc": [C.c_size_t, C.POINTER(vp)],
            "ppa_dev_free": [vp],
            "ppa_ipc_get_handle": [vp, vp],
            "ppa_ipc_open": [vp, C.POINTER(vp)],
            "ppa_ipc_close": [vp],
            "ppa_halo_publish": [vp, C.c_longlong],
            "ppa_halo_pull": [vp, C.c_int, C.c_longlong, vp, C.c_longlong, vp],
            "ppa_grid2_slab_chain": [C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int,
                                     C.c_int, _ip, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, vp,
                                     vp, vp, C.c_longlong, vp, vp, _ip],
            "ppa_grid2_slab_pass": [C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int,
                                    C.c_int, C.c_double, C.c_double, C.c_double, vp, vp, vp,
                                    C.c_int, vp, vp, vp, C.c_longlong, vp, vp],
            "ppa_op_create_callback": [C.c_int, C.c_int, C.c_double, _APPLY_FN, vp,
                                       C.POINTER(vp)],
            "ppa_arnoldi_ritz_vectors": [vp, C.c_int, vp, vp, vp, vp, vp],
            "ppa_arnoldi_harmonic_selection": [vp, C.c_int, vp, vp, vp, vp, vp],
            "ppa_arnoldi_restart_keep": [vp, C.c_int, vp, vp, vp, vp, C.c_int,
                                         C.POINTER(CostRecord), _ip],
            "ppa_leja_order": [vp, vp, C.c_int, vp, vp],
            "ppa_compute_pof": [vp, vp, C.c_int, vp, vp, _ip, _dp, _ip],
            "ppa_add_stability_roots": [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, _ip],
            "ppa_eval_poly": [vp, vp, C.c_int, C.c_double, C.c_double, _dp, _dp],
            "ppa_arnoldi_init": [vp, C.c_int, C.c_int, C.POINTER(CostRecord), C.POINTER(vp)],
            "ppa_arnoldi_extend": [vp, vp, C.c_int, C.POINTER(CostRecord)],
            "ppa_arnoldi_info": [vp, _ip, _ip, _ip, C.POINTER(C.c_longlong), C.POINTER(vp)],
            "ppa_arnoldi_get_H": [vp, vp],
            "ppa_arnoldi_ritz": [vp, C.c_int, vp, vp, vp],
            "ppa_arnoldi_harmonic": [vp, vp, vp],
            "ppa_arnoldi_ritz_vector": [vp, C.c_int, C.c_int, vp, vp, _ip, C.POINTER(CostRecord)],
            "ppa_arnoldi_restart": [vp, C.c_int, C.c_int, C.POINTER(CostRecord), _ip],
            "ppa_spmv": [vp, vp, vp],
            "ppa_spmm": [vp, vp, C.c_longlong, C.c_int, vp, C.c_longlong],
            "ppa_cgs2_step": [vp, C.c_longlong, C.c_int, C.c_int, vp, vp, vp],
            "ppa_ts_combine": [vp, C.c_longlong, C.c_int, C.c_int, vp, C.c_int, vp, C.c_longlong],
            "ppa_solve": [vp, C.POINTER(_SolveConfigC), C.POINTER(_SolveResultC)],
            "ppa_check_ideal_order": [vp, vp, C.c_int, C.c_int, _ip],
            "ppa_damping_heuristic": [vp, C.POINTER(_SolveConfigC), vp, vp, C.c_int, _ip,
                                      C.POINTER(CostRecord)],
            "ppa_block2_operator": [vp, C.POINTER(vp)],
            "ppa_shifted_operator": [vp, C.c_double, C.POINTER(vp)],
            "ppa_build_two_vector_poly": [vp, vp, vp, C.c_int, vp, vp, _ip, C.POINTER(CostRecord)],
            "ppa_damped_start": [vp, vp, C.c_double, C.c_int, vp, C.POINTER(CostRecord)],
            "ppa_read_matrix_market": [C.c_char_p, C.POINTER(vp)],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        for name in ("ppa_host_csr_free", "ppa_op_free", "ppa_arnoldi_free"):
            f = getattr(L, name)
            f.argtypes = [vp]
            f.restype = None
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().ppa_last_error().decode()
    if status == 1:
        raise ValueError(msg)
    if status == 3:
        raise LogicError(msg)
    if status == 2:
        raise RuntimeError(msg)
    raise PPAError(f"[status {status}] {msg}")


def _ptr(x) -> int:
    """Device pointer of a torch tensor (or a raw int)."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _roots(roots) -> tuple[np.ndarray, np.ndarray]:
    r = np.asarray(roots, dtype=np.complex128).ravel()
    return _f64(r.real), _f64(r.imag)


def set_stream(stream) -> None:
    """Launch subsequent kernels of this thread on `stream` (torch.cuda.Stream or handle)."""
    h = getattr(stream, "cuda_stream", stream)
    _check(lib().ppa_set_stream(C.c_void_p(int(h) if h else 0)))


def synchronize() -> None:
    _check(lib().ppa_synchronize())


# --------------------------------------------------------------------- CSR --
class CsrMatrix:
    """Host CSR matrix (inc/operators.hpp:15-33), validated on construction."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ppa_host_csr_free(self._h)
            self._h = None

    @classmethod
    def from_arrays(cls, n, row_ptr, col_idx, values):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = _f64(values)
        h = C.c_void_p()
        _check(lib().ppa_host_csr_create(n, len(v), _np_ptr(rp), _np_ptr(ci), _np_ptr(v), C.byref(h)))
        return cls(h)

    @classmethod
    def from_triplets(cls, n, rows, cols, vals):
        r = np.ascontiguousarray(rows, dtype=np.int32)
        c = np.ascontiguousarray(cols, dtype=np.int32)
        v = _f64(vals)
        h = C.c_void_p()
        _check(lib().ppa_host_csr_from_triplets(n, len(v), _np_ptr(r), _np_ptr(c), _np_ptr(v),
                                                C.byref(h)))
        return cls(h)

    @classmethod
    def _gen(cls, fn, *args):
        h = C.c_void_p()
        _check(fn(*args, C.byref(h)))
        return cls(h)

    @classmethod
    def config(cls, k: int):
        return cls._gen(lib().ppa_gen_config, k)

    @classmethod
    def convection_diffusion(cls, grid_n: int):
        """make_convection_diffusion (src/operators.cpp:190-244)."""
        return cls._gen(lib().ppa_gen_convdiff_ref, grid_n)

    @classmethod
    def convection_diffusion_const(cls, grid_n: int, peclet: float = 0.5):
        return cls._gen(lib().ppa_gen_convdiff_const, grid_n, C.c_double(peclet))

    @classmethod
    def laplacian_3d(cls, grid_n: int):
        return cls._gen(lib().ppa_gen_laplacian_3d, grid_n)

    @classmethod
    def bidiagonal(cls, n: int):
        return cls._gen(lib().ppa_gen_bidiagonal, n)

    @classmethod
    def random_poisson(cls, n: int, lam: float = 16.0, seed: int = 4):
        return cls._gen(lib().ppa_gen_random_poisson, n, C.c_double(lam), C.c_ulonglong(seed))

    def info(self):
        n = C.c_int()
        nnz = C.c_longlong()
        fp = C.c_ulonglong()
        _check(lib().ppa_host_csr_info(self._h, C.byref(n), C.byref(nnz), C.byref(fp)))
        return n.value, nnz.value, fp.value

    @property
    def n(self):
        return self.info()[0]

    @property
    def nnz(self):
        return self.info()[1]

    def fingerprint(self) -> int:
        return self.info()[2]

    def multiply(self, x, y) -> None:
        """CsrMatrix::multiply: y = A x on device vectors, uncounted."""
        _check(lib().ppa_host_csr_multiply(self._h, _ptr(x), _ptr(y)))

    def arrays(self):
        """Copies of (row_ptr, col_idx, values)."""
        n, nnz, _ = self.info()
        rp, ci, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().ppa_host_csr_arrays(self._h, C.byref(rp), C.byref(ci), C.byref(v)))
        a = np.ctypeslib.as_array(C.cast(rp, C.POINTER(C.c_int)), (n + 1,)).copy()
        b = np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_int)), (max(nnz, 1),))[:nnz].copy()
        c = np.ctypeslib.as_array(C.cast(v, C.POINTER(C.c_double)), (max(nnz, 1),))[:nnz].copy()
        return a, b, c


def normal_vector(n: int, seed: int, stream: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(lib().ppa_normal_vector(n, seed, stream, _np_ptr(out)))
    return out


# --------------------------------------------------------------- operators --
class LinearOperator:
    """OperatorPtr (inc/operators.hpp:49-78); vectors are device pointers."""

    def __init__(self, handle, keep=()):
        self._h = handle
        self._keep = keep  # base operators must outlive wrappers

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ppa_op_free(self._h)
            self._h = None

    def _info(self):
        d, mv, k = C.c_int(), C.c_int(), C.c_int()
        nz = C.c_double()
        _check(lib().ppa_op_info(self._h, C.byref(d), C.byref(mv), C.byref(nz), C.byref(k)))
        return d.value, mv.value, nz.value, KINDS[k.value]

    def dim(self):
        return self._info()[0]

    def mvps_per_apply(self):
        return self._info()[1]

    def nnzr(self):
        return self._info()[2]

    def kind(self):
        return self._info()[3]

    def apply(self, x, y, rec: Optional[CostRecord] = None):
        rec = rec if rec is not None else CostRecord()
        _check(lib().ppa_op_apply(self._h, _ptr(x), _ptr(y), C.byref(rec)))
        return rec

    def apply_host(self, x: np.ndarray, rec: Optional[CostRecord] = None) -> np.ndarray:
        x = _f64(x)
        y = np.empty_like(x)
        rec = rec if rec is not None else CostRecord()
        _check(lib().ppa_op_apply_host(self._h, _np_ptr(x), _np_ptr(y), C.byref(rec)))
        return y

    def apply_host_batch(self, X, Y=None, rec: Optional[CostRecord] = None):
        """Apply to each row of X (count x dim, host) with H2D/compute/D2H
        overlapped across rows.  X/Y may be numpy arrays or pinned torch CPU
        tensors; returns Y."""
        rec = rec if rec is not None else CostRecord()
        if hasattr(X, "data_ptr"):
            count = X.shape[0]
            _check(lib().ppa_op_apply_host_batch(self._h, count, C.c_void_p(X.data_ptr()),
                                                 C.c_void_p(Y.data_ptr()), C.byref(rec)))
            return Y
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.empty_like(X) if Y is None else Y
        _check(lib().ppa_op_apply_host_batch(self._h, X.shape[0], _np_ptr(X), _np_ptr(Y),
                                             C.byref(rec)))
        return Y

    def model_bytes(self):
        b = C.c_double()
        nnz = C.c_longlong()
        _check(lib().ppa_csr_model_bytes(self._h, C.byref(b), C.byref(nnz)))
        return b.value

    def layout(self) -> dict:
        """Device layout of a CSR operator (ppa_csr_layout)."""
        lay, sig, nd = C.c_int(), C.c_int(), C.c_int()
        sb = C.c_double()
        _check(lib().ppa_csr_layout(self._h, C.byref(lay), C.byref(sb), C.byref(sig),
                                    C.byref(nd)))
        two = C.c_int()
        _check(lib().ppa_csr_two_factor_pass(self._h, C.byref(two)))
        gx, gy, gz, g2 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().ppa_csr_grid_form(self._h, C.byref(gx), C.byref(gy), C.byref(gz),
                                       C.byref(g2)))
        l1, l2 = C.c_longlong(), C.c_longlong()
        _check(lib().ppa_csr_grid_work(self._h, C.byref(l1), C.byref(l2)))
        return {"layout": ("csr", "sell32", "sell32_packed", "dia_coded")[lay.value],
                "stream_bytes": sb.value, "sigma": sig.value, "dict_size": nd.value,
                "two_factor_pass": bool(two.value),
                "grid": (gx.value, gy.value, gz.value) if gx.value else None,
                "grid_pass": bool(g2.value),
                "grid_rows_per_pass": (l1.value, l2.value) if g2.value else None}


LAYOUTS = {"auto": 0, "csr": 1, "sell32": 2, "sell32_packed": 3, "dia_coded": 4}


def make_csr_operator(m: CsrMatrix, layout: str = "auto") -> LinearOperator:
    """make_csr_operator (inc/operators.hpp:83); `layout` caps the device
    layout (ppa_csr_operator_layout), results are bit-identical."""
    h = C.c_void_p()
    if layout == "auto":
        _check(lib().ppa_csr_operator(m._h, C.byref(h)))
    else:
        _check(lib().ppa_csr_operator_layout(m._h, LAYOUTS[layout], C.byref(h)))
    return LinearOperator(h)


def make_diagonal(diag) -> LinearOperator:
    d = _f64(diag)
    h = C.c_void_p()
    _check(lib().ppa_diagonal_operator(len(d), _np_ptr(d), C.byref(h)))
    return LinearOperator(h)


def _poly_op(a: LinearOperator, roots, base_degree, complement):
    re, im = _roots(roots)
    h = C.c_void_p()
    _check(lib().ppa_poly_operator(a._h, _np_ptr(re), _np_ptr(im), len(re), int(base_degree or 0),
                                   int(complement), C.byref(h)))
    return LinearOperator(h, keep=(a,))


def make_poly_operator(a: LinearOperator, roots, base_degree=None) -> LinearOperator:
    return _poly_op(a, roots, base_degree, False)


def make_poly_complement_operator(a: LinearOperator, roots, base_degree=None) -> LinearOperator:
    return _poly_op(a, roots, base_degree, True)


def spmv(a: LinearOperator, x, y) -> None:
    _check(lib().ppa_spmv(a._h, _ptr(x), _ptr(y)))


def spmv_factor(a: LinearOperator, x, y, mode: int = 0, c0: float = 0.0, c1: float = 0.0,
                o=None, base=None) -> None:
    """One fused polynomial factor on device vectors (ppa_spmv_factor)."""
    _check(lib().ppa_spmv_factor(a._h, _ptr(x), _ptr(y), int(mode), C.c_double(c0),
                                 C.c_double(c1), _ptr(o) if o is not None else None,
                                 _ptr(base) if base is not None else None))


def factor_plan(roots):
    """apply_poly's factor plan: list of (pair, c0, c1) (ppa_factor_plan)."""
    r = np.ascontiguousarray(np.real(roots), dtype=np.float64)
    i = np.ascontiguousarray(np.imag(roots), dtype=np.float64)
    k = len(r)
    pair = np.zeros(max(k, 1), dtype=np.int32)
    c0, c1 = np.zeros(max(k, 1)), np.zeros(max(k, 1))
    nf = C.c_int()
    _check(lib().ppa_factor_plan(_np_ptr(r), _np_ptr(i), k, pair.ctypes.data_as(_ip),
                                 _np_ptr(c0), _np_ptr(c1), C.byref(nf)))
    return [(bool(pair[j]), float(c0[j]), float(c1[j])) for j in range(nf.value)]


def spmm(a: LinearOperator, Y, ldy: int, p: int, AY, ldo: int) -> None:
    """AY[:, j] = A Y[:, j], j < p (column-major device storage)."""
    _check(lib().ppa_spmm(a._h, _ptr(Y), ldy, p, _ptr(AY), ldo))


# -------------------------------------------------------------- polynomial --
def apply_poly(roots, a: LinearOperator, v, out, rec: Optional[CostRecord] = None):
    re, im = _roots(roots)
    rec = rec if rec is not None else CostRecord()
    _check(lib().ppa_apply_poly(_np_ptr(re), _np_ptr(im), len(re), a._h, _ptr(v), _ptr(out),
                                C.byref(rec)))
    return rec


def build_gmres_poly(a: LinearOperator, b, degree: int, rec: Optional[CostRecord] = None,
                     orthogonalization: str = "dcgs2"):
    """Returns (roots complex128 in Leja order, truncated)."""
    re = np.zeros(max(degree, 1))
    im = np.zeros(max(degree, 1))
    nr, tr = C.c_int(), C.c_int()
    rec = rec if rec is not None else CostRecord()
    _check(lib().ppa_build_gmres_poly_ortho(a._h, _ptr(b), degree,
                                            {"cgs2": 0, "dcgs2": 1}[orthogonalization],
                                            _np_ptr(re), _np_ptr(im),
                                            C.byref(nr), C.byref(tr), C.byref(rec)))
    return re[:nr.value] + 1j * im[:nr.value], bool(tr.value)


def leja_order(roots) -> np.ndarray:
    re, im = _roots(roots)
    ore, oim = np.zeros_like(re), np.zeros_like(im)
    _check(lib().ppa_leja_order(_np_ptr(re), _np_ptr(im), len(re), _np_ptr(ore), _np_ptr(oim)))
    return ore + 1j * oim


def compute_pof(roots):
    """Returns dict(log10_pof, copies_needed, max_log10_pof, total_copies)."""
    re, im = _roots(roots)
    n = len(re)
    lg = np.zeros(max(n, 1))
    cp = np.zeros(max(n, 1), dtype=np.int32)
    nd, tot = C.c_int(), C.c_int()
    mx = C.c_double()
    _check(lib().ppa_compute_pof(_np_ptr(re), _np_ptr(im), n, _np_ptr(lg), _np_ptr(cp),
                                 C.byref(nd), C.byref(mx), C.byref(tot)))
    return {"log10_pof": lg[:nd.value], "copies_needed": cp[:nd.value],
            "max_log10_pof": mx.value, "total_copies": tot.value}


def add_stability_roots(roots, base_degree=None, max_copies_per_root=1 << 20) -> np.ndarray:
    re, im = _roots(roots)
    cap = 8 * len(re) + 64
    ore, oim = np.zeros(cap), np.zeros(cap)
    on = C.c_int()
    _check(lib().ppa_add_stability_roots(_np_ptr(re), _np_ptr(im), len(re),
                                         int(base_degree or len(re)), int(max_copies_per_root),
                                         cap, _np_ptr(ore), _np_ptr(oim), C.byref(on)))
    return ore[:on.value] + 1j * oim[:on.value]


def eval_poly(roots, z: complex) -> complex:
    re, im = _roots(roots)
    a, b = C.c_double(), C.c_double()
    _check(lib().ppa_eval_poly(_np_ptr(re), _np_ptr(im), len(re), C.c_double(complex(z).real),
                               C.c_double(complex(z).imag), C.byref(a), C.byref(b)))
    return complex(a.value, b.value)


# ----------------------------------------------------------------- Arnoldi --
class ArnoldiState:
    """ArnoldiState (inc/arnoldi.hpp:18-26); V lives in HBM."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ppa_arnoldi_free(self._h)
            self._h = None

    def _info(self):
        cur, mx, bd = C.c_int(), C.c_int(), C.c_int()
        ld = C.c_longlong()
        V = C.c_void_p()
        _check(lib().ppa_arnoldi_info(self._h, C.byref(cur), C.byref(mx), C.byref(bd),
                                      C.byref(ld), C.byref(V)))
        return cur.value, mx.value, bool(bd.value), ld.value, V.value

    @property
    def cur_dim(self):
        return self._info()[0]

    @property
    def max_dim(self):
        return self._info()[1]

    @property
    def breakdown(self):
        return self._info()[2]

    @property
    def ld(self):
        return self._info()[3]

    @property
    def V_ptr(self):
        return self._info()[4]

    @property
    def H(self) -> np.ndarray:
        m = self.max_dim
        h = np.zeros((m + 1) * m)
        _check(lib().ppa_arnoldi_get_H(self._h, _np_ptr(h)))
        return h.reshape((m, m + 1)).T.copy()

    def set_orthogonalization(self, mode: str) -> None:
        """cgs2 (the Arnoldi state's default) or dcgs2 for later extends
        (ppa_arnoldi_set_orthogonalization); solve() defaults to dcgs2."""
        _check(lib().ppa_arnoldi_set_orthogonalization(self._h, {"cgs2": 0, "dcgs2": 1}[mode]))

    def extend(self, op: LinearOperator, to_dim: int, rec: Optional[CostRecord] = None):
        rec = rec if rec is not None else CostRecord()
        _check(lib().ppa_arnoldi_extend(self._h, op._h, to_dim, C.byref(rec)))
        return rec

    def ritz_pairs(self, ordering=SMALLEST_MAGNITUDE):
        d = self.cur_dim
        re, im, rs = np.zeros(d), np.zeros(d), np.zeros(d)
        _check(lib().ppa_arnoldi_ritz(self._h, ordering, _np_ptr(re), _np_ptr(im), _np_ptr(rs)))
        return re + 1j * im, rs

    def ritz_pairs_vectors(self, ordering=SMALLEST_MAGNITUDE):
        """ritz_pairs with the eigenvectors of H: (values, residuals, G) with
        G[:, i] the vector of pair i (ppa_arnoldi_ritz_vectors)."""
        d = self.cur_dim
        re, im, rs = np.zeros(d), np.zeros(d), np.zeros(d)
        vr, vi = np.zeros((d, d)), np.zeros((d, d))
        _check(lib().ppa_arnoldi_ritz_vectors(self._h, ordering, _np_ptr(re), _np_ptr(im),
                                              _np_ptr(rs), _np_ptr(vr), _np_ptr(vi)))
        return re + 1j * im, rs, (vr + 1j * vi).T.copy()

    def harmonic_restart_selection(self, ordering=SMALLEST_MAGNITUDE):
        """harmonic_restart_selection (inc/arnoldi.hpp:68-69): (values,
        residuals, G) as ritz_pairs_vectors."""
        d = self.cur_dim
        re, im, rs = np.zeros(d), np.zeros(d), np.zeros(d)
        vr, vi = np.zeros((d, d)), np.zeros((d, d))
        _check(lib().ppa_arnoldi_harmonic_selection(self._h, ordering, _np_ptr(re), _np_ptr(im),
                                                    _np_ptr(rs), _np_ptr(vr), _np_ptr(vi)))
        return re + 1j * im, rs, (vr + 1j * vi).T.copy()

    def thick_restart_keep(self, values, G, k: int, rec=None) -> int:
        """thick_restart(state, keep, k) (inc/arnoldi.hpp:79-80) with a
        caller-built keep set: values[i] and H-eigenvector G[:, i]."""
        rec = rec if rec is not None else CostRecord()
        vals = np.asarray(values, dtype=np.complex128)
        G = np.asarray(G, dtype=np.complex128)
        re, im = np.ascontiguousarray(vals.real), np.ascontiguousarray(vals.imag)
        vr = np.ascontiguousarray(G.real.T)
        vi = np.ascontiguousarray(G.imag.T)
        kk = C.c_int()
        _check(lib().ppa_arnoldi_restart_keep(self._h, len(vals), _np_ptr(re), _np_ptr(im),
                                              _np_ptr(vr), _np_ptr(vi), k, C.byref(rec),
                                              C.byref(kk)))
        return kk.value

    def harmonic_ritz_values(self):
        d = self.cur_dim
        re, im = np.zeros(d), np.zeros(d)
        _check(lib().ppa_arnoldi_harmonic(self._h, _np_ptr(re), _np_ptr(im)))
        return re + 1j * im

    def ritz_vector(self, j, y_re, y_im=None, ordering=SMALLEST_MAGNITUDE, rec=None):
        rec = rec if rec is not None else CostRecord()
        cx = C.c_int()
        _check(lib().ppa_arnoldi_ritz_vector(self._h, ordering, j, _ptr(y_re), _ptr(y_im),
                                             C.byref(cx), C.byref(rec)))
        return bool(cx.value)

    def thick_restart(self, k: int, ordering=SMALLEST_MAGNITUDE, rec=None) -> int:
        rec = rec if rec is not None else CostRecord()
        kk = C.c_int()
        _check(lib().ppa_arnoldi_restart(self._h, ordering, k, C.byref(rec), C.byref(kk)))
        return kk.value


def arnoldi_init(v0, n: int, m: int, rec: Optional[CostRecord] = None) -> ArnoldiState:
    rec = rec if rec is not None else CostRecord()
    h = C.c_void_p()
    _check(lib().ppa_arnoldi_init(_ptr(v0), n, m, C.byref(rec), C.byref(h)))
    return ArnoldiState(h)


def cgs2_step(V, ld, n, c, w, Hcol, flag) -> None:
    _check(lib().ppa_cgs2_step(_ptr(V), ld, n, c, _ptr(w), _ptr(Hcol), _ptr(flag)))


def ts_combine(V, ldv, n, d, G, p, Out, ldo) -> None:
    _check(lib().ppa_ts_combine(_ptr(V), ldv, n, d, _ptr(G), p, _ptr(Out), ldo))


# Row-sharded CGS2 building blocks (rank-local sums; dist.py ShardedSolver).
def cgs_dot_local(V, ld, n, c, w, out) -> None:
    _check(lib().ppa_cgs_dot_local(_ptr(V), ld, n, c, _ptr(w), _ptr(out)))


def cgs_update_dot_local(V, ld, n, c, w, h, out) -> None:
    _check(lib().ppa_cgs_update_dot_local(_ptr(V), ld, n, c, _ptr(w), _ptr(h), _ptr(out)))


def cgs_store_local(V, ld, n, c, w, h2, hsub) -> None:
    _check(lib().ppa_cgs_store_local(_ptr(V), ld, n, c, _ptr(w), _ptr(h2), _ptr(hsub)))


def dot_local(x, y, n, out) -> None:
    _check(lib().ppa_dot_local(_ptr(x), _ptr(y), n, _ptr(out)))


# Peer-memory halo (dist.py PeerHalo).
def dev_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    _check(lib().ppa_dev_alloc(nbytes, C.byref(p)))
    return p.value


def dev_free(ptr: int) -> None:
    _check(lib().ppa_dev_free(ptr))


def ipc_get_handle(ptr: int) -> bytes:
    buf = (C.c_ubyte * 64)()
    _check(lib().ppa_ipc_get_handle(ptr, buf))
    return bytes(buf)


def ipc_open(handle: bytes) -> int:
    buf = (C.c_ubyte * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib().ppa_ipc_open(buf, C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    _check(lib().ppa_ipc_close(ptr))


def halo_publish(flag_ptr: int, epoch: int) -> None:
    _check(lib().ppa_halo_publish(flag_ptr, epoch))


def halo_pull(peers_ptr: int, npeers: int, max_count: int, x_ext, epoch: int,
              error_ptr: int) -> None:
    _check(lib().ppa_halo_pull(peers_ptr, npeers, max_count, _ptr(x_ext), epoch, error_ptr))


def grid2_slab_pass(nd, nx, ny, nz, vals, zo0, zo1, kind, a0, a1, b0, x, y, xl=0, zl0=0,
                    fl=0, xr=0, fr=0, epoch=0, err=0, own=0) -> None:
    """The sharded box-grid pass with the halo planes read from the
    neighbours' buffers inside the kernel (ppa_grid2_slab_pass; kind 0: two
    real roots, 1: a conjugate pair, 2: one real root)."""
    v = np.ascontiguousarray(vals, dtype=np.float64)
    _check(lib().ppa_grid2_slab_pass(nd, nx, ny, nz, _np_ptr(v), zo0, zo1, int(kind), a0, a1, b0,
                                     _ptr(x), _ptr(y), xl or None, zl0, fl or None, xr or None,
                                     fr or None, epoch, err or None, own or None))


def grid2_slab_chain(nd, nx, ny, nz, vals, zo0, zo1, passes, buf0, buf1, xl=(0, 0), zl0=0,
                     fl=0, xr=(0, 0), fr=0, epoch0=0, err=0, own=0) -> int:
    """All passes [(kind, a0, a1, b0), ...] of one sharded pi(A)v in one call
    (ppa_grid2_slab_chain); returns the role (0, 1) holding the result."""
    v = np.ascontiguousarray(vals, dtype=np.float64)
    k = len(passes)
    kinds = np.array([p[0] for p in passes] or [0], dtype=np.int32)
    a0, a1, b0 = (np.array([p[i] for p in passes] or [0.0], dtype=np.float64) for i in (1, 2, 3))
    role = C.c_int()
    _check(lib().ppa_grid2_slab_chain(nd, nx, ny, nz, _np_ptr(v), zo0, zo1, k,
                                      kinds.ctypes.data_as(_ip), _np_ptr(a0), _np_ptr(a1),
                                      _np_ptr(b0), _ptr(buf0), _ptr(buf1), xl[0] or None,
                                      xl[1] or None, zl0, fl or None, xr[0] or None,
                                      xr[1] or None, fr or None, epoch0, err or None, own or None,
                                      C.byref(role)))
    return role.value


# ------------------------------------------------------------------ solver --
@dataclass
class SolveConfig:
    """SolveConfig (inc/solver.hpp:21-58)."""

    m: int = 50
    k: int = 20
    nev: int = 15
    degree: int = 0
    rtol_multiplier: float = 1e-8
    rtol_absolute: Optional[float] = None
    variant: str = "ritz"
    stability: str = "off"
    double_d1: int = 0
    double_d2: int = 0
    max_cycles: int = 100
    seed: int = 1
    allow_nev_above_k: bool = False
    damping: str = "off"          # off | auto_heuristic | forced
    damping_alpha: float = 0.0
    damping_power: int = 1
    check_mid_cycle: bool = False
    mid_cycle_stride: int = 5
    stagnation_stop: bool = False
    stagnation_window: int = 5
    stagnation_rtol: float = 0.01
    want_eigenvectors: bool = False
    orthogonalization: str = "dcgs2"  # dcgs2 (delayed CGS2, default) | cgs2
    reference: Sequence[complex] = field(default_factory=list)

    def _c(self, use_double: bool) -> _SolveConfigC:
        damp = {"off": 0, "auto_heuristic": 1, "forced": 2}[self.damping]
        return _SolveConfigC(self.m, self.k, self.nev, self.degree, self.rtol_multiplier,
                             self.rtol_absolute or 0.0, 1 if self.variant == "harmonic" else 0,
                             1 if self.stability == "pof_auto" else 0, self.double_d1,
                             self.double_d2, 1 if use_double else 0, self.max_cycles, self.seed,
                             1 if self.allow_nev_above_k else 0, damp, self.damping_alpha,
                             self.damping_power, int(self.check_mid_cycle),
                             self.mid_cycle_stride, int(self.stagnation_stop),
                             self.stagnation_window, self.stagnation_rtol,
                             int(self.want_eigenvectors),
                             {"cgs2": 0, "dcgs2": 1}[self.orthogonalization])


def _solve(a: LinearOperator, cfg: SolveConfig, use_double: bool) -> dict:
    cap_nev, cap_roots, cap_cyc = max(cfg.nev, 1), 4096, max(cfg.max_cycles, 1)
    bufs = {k: np.zeros(cap_nev) for k in ("eig_re", "eig_im", "residuals")}
    conv = np.zeros(cap_nev, dtype=np.int32)
    roots = {k: np.zeros(cap_roots) for k in ("poly_re", "poly_im", "inner_re", "inner_im")}
    cyc = np.zeros(cap_cyc)
    r = _SolveResultC()
    r.cap_nev, r.cap_roots, r.cap_cycles = cap_nev, cap_roots, cap_cyc
    for k, v in {**bufs, **roots}.items():
        setattr(r, k, v.ctypes.data_as(_dp))
    r.converged_flags = conv.ctypes.data_as(_ip)
    r.cycle_max_residual = cyc.ctypes.data_as(_dp)
    evec = None
    if cfg.want_eigenvectors:
        evec = np.zeros((2, cap_nev, a.dim()))
        r.evec_re = evec[0].ctypes.data_as(_dp)
        r.evec_im = evec[1].ctypes.data_as(_dp)
        r.evec_ld = a.dim()
    c = cfg._c(use_double)
    _check(lib().ppa_solve(a._h, C.byref(c), C.byref(r)))
    ne = min(r.n_eig, cap_nev)
    eig = bufs["eig_re"][:ne] + 1j * bufs["eig_im"][:ne]
    out = {
        "eigenvalues": eig,
        "residuals": bufs["residuals"][:ne].copy(),
        "converged_flags": conv[:ne].astype(bool),
        "converged": bool(r.converged),
        "cycles": r.cycles,
        "composite_degree": r.composite_degree,
        "poly": roots["poly_re"][:r.n_poly] + 1j * roots["poly_im"][:r.n_poly],
        "poly_base_degree": r.poly_base_degree,
        "inner_poly": roots["inner_re"][:r.n_inner] + 1j * roots["inner_im"][:r.n_inner],
        "rtol": r.rtol,
        "max_err": r.max_err,
        "norm_estimate": r.norm_estimate,
        "cost": {"mvps": r.cost.mvps, "dots": r.cost.dots, "vops": r.cost.vops,
                 "nnzr": r.cost.nnzr},
        "cycle_max_residual": cyc[:r.n_cycles].copy(),
        "discarded_probes": r.discarded_probes,
        "timing": {"total": r.t_total, "setup": r.t_setup, "extend": r.t_extend,
                   "check": r.t_check, "restart": r.t_restart},
    }
    if evec is not None:
        out["eigenvectors"] = (evec[0, :ne] + 1j * evec[1, :ne]).T.copy()
    if cfg.reference:
        ref = np.asarray(cfg.reference, dtype=np.complex128)
        out["correct_count"] = int(sum(
            1 for z, ok in zip(eig, out["converged_flags"])
            if ok and np.any(np.abs(z - ref) <= 1e-6 * np.abs(ref))))
    return out


def check_ideal_order(mu, nev: int) -> bool:
    """check_ideal_order (inc/solver.hpp:99)."""
    re, im = _roots(mu)
    h = C.c_int()
    _check(lib().ppa_check_ideal_order(_np_ptr(re), _np_ptr(im), len(re), nev, C.byref(h)))
    return bool(h.value)


def damping_heuristic(a: LinearOperator, cfg: SolveConfig, rec: Optional[CostRecord] = None):
    """damping_heuristic (inc/solver.hpp:105-106): the polynomial it settles on."""
    cap = max(8 * cfg.degree, 64)
    re, im = np.zeros(cap), np.zeros(cap)
    nr = C.c_int()
    rec = rec if rec is not None else CostRecord()
    c = cfg._c(False)
    _check(lib().ppa_damping_heuristic(a._h, C.byref(c), _np_ptr(re), _np_ptr(im), cap,
                                       C.byref(nr), C.byref(rec)))
    return re[:nr.value] + 1j * im[:nr.value]


def make_callback_operator(dim: int, apply, mvps_per_apply: int = 1,
                           nnzr: float = 0.0) -> LinearOperator:
    """A caller-defined device operator (ppa_op_create_callback): the
    reference's LinearOperator plugin point (inc/operators.hpp:49-76).
    ``apply(x_ptr, y_ptr, stream_ptr)`` must enqueue y = Op x on the CUDA
    stream ``stream_ptr`` for device vectors of length ``dim`` and return 0
    (or None); an exception or nonzero return fails the calling entry point."""

    def tramp(ctx, x, y, stream):
        try:
            rc = apply(x or 0, y or 0, stream or 0)
            return 0 if rc is None else int(rc)
        except Exception:  # noqa: BLE001  (reported as PPA_RUNTIME_ERROR)
            import traceback

            traceback.print_exc()
            return -1

    fn = _APPLY_FN(tramp)
    h = C.c_void_p()
    _check(lib().ppa_op_create_callback(dim, mvps_per_apply, C.c_double(nnzr), fn, None,
                                        C.byref(h)))
    return LinearOperator(h, keep=(fn, apply))


def make_block2(a: LinearOperator) -> LinearOperator:
    """make_block2 (inc/operators.hpp:87): diag(A, A), 2 mvps per apply."""
    h = C.c_void_p()
    _check(lib().ppa_block2_operator(a._h, C.byref(h)))
    return LinearOperator(h, keep=(a,))


def make_shifted(a: LinearOperator, mu: float) -> LinearOperator:
    """make_shifted (inc/operators.hpp:90): v -> Av - mu v."""
    h = C.c_void_p()
    _check(lib().ppa_shifted_operator(a._h, C.c_double(mu), C.byref(h)))
    return LinearOperator(h, keep=(a,))


def build_two_vector_poly(a: LinearOperator, b1, b2, degree: int,
                          rec: Optional[CostRecord] = None) -> np.ndarray:
    """build_two_vector_poly (src/gmres_poly.cpp:228-264); b1, b2 device vectors."""
    re, im = np.zeros(max(degree, 1)), np.zeros(max(degree, 1))
    nr = C.c_int()
    rec = rec if rec is not None else CostRecord()
    _check(lib().ppa_build_two_vector_poly(a._h, _ptr(b1), _ptr(b2), degree, _np_ptr(re),
                                           _np_ptr(im), C.byref(nr), C.byref(rec)))
    return re[:nr.value] + 1j * im[:nr.value]


def damped_start(a: LinearOperator, b, alpha: float, power: int, out,
                 rec: Optional[CostRecord] = None):
    """damped_start (src/gmres_poly.cpp:266-283) into the device vector `out`."""
    rec = rec if rec is not None else CostRecord()
    _check(lib().ppa_damped_start(a._h, _ptr(b), C.c_double(alpha), power, _ptr(out),
                                  C.byref(rec)))
    return rec


def read_matrix_market(path: str) -> "CsrMatrix":
    """read_matrix_market (src/operators.cpp:246-305)."""
    h = C.c_void_p()
    _check(lib().ppa_read_matrix_market(str(path).encode(), C.byref(h)))
    return CsrMatrix(h)


def solve(a: LinearOperator, cfg: SolveConfig) -> dict:
    """solve (inc/solver.hpp:94)."""
    return _solve(a, cfg, False)


def solve_double(a: LinearOperator, cfg: SolveConfig) -> dict:
    """solve_double (inc/solver.hpp:111)."""
    return _solve(a, cfg, True)
