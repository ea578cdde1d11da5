"""The reference's plugin points at the C-ABI (include/ppa_b200.h):

* a caller-defined device operator (ppa_op_create_callback) - the abstract
  LinearOperator (inc/operators.hpp:49-76) that arnoldi_extend,
  build_gmres_poly and solve accept whatever its implementation;
* thick_restart(state, keep, k) with a caller-built keep set
  (ppa_arnoldi_restart_keep; inc/arnoldi.hpp:79-80), fed by ritz_pairs or
  harmonic_restart_selection (inc/arnoldi.hpp:58, 68-69)."""
import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

pytestmark = pytest.mark.gpu


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (no copy)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _stencil_apply(torch, N):
    """Matrix-free 7-point Laplacian (1/h^2 scaling, Dirichlet) in torch: the
    caller's own device code, run on the stream the library passes."""
    h2 = float((N + 1) ** 2)
    n = N ** 3

    def apply(xp, yp, sp):
        s = torch.cuda.ExternalStream(sp) if sp else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            x = torch.as_tensor(_DevView(xp, n), device="cuda").view(N, N, N)
            y = torch.as_tensor(_DevView(yp, n), device="cuda").view(N, N, N)
            t = 6.0 * x
            t[1:] -= x[:-1]
            t[:-1] -= x[1:]
            t[:, 1:] -= x[:, :-1]
            t[:, :-1] -= x[:, 1:]
            t[:, :, 1:] -= x[:, :, :-1]
            t[:, :, :-1] -= x[:, :, 1:]
            y.copy_(t * h2)
        return 0

    return apply


def test_callback_operator_info_and_apply(cuda):
    N = 12
    op = ppa.make_callback_operator(N ** 3, _stencil_apply(cuda, N), mvps_per_apply=1, nnzr=7.0)
    assert (op.dim(), op.mvps_per_apply(), op.nnzr(), op.kind()) == (N ** 3, 1, 7.0, "external")
    x = O.normal_vector(N ** 3, 3, 3)
    y = cuda.empty(N ** 3, dtype=cuda.float64, device="cuda")
    rec = op.apply(cuda.tensor(x, device="cuda"), y)
    assert rec.mvps == 1
    ref = O.csr_operator(O.Csr.laplacian_3d(N)).apply(x)
    assert np.allclose(y.cpu().numpy(), ref, rtol=1e-12, atol=1e-9 * np.abs(ref).max())


def test_callback_failure_is_runtime_error(cuda):
    op = ppa.make_callback_operator(100, lambda x, y, s: 7)
    y = cuda.empty(100, dtype=cuda.float64, device="cuda")
    with pytest.raises(RuntimeError, match="callback operator: apply returned 7"):
        op.apply(cuda.zeros(100, dtype=cuda.float64, device="cuda"), y)


def test_callback_wrapping_csr_is_bit_identical(cuda):
    # the generic path over a caller operator reproduces the CSR operator's
    # solve bit for bit (same polynomial, same Ritz values, same counters)
    P = ppa.CsrMatrix.convection_diffusion(40)
    A = ppa.make_csr_operator(P)
    cb = ppa.make_callback_operator(P.n, lambda x, y, s: ppa.spmv(A, x, y), 1, A.nnzr())
    cfg = ppa.SolveConfig(m=40, k=20, nev=8, degree=12, seed=5, max_cycles=60)
    r_csr, r_cb = ppa.solve(A, cfg), ppa.solve(cb, cfg)
    assert r_cb["converged"] and r_csr["converged"]
    assert np.array_equal(r_cb["poly"], r_csr["poly"])
    assert np.array_equal(r_cb["eigenvalues"], r_csr["eigenvalues"])
    assert r_cb["cost"] == r_csr["cost"] and r_cb["cycles"] == r_csr["cycles"]


def test_matrix_free_solve_matches_oracle(cuda):
    # a matrix-free stencil written by the caller drives the whole
    # polynomial-preconditioned solve; eigenvalues and matvec count match the
    # oracle's solve on the same operator in CSR form
    N = 20
    op = ppa.make_callback_operator(N ** 3, _stencil_apply(cuda, N), 1, 7.0)
    cfg = ppa.SolveConfig(m=30, k=15, nev=6, degree=15, seed=4, max_cycles=100)
    r = ppa.solve(op, cfg)
    o = O.solve(O.csr_operator(O.Csr.laplacian_3d(N)), 30, 15, 6, degree=15, seed=4,
                max_cycles=100)
    assert r["converged"] and o["converged"]
    assert np.all(r["residuals"] <= r["rtol"])
    got, ref = np.sort(r["eigenvalues"].real), np.sort(o["eigenvalues"].real)
    assert np.max(np.abs(got - ref) / ref) < 1e-8
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]
    # the polynomial build and Arnoldi ran on the callback (no CSR anywhere)
    roots, _ = ppa.build_gmres_poly(op, cuda.tensor(O.normal_vector(N ** 3, 1, 2),
                                                    device="cuda"), 10)
    oroots, _ = O.build_gmres_poly(O.csr_operator(O.Csr.laplacian_3d(N)),
                                   O.normal_vector(N ** 3, 1, 2), 10)
    assert np.max(np.abs(roots - oroots) / np.abs(oroots)) < 1e-8


def _state(cuda, P, m, seed=6):
    A = ppa.make_csr_operator(P)
    st = ppa.arnoldi_init(cuda.tensor(O.normal_vector(P.n, seed, 3), device="cuda"), P.n, m)
    st.extend(A, m)
    return A, st


@pytest.mark.parametrize("ordering", [ppa.SMALLEST_MAGNITUDE, ppa.LARGEST_MAGNITUDE,
                                      ppa.TARGET_ONE])
def test_restart_keep_equals_ritz_restart(cuda, ordering):
    # thick_restart with ritz_pairs(ordering) passed explicitly as the keep
    # set is the same restart as ppa_arnoldi_restart(ordering), bit for bit
    P = ppa.CsrMatrix.convection_diffusion(24)
    _, s1 = _state(cuda, P, 30)
    _, s2 = _state(cuda, P, 30)
    vals, res, G = s1.ritz_pairs_vectors(ordering)
    v2, r2 = s2.ritz_pairs(ordering)
    assert np.array_equal(vals, v2) and np.array_equal(res, r2)
    k1 = s1.thick_restart_keep(vals, G, 12)
    k2 = s2.thick_restart(12, ordering)
    assert k1 == k2 and np.array_equal(s1.H, s2.H)


def test_restart_keep_caller_selection(cuda):
    # a caller's own selection (every other real Ritz pair of the spectrum's
    # left end) restarts into a factorisation whose kept Ritz values are
    # exactly the selected ones and that stays an Arnoldi relation
    d = np.arange(1.0, 301.0)
    A = ppa.make_diagonal(d)
    st = ppa.arnoldi_init(cuda.tensor(O.normal_vector(300, 4, 3), device="cuda"), 300, 40)
    st.extend(A, 40)
    vals, _, G = st.ritz_pairs_vectors(ppa.SMALLEST_MAGNITUDE)
    pick = np.arange(0, 20, 2)
    kk = st.thick_restart_keep(vals[pick], G[:, pick], len(pick))
    assert kk == len(pick)
    kept = np.sort(np.linalg.eigvals(st.H[:kk, :kk]).real)
    assert np.allclose(kept, np.sort(vals[pick].real), rtol=1e-10)
    st.extend(A, 40)
    ld = st.ld
    buf = cuda.empty(41 * ld, dtype=cuda.float64, device="cuda")
    ppa.ts_combine(st.V_ptr, ld, 300, 41, cuda.tensor(np.eye(41).T.ravel(), device="cuda"), 41,
                   buf, ld)
    V = buf.cpu().numpy().reshape(41, ld)[:, :300].T
    assert np.linalg.norm(V.T @ V - np.eye(41)) < 1e-10
    assert np.linalg.norm(np.diag(d) @ V[:, :40] - V @ st.H) < 1e-9 * np.linalg.norm(st.H)


def test_restart_keep_harmonic_selection(cuda):
    # harmonic_restart_selection's set drives thick_restart from outside the
    # solver; the compressed basis stays orthonormal
    P = ppa.CsrMatrix.convection_diffusion(20)
    _, st = _state(cuda, P, 30)
    vals, res, G = st.harmonic_restart_selection(ppa.SMALLEST_MAGNITUDE)
    assert vals.size == 30 and np.all(res >= 0)
    kk = st.thick_restart_keep(vals, G, 10)
    assert kk in (9, 10) and st.cur_dim == kk


def test_restart_keep_errors(cuda):
    P = ppa.CsrMatrix.convection_diffusion(16)
    _, st = _state(cuda, P, 20)
    vals, _, G = st.ritz_pairs_vectors(ppa.SMALLEST_MAGNITUDE)
    with pytest.raises(ValueError, match="selection smaller than k"):
        st.thick_restart_keep(vals[:3], G[:, :3], 8)
    with pytest.raises(ValueError, match="bad k"):
        st.thick_restart_keep(vals, G, 20)
