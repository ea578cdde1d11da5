"""SPEC.md solver invariants on the device solve:
eigenvector consistency under pi(A), the spectral mapping on a diagonal
matrix, the cost bookkeeping identity, and determinism.  The independent
residual check (invariant 1) is test_gpu_solver_options.py::
test_eigenvectors_output.  The bookkeeping identity is pinned on the oracle
first (CPU)."""
import numpy as np
import pytest

from oracle import oracle as O

LAM = np.arange(1.0, 1001.0)


def _predicted_mvps(m, k, nev, degree, eff, cycles, norm_mvps):
    # poly build (degree mvps) + norm estimate + first cycle (m steps) + later
    # cycles (m - k steps after a k-vector thick restart), each step costing
    # eff base mvps, + one mvp per real Ritz check (nev per cycle)
    return degree + norm_mvps + eff * (m + (cycles - 1) * (m - k)) + cycles * nev


@pytest.mark.parametrize("m,k,nev,degree", [(30, 15, 10, 10), (40, 20, 15, 6), (50, 20, 15, 0)])
def test_bookkeeping_identity_oracle(m, k, nev, degree):
    r = O.solve(O.diagonal_operator(LAM), m, k, nev, degree=degree, seed=5, max_cycles=50)
    assert r["converged"]
    eff = len(r["poly"]) if degree else 1
    assert r["cost"]["mvps"] == _predicted_mvps(m, k, nev, degree, eff, r["cycles"], 0)


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,nev,degree", [(30, 15, 10, 10), (40, 20, 15, 6), (50, 20, 15, 0)])
def test_bookkeeping_identity_diag(cuda, m, k, nev, degree):
    import paper_1806_08020_b200 as ppa

    r = ppa.solve(ppa.make_diagonal(LAM), ppa.SolveConfig(m=m, k=k, nev=nev, degree=degree,
                                                          seed=5, max_cycles=50))
    assert r["converged"]
    eff = len(r["poly"]) if degree else 1
    # diagonal operators take max|diag| as the norm: no power-iteration mvps
    assert r["cost"]["mvps"] == _predicted_mvps(m, k, nev, degree, eff, r["cycles"], 0)


@pytest.mark.gpu
def test_bookkeeping_identity_csr_stability(cuda):
    # symmetric CSR operator (real Ritz values: every restart keeps exactly k),
    # 5 power-iteration mvps for the norm, stability copies in eff
    import paper_1806_08020_b200 as ppa

    A = ppa.make_csr_operator(ppa.CsrMatrix.laplacian_3d(14))
    cfg = ppa.SolveConfig(m=30, k=15, nev=6, degree=12, stability="pof_auto", seed=2,
                          max_cycles=80)
    r = ppa.solve(A, cfg)
    assert r["converged"]
    eff = len(r["poly"])
    assert eff >= 12
    assert r["cost"]["mvps"] == _predicted_mvps(30, 15, 6, 12, eff, r["cycles"], 5)


@pytest.mark.gpu
def test_spectral_mapping_and_pi_consistency(cuda):
    # on diag(1..1000): each converged mu_j maps to the Ritz value of pi(A),
    # nu_j = y^H pi(A) y, within 1e-8 |nu_j|; and ||pi(A) y - nu y|| is small
    # (<= 100 rtol scale, scale = max |pi(lambda)| over the spectrum)
    import paper_1806_08020_b200 as ppa

    A = ppa.make_diagonal(LAM)
    r = ppa.solve(A, ppa.SolveConfig(m=40, k=20, nev=10, degree=10, seed=3, max_cycles=50,
                                     want_eigenvectors=True))
    assert r["converged"]
    roots = r["poly"]
    scale = max(abs(O.eval_poly(roots, x)) for x in LAM)
    Y = r["eigenvectors"]
    for j, mu in enumerate(r["eigenvalues"]):
        y = Y[:, j]
        py = np.zeros(len(LAM), dtype=np.complex128)
        for part, unit in ((y.real, 1.0), (y.imag, 1j)):
            out = cuda.empty(len(LAM), dtype=cuda.float64, device="cuda")
            ppa.apply_poly(roots, A, cuda.tensor(np.ascontiguousarray(part), device="cuda"), out)
            py += unit * out.cpu().numpy()
        nu = np.vdot(y, py)
        ev = O.eval_poly(roots, mu)
        assert abs(ev - nu) <= 1e-8 * abs(nu)
        assert np.linalg.norm(py - nu * y) <= 100 * r["rtol"] * scale


@pytest.mark.gpu
@pytest.mark.parametrize("ortho", ["cgs2", "dcgs2"])
def test_determinism(cuda, ortho):
    # fixed seed -> bitwise-identical EigResult across runs
    import paper_1806_08020_b200 as ppa

    A = ppa.make_csr_operator(ppa.CsrMatrix.convection_diffusion_const(60, 0.5))
    cfg = ppa.SolveConfig(m=40, k=20, nev=8, degree=15, seed=9, max_cycles=60,
                          orthogonalization=ortho, want_eigenvectors=True)
    a, b = ppa.solve(A, cfg), ppa.solve(A, cfg)
    for key in ("eigenvalues", "residuals", "poly", "cycle_max_residual", "eigenvectors"):
        assert np.array_equal(a[key], b[key]), key
    assert a["cost"] == b["cost"] and a["cycles"] == b["cycles"]
    assert a["norm_estimate"] == b["norm_estimate"] and a["rtol"] == b["rtol"]
