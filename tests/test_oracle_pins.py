"""Pins the CPU oracle (test infrastructure) against every known-answer
example SPEC.md gives for the hot path and against closed-form spectra
(SURVEY.md §4, §8c, Appendix B).  The reference ships no test vectors and
cannot be built here, so these are the pins."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- apply_poly
def test_apply_poly_kat_real_root():
    # roots {2}, A = diag[1,3], v = (1,1) -> (0.5, -0.5)
    out = O.apply_poly([2.0], O.diagonal_operator([1.0, 3.0]), [1.0, 1.0])
    assert np.array_equal(out, [0.5, -0.5])


def test_apply_poly_kat_conjugate_pair():
    # roots {1 +- i} on diag[2]: pi(2) = 1
    out = O.apply_poly([1 + 1j, 1 - 1j], O.diagonal_operator([2.0]), [1.0])
    assert out[0] == pytest.approx(1.0, abs=1e-15)


def test_apply_poly_eigenvectors_match_eval():
    # on eigenvectors of diagonal A, apply = eval to 1e-13
    d = np.linspace(0.5, 20.0, 40)
    roots = O.leja_order([19.0, 7 + 2j, 7 - 2j, 3.0, 0.9])
    out = O.apply_poly(roots, O.diagonal_operator(d), np.ones_like(d))
    want = np.array([O.eval_poly(roots, z).real for z in d])
    assert np.allclose(out, want, rtol=1e-13, atol=1e-13)


def test_apply_poly_counts_mvps():
    cost = np.zeros(3)
    O.apply_poly([3.0, 2 + 1j, 2 - 1j], O.diagonal_operator([1.0, 2.0, 4.0]), [1.0, 1.0, 1.0],
                 cost)
    assert cost[0] == 3 and cost[2] == 3  # 1 + 2 mvps, 1 + 2 axpys


def test_apply_poly_unpaired_complex_raises():
    with pytest.raises(O.OracleLogicError, match="adjacent conjugate"):
        O.apply_poly([2 + 1j, 3.0, 2 - 1j], O.diagonal_operator([1.0, 2.0]), [1.0, 1.0])


# ----------------------------------------------------------------- leja_order
def test_leja_kat():
    # {1, 10, 5} -> (10, 1, 5)
    assert np.array_equal(O.leja_order([1, 10, 5]), [10, 1, 5])
    # {2+i, 2-i, 7}: 7 first, then the adjacent pair
    o = O.leja_order([2 + 1j, 2 - 1j, 7])
    assert o[0] == 7 and {o[1], o[2]} == {2 + 1j, 2 - 1j}
    # single root
    assert np.array_equal(O.leja_order([4.0]), [4.0])


def test_leja_properties():
    # permutation, first element of maximal modulus
    rng = np.random.default_rng(0)
    r = rng.uniform(0.1, 100, 30)
    z = rng.uniform(1, 50, 10) + 1j * rng.uniform(0.5, 5, 10)
    roots = np.concatenate([r, z, np.conj(z)])
    o = O.leja_order(roots)
    assert sorted(o, key=lambda c: (c.real, c.imag)) == sorted(roots, key=lambda c: (c.real, c.imag))
    assert abs(o[0]) == np.max(np.abs(roots))
    # conjugates adjacent
    for i, c in enumerate(o):
        if abs(c.imag) > 1e-13 * abs(c) and c.imag > 0:
            assert o[i + 1] == np.conj(c)


def test_leja_brute_force_objective():
    # SPEC.md:258 [DERIVED] - greedy choice maximises sum of log distances
    roots = np.array([1.0, 3.0, 4.5, 9.0, 12.0])
    o = O.leja_order(roots)
    for k in range(1, len(o)):
        chosen = o[:k]
        scores = {c: np.sum(np.log(np.abs(c - chosen))) for c in roots if c not in chosen}
        assert o[k] == max(scores, key=scores.get)


def test_leja_errors():
    with pytest.raises(ValueError, match="empty"):
        O.leja_order([])
    with pytest.raises(ValueError, match="zero root"):
        O.leja_order([1.0, 0.0])


# --------------------------------------------------------------------- pof
def test_pof_kat():
    # {1, 2} -> pof = (0.5, 1)
    r = O.compute_pof([1.0, 2.0])
    assert np.allclose(10 ** r["log10_pof"], [0.5, 1.0], rtol=1e-15)


def test_pof_scale_invariance():
    # SPEC.md:288, 327
    roots = [3.0, 7.5, 11.0, 2 + 1j, 2 - 1j]
    a = O.compute_pof(roots)["log10_pof"]
    b = O.compute_pof(np.array(roots) * 1234.5)["log10_pof"]
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12)


def test_pof_needs_two_roots():
    with pytest.raises(ValueError):
        O.compute_pof([3.0])


# ---------------------------------------------------------- stability roots
def _pof_roots(lg):
    # two roots with pof(theta1) = |1 - theta1/theta2| = 10^lg
    return [1.0 - 10.0 ** lg, 1.0]


def test_stability_kat_one_copy():
    # pof 1e10 -> ceil((10-4)/14) = 1 copy, appended at the end
    roots = _pof_roots(10)
    out = O.add_stability_roots(roots)
    assert len(out) == 3 and out[-1] == roots[0] and out[0] == roots[0]


def test_stability_kat_two_copies():
    # pof 1e20 -> 2 copies; src/gmres_poly.cpp:209-222 placement
    roots = _pof_roots(20)
    out = O.add_stability_roots(roots)
    assert len(out) == 4
    assert list(out) == [roots[0], roots[0], roots[1], roots[0]]


def test_stability_threshold_and_eval_zero():
    # all pof <= 1e4: unchanged; SPEC.md:326 eval at a duplicated root is 0
    roots = [1.0, 2.0, 3.0]
    assert np.array_equal(O.add_stability_roots(roots), roots)
    aug = O.add_stability_roots(_pof_roots(12))
    assert O.eval_poly(aug, aug[0]) == 0


def test_stability_conjugate_group():
    # a complex root needing a copy brings its conjugate along (adjacent)
    big = 1e12 + 1e11j
    roots = [big, np.conj(big), 1.0]
    out = O.add_stability_roots(roots)
    assert len(out) == 5 and out[-2] == big and out[-1] == np.conj(big)


def test_eval_poly_kats():
    # pi(0) = 1; root of {1, 2} at z = 1 -> 0
    assert O.eval_poly([3.0, 5 + 1j, 5 - 1j], 0) == 1
    assert O.eval_poly([1.0, 2.0], 1.0) == 0


# --------------------------------------------------------- build / arnoldi
def test_build_gmres_poly_kat_exact_termination():
    # SPEC.md:246 (with n >= d+1): diag[1,2,3], b with e3 component
    # 0 -> d = 2 finds roots {1, 2} exactly and pi(A) b = 0
    A = O.diagonal_operator([1.0, 2.0, 3.0])
    b = np.array([1.0, 1.0, 0.0]) / np.sqrt(2)
    roots, trunc = O.build_gmres_poly(A, b, 2)
    assert np.allclose(np.sort(roots.real), [1.0, 2.0], rtol=1e-12)
    assert np.linalg.norm(O.apply_poly(roots, A, b)) < 1e-13


def test_build_gmres_poly_min_residual():
    # ||pi(A) b|| = GMRES(d) residual; beats random competitors
    d = np.linspace(1.0, 10.0, 60)
    A = O.diagonal_operator(d)
    b = O.normal_vector(60, 3, 2)
    roots, _ = O.build_gmres_poly(A, b, 5)
    res = np.linalg.norm(O.apply_poly(roots, A, b))
    K = np.stack([d ** k * b for k in range(1, 6)], axis=1)
    c = np.linalg.lstsq(K, b, rcond=None)[0]
    assert res == pytest.approx(np.linalg.norm(b - K @ c), rel=1e-10)
    rng = np.random.default_rng(1)
    for _ in range(200):
        rr = rng.uniform(0.5, 12.0, 5)
        assert res <= np.linalg.norm(O.apply_poly(rr, A, b)) * (1 + 1e-12)


def test_arnoldi_breakdown_kat():
    # diag with e1 breaks down at dimension 1
    A = O.diagonal_operator([1.0, 2.0, 3.0, 4.0])
    r = O.arnoldi(A, [1.0, 0.0, 0.0, 0.0], 3)
    assert r["breakdown"] and r["cur_dim"] == 1 and r["H"][1, 0] == 0.0


def test_arnoldi_relation_orthonormality():
    # SPEC.md:133-134, 196
    m = O.Csr.convection_diffusion(20)
    A = O.csr_operator(m)
    v0 = O.normal_vector(400, 1, 3)
    r = O.arnoldi(A, v0, 30, want_V=True)
    V, H = r["V"], r["H"]
    assert np.linalg.norm(V.T @ V - np.eye(31)) <= 1e-10
    rp, ci, vv = m.arrays()
    D = np.zeros((400, 400))
    for i in range(400):
        D[i, ci[rp[i]:rp[i + 1]]] = vv[rp[i]:rp[i + 1]]
    assert np.linalg.norm(D @ V[:, :30] - V @ H) <= 1e-9 * max(1, np.linalg.norm(H))


def test_harmonic_one_step_kat():
    # 1-step Arnoldi: the harmonic Ritz value is the root of the
    # degree-1 GMRES polynomial, argmin_theta ||(I - A/theta) b||, i.e.
    # theta = ||Ab||^2 / (b . Ab) (n >= m+1: diag[1,2,5])
    d = np.array([1.0, 2.0, 5.0])
    b = np.array([0.3, 0.5, 0.8])
    r = O.arnoldi(O.diagonal_operator(d), b, 1)
    theta = O.harmonic_from_H(r["H"], 1)[0]
    Ab = d * b
    assert theta.real == pytest.approx(Ab @ Ab / (b @ Ab), rel=1e-13)
    ts = np.linspace(theta.real * 0.9, theta.real * 1.1, 2001)
    res = [np.linalg.norm(b - Ab / t) for t in ts]
    assert abs(ts[int(np.argmin(res))] - theta.real) < 1e-3 * theta.real


def test_harmonic_reciprocal_rayleigh_ritz_kat():
    # diag[1..10], d = 4: harmonic Ritz values are reciprocals of
    # the Rayleigh-Ritz values of A^-1 on A K_d(A, b) (explicit projection)
    d = np.arange(1.0, 11.0)
    b = O.normal_vector(10, 5, 2)
    r = O.arnoldi(O.diagonal_operator(d), b, 4)
    hv = np.sort(O.harmonic_from_H(r["H"], 4).real)
    K = np.stack([d ** k * b for k in range(1, 5)], axis=1)  # A K_4
    Q, _ = np.linalg.qr(K)
    ev = np.linalg.eigvals(Q.T @ np.diag(1.0 / d) @ Q)
    assert np.allclose(hv, np.sort(1.0 / ev.real), rtol=1e-9)


def test_arnoldi_invariant_subspace_spectrum():
    # SPEC.md:152 (n >= m+1 form): diag[1,2,3,4] from (1,1,1,0)/sqrt3 spans an
    # invariant 3-dim space; H_3 has eigenvalues {1,2,3} to 1e-12
    r = O.arnoldi(O.diagonal_operator([1.0, 2.0, 3.0, 4.0]), np.array([1.0, 1, 1, 0]) / np.sqrt(3), 3)
    ev = np.sort(np.linalg.eigvals(r["H"][:3, :3]).real)
    assert np.allclose(ev, [1.0, 2.0, 3.0], atol=1e-12)
    assert np.allclose(r["H"][:3, :3], r["H"][:3, :3].T, atol=1e-12)  # symmetric op -> tridiagonal


def test_harmonic_full_dimension_equals_eigenvalues():
    # d = n: harmonic Ritz values are the exact eigenvalues
    d = np.array([1.0, 2.5, 4.0, 7.0, 11.0, 13.0])
    r = O.arnoldi(O.diagonal_operator(d), np.ones(6), 5, to_dim=5)
    hv = O.harmonic_from_H(r["H"], 5)
    # 5 of 6 eigenvalues after 5 steps is not exact; use the full 6-dim space via n = 7
    d7 = np.append(d, 20.0)
    r7 = O.arnoldi(O.diagonal_operator(d7), np.ones(7), 6, to_dim=6)
    hv = O.harmonic_from_H(r7["H"], 6)
    assert hv.shape == (6,)
    assert np.all(np.abs(hv.imag) < 1e-8)


# ---------------------------------------------------------------- solver
def test_solve_diag1000_one_cycle():
    # SPEC.md:374 / PAPER Example 4: diag[1..1000], Arnoldi(50,20), d=10, nev=15
    r = O.solve(O.diagonal_operator(np.arange(1.0, 1001.0)), m=50, k=20, nev=15, degree=10)
    assert r["converged"] and r["cycles"] <= 2
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1, 16), rtol=1e-8)


def test_solve_config1_analytic():
    # config 1: sigma(A) = {1..5000}; 10 smallest = 1..10 exactly
    r = O.solve(O.csr_operator(O.Csr.config(1)), m=30, k=15, nev=10, degree=10, seed=1)
    assert r["converged"]
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1, 11), rtol=1e-8)
    g = json.load(open(os.path.join(GOLDEN, "c1_solve.json")))
    assert r["cost"]["mvps"] == g["cost"]["mvps"] and r["cycles"] == g["cycles"]


def test_solve_laplace3d_small_analytic():
    # 7-point Laplacian N=12: lambda = 4/h^2 sum sin^2(i pi h / 2)
    N = 12
    h = 1.0 / (N + 1)
    s = 4 / h ** 2 * np.sin(np.arange(1, N + 1) * np.pi * h / 2) ** 2
    lam = np.sort((s[:, None, None] + s[None, :, None] + s[None, None, :]).ravel())
    r = O.solve(O.csr_operator(O.Csr.laplacian_3d(N)), m=30, k=15, nev=6, degree=12,
                stability=True, seed=2)
    assert r["converged"]
    got = np.sort(r["eigenvalues"].real)
    # multiset check against the analytic spectrum (multiplicities 1, 3, 3, ...)
    for z in got:
        assert np.min(np.abs(lam - z) / lam) < 1e-8


def test_solve_validation():
    A = O.diagonal_operator(np.arange(1.0, 101.0))
    with pytest.raises(ValueError, match="nev <= k"):
        O.solve(A, m=20, k=5, nev=8)
    with pytest.raises(ValueError, match="0 < k < m"):
        O.solve(A, m=20, k=20, nev=5)


# -------------------------------------------------------------- generators
def test_generator_shapes_and_fingerprints():
    fp = json.load(open(os.path.join(GOLDEN, "fingerprints.json")))
    n, nnz, f = O.Csr.config(1).info()
    assert (n, nnz, str(f)) == (5000, 9999, fp["config1"]["fingerprint"])
    # nnz formulas
    assert O.Csr.convection_diffusion_const(45, 0.5).info()[1] == 5 * 45 ** 2 - 4 * 45
    assert O.Csr.laplacian_3d(17).info()[1] == 7 * 17 ** 3 - 6 * 17 ** 2
    assert O.Csr.random_poisson(20000, 16.0, 7).info()[2] == int(
        fp["random_poisson20000_s7"]["fingerprint"])


def test_convdiff_ref_hand_assembled():
    # SPEC.md:59 [DERIVED] - grid_n = 2: 4x4 matrix from the stencil formulas
    rp, ci, v = O.Csr.convection_diffusion(2).arrays()
    h = 1 / 3
    c, e, w, s = 4 / h ** 2, -1 / h ** 2 + 20 / (2 * h), -1 / h ** 2 - 20 / (2 * h), -1 / h ** 2
    # y = (iy+1) h: row iy=0 (y=1/3) lower; iy=1 (y=2/3) upper (eps 100, c 2000)
    cu, eu, wu, su = 400 / h ** 2, -100 / h ** 2 + 2000 / (2 * h), -100 / h ** 2 - 2000 / (2 * h), -100 / h ** 2
    D = np.zeros((4, 4))
    for i in range(4):
        D[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    want = np.array([[c, e, s, 0], [w, c, 0, s], [su, 0, cu, eu], [0, su, wu, cu]])
    assert np.allclose(D, want, rtol=1e-15)


def test_csr_validate_errors():
    with pytest.raises(ValueError, match="strictly increasing"):
        O.Csr.from_arrays(2, [0, 2, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="out of range"):
        O.Csr.from_arrays(2, [0, 1, 2], [0, 5], [1.0, 1.0])
    with pytest.raises(ValueError, match="endpoints"):
        O.Csr.from_arrays(2, [0, 1, 3], [0, 1], [1.0, 1.0])


def test_from_triplets_sums_duplicates():
    m = O.Csr.from_triplets(3, [2, 0, 2, 0], [1, 0, 1, 2], [1.0, 2.0, 3.0, 4.0])
    rp, ci, v = m.arrays()
    assert list(rp) == [0, 2, 2, 3] and list(ci) == [0, 2, 1] and list(v) == [2.0, 4.0, 4.0]


def test_oracle_mid_cycle_and_stagnation():
    # SPEC.md:421 / SPEC.md:621 options of the solver restatement
    A = O.diagonal_operator(np.arange(1.0, 1001.0))
    full = O.solve(A, 50, 20, 15, degree=60, seed=1)
    mid = O.solve(A, 50, 20, 15, degree=60, seed=1, mid_cycle_stride=5)
    assert full["converged"] and mid["converged"] and mid["cycles"] == full["cycles"] == 2
    # the last cycle stops before m: fewer pi(A) applications in total
    assert mid["cost"]["mvps"] < 0.8 * full["cost"]["mvps"]
    stag = O.solve(A, 30, 15, 10, degree=0, seed=1, max_cycles=200, stagnation_window=3)
    best = np.minimum.accumulate(stag["cycle_max_residual"])
    assert stag["cycles"] < 200 and best[-1] > 0.99 * best[-4]
    assert np.all(best[3:-1] <= 0.99 * best[:-4])


def test_oracle_harmonic_variant_solve():
    # RestartVariant::harmonic (inc/solver.hpp:17, src/arnoldi.cpp:208-246):
    # restarts on harmonic Ritz vectors; same smallest eigenvalues
    A = O.diagonal_operator(np.arange(1.0, 1001.0))
    r = O.solve(A, 40, 20, 10, degree=0, seed=3, max_cycles=300, variant="harmonic")
    p = O.solve(A, 40, 20, 10, degree=0, seed=3, max_cycles=300)
    assert r["converged"] and p["converged"]
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1.0, 11.0), rtol=1e-8)
    assert r["cycles"] != p["cycles"] or r["cost"]["mvps"] != p["cost"]["mvps"] or \
        not np.array_equal(r["eigenvalues"], p["eigenvalues"])


def test_bench_timers_run():
    # the two timers bench.py's CPU arms call (orc_time_poly_factors,
    # orc_time_mgs2_step): small sizes, finite positive seconds
    A = O.csr_operator(O.Csr.laplacian_3d(10))
    roots = O.leja_order([40.0, 30.0 + 5.0j, 30.0 - 5.0j, 12.0])
    t = O.time_poly_factors(A, roots, 3, 1)
    assert 0.0 < t < 10.0
    t = O.time_mgs2_step(20000, 6, 2)
    assert 0.0 < t < 10.0
