"""Solver-level known-answer examples from SPEC.md that need a whole solve (or a
whole polynomial build) on the paper's example spectra: Example 7's outlying
root and its stability copy, Example 9's double polynomial (with and without
stability roots), the d1 = 1 reduction of solve_double, Example 4's skewed
two-vector start, and the damping heuristic's halving on an adversarial
spectrum.  Oracle pins on CPU; the product against the same pins (and the
oracle) on the GPU."""
import numpy as np
import pytest

from oracle import oracle as O

# PAPER.md:938 (Example 7): 0.1, 0.2, ..., 9.9, 10, 11, ..., 9909, 20000
EX7 = np.concatenate([np.arange(1, 100) / 10.0, np.arange(10.0, 9910.0), [20000.0]])
EX7_SMALLEST = np.sort(EX7)[:15]


def _example4_starts(seed):
    # PAPER.md section 5 / SPEC.md:291: diag[1..1000], b1 with its last 100
    # components scaled by 0.01 (skewed away from the top of the spectrum)
    b1 = O.normal_vector(1000, 5 + seed, 2)
    b1[-100:] *= 0.01
    return b1, O.normal_vector(1000, 16 + seed, 2)


# ------------------------------------------------------------ oracle pins --
def test_example7_outlying_root_and_one_copy():
    # d = 15, b = all-ones -> a root at 20000 whose pof exceeds
    # 1e4, so add_stability_roots appends exactly one copy of it
    assert len(EX7) == 10000 and EX7[98:101].tolist() == [9.9, 10.0, 11.0]
    roots, _ = O.build_gmres_poly(O.diagonal_operator(EX7), np.ones(10000), 15)
    j = int(np.argmin(np.abs(roots - 20000.0)))
    assert abs(roots[j] - 20000.0) < 1e-9 * 20000.0
    rep = O.compute_pof(roots)
    assert 4.0 < rep["log10_pof"][j] < 18.0  # one copy: ceil((lg - 4)/14) = 1
    assert rep["copies_needed"][j] == 1 and rep["total_copies"] == 1
    aug = O.add_stability_roots(roots)
    assert len(aug) == 16 and aug[-1] == roots[j]


def test_example9_double_converges_in_two_cycles():
    # Example-7 matrix, d1 = 6, d2 = 20, Arnoldi(50,20), nev = 15
    r = O.solve(O.diagonal_operator(EX7), 50, 20, 15, double=(6, 20), seed=1)
    assert r["converged"] and r["cycles"] <= 2
    assert r["composite_degree"] == 120
    assert np.allclose(np.sort(r["eigenvalues"].real), EX7_SMALLEST, rtol=1e-8)


def test_example9_variant_needs_stability_roots():
    # d1 = 5, d2 = 20 without stability roots -> no progress in 50
    # cycles; with the pof-auto double root -> about two cycles
    A = O.diagonal_operator(EX7)
    bad = O.solve(A, 50, 20, 15, double=(5, 20), seed=1, max_cycles=50)
    assert not bad["converged"] and bad["cycles"] == 50
    assert bad["max_err"] > 1e3 * bad["rtol"]
    good = O.solve(A, 50, 20, 15, double=(5, 20), seed=1, stability=True)
    assert good["converged"] and good["cycles"] <= 3
    assert np.allclose(np.sort(good["eigenvalues"].real), EX7_SMALLEST, rtol=1e-8)


def test_solve_double_d1_is_scaled_single():
    # d1 = 1 -> tau(A) = A / theta1; the outer polynomial is the
    # single polynomial of the scaled operator: same eigenpairs, same cycles
    A = O.diagonal_operator(np.arange(1.0, 1001.0))
    dbl = O.solve(A, 50, 20, 15, double=(1, 10), seed=3)
    one = O.solve(A, 50, 20, 15, degree=10, seed=3)
    assert dbl["converged"] and one["converged"]
    assert len(dbl["inner_poly"]) == 1 and dbl["composite_degree"] == 10
    assert dbl["cycles"] == one["cycles"]
    assert np.allclose(np.sort(dbl["eigenvalues"].real), np.sort(one["eigenvalues"].real),
                       rtol=1e-8)
    # the scaling behind it: the GMRES polynomial of A / theta1 from the same
    # start vector has the roots of A's polynomial divided by theta1
    th = dbl["inner_poly"][0].real
    b = O.normal_vector(1000, 3, 2)
    r1, _ = O.build_gmres_poly(A, b, 10)
    rs, _ = O.build_gmres_poly(O.diagonal_operator(np.arange(1.0, 1001.0) / th), b, 10)
    assert np.allclose(np.sort_complex(rs * th), np.sort_complex(r1), rtol=1e-8)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_example4_skewed_two_vector(seed):
    # the skewed b1 alone gives a polynomial that needs many
    # Arnoldi(50,20) cycles on pi(A); the two-vector polynomial needs <= 2
    A = O.diagonal_operator(np.arange(1.0, 1001.0))
    b1, b2 = _example4_starts(seed)
    single, _ = O.build_gmres_poly(A, b1, 10)
    two = O.build_two_vector_poly(A, b1, b2, 10)
    cyc = {}
    for name, roots in (("single", single), ("two", two)):
        r = O.solve(O.poly_operator(A, roots, complement=True), 50, 20, 15, degree=0, seed=3,
                    max_cycles=50)
        assert r["converged"]
        nu = np.sort(np.abs([1.0 - O.eval_poly(roots, x) for x in np.arange(1.0, 1001.0)]))
        assert np.allclose(np.sort(np.abs(r["eigenvalues"])), nu[:15], rtol=1e-8)
        cyc[name] = r["cycles"]
    assert cyc["two"] <= 2 < 5 < cyc["single"]


def test_damping_halves_on_adversarial_spectrum():
    # d = 40 far too large for a 100-fold cluster of width 1e-3:
    # undamped and Ab-damped probes fail, d halves down to 1, and the solve
    # still terminates converged
    d = np.concatenate([np.linspace(1.0, 1.001, 100), np.linspace(2.0, 3.0, 100)])
    r = O.solve(O.diagonal_operator(d), 50, 20, 15, degree=40, seed=7, damping=1,
                max_cycles=30)
    assert r["converged"]
    assert 1 <= r["composite_degree"] < 40 and r["discarded"] >= 3
    # and Example 6 at d = 200 settles after halving (200 -> 100 -> 50)
    r6 = O.solve(O.diagonal_operator(np.arange(1.0, 10001.0)), 50, 20, 15, degree=200, seed=7,
                 damping=1, max_cycles=30)
    assert r6["converged"] and r6["composite_degree"] in (50, 100)
    assert np.allclose(np.sort(r6["eigenvalues"].real), np.arange(1.0, 16.0), rtol=1e-8)


# ----------------------------------------------------------------- GPU parity --
@pytest.mark.gpu
def test_example7_pof_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    A = ppa.make_diagonal(EX7)
    roots, _ = ppa.build_gmres_poly(A, cuda.ones(10000, dtype=cuda.float64, device="cuda"), 15)
    oroots, _ = O.build_gmres_poly(O.diagonal_operator(EX7), np.ones(10000), 15)
    assert np.max(np.abs(roots - oroots) / np.abs(oroots)) < 1e-8
    j = int(np.argmin(np.abs(roots - 20000.0)))
    rep = ppa.compute_pof(roots)
    assert rep["copies_needed"][j] == 1 and rep["total_copies"] == 1
    aug = ppa.add_stability_roots(roots)
    assert len(aug) == 16 and aug[-1] == roots[j]


@pytest.mark.gpu
def test_example9_double_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    A = ppa.make_diagonal(EX7)
    r = ppa.solve_double(A, ppa.SolveConfig(m=50, k=20, nev=15, double_d1=6, double_d2=20,
                                            seed=1))
    assert r["converged"] and r["cycles"] <= 2 and r["composite_degree"] == 120
    assert np.allclose(np.sort(r["eigenvalues"].real), EX7_SMALLEST, rtol=1e-8)
    o = O.solve(O.diagonal_operator(EX7), 50, 20, 15, double=(6, 20), seed=1)
    assert r["cycles"] == o["cycles"] and r["cost"]["mvps"] == o["cost"]["mvps"]
    # the variant: no progress without stability roots, ~2 cycles with them
    bad = ppa.solve_double(A, ppa.SolveConfig(m=50, k=20, nev=15, double_d1=5, double_d2=20,
                                              seed=1, max_cycles=50))
    assert not bad["converged"] and bad["cycles"] == 50
    assert bad["max_err"] > 1e3 * bad["rtol"]
    good = ppa.solve_double(A, ppa.SolveConfig(m=50, k=20, nev=15, double_d1=5, double_d2=20,
                                               seed=1, stability="pof_auto"))
    assert good["converged"] and good["cycles"] <= 3
    assert np.allclose(np.sort(good["eigenvalues"].real), EX7_SMALLEST, rtol=1e-8)


@pytest.mark.gpu
def test_solve_double_d1_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    A = ppa.make_diagonal(np.arange(1.0, 1001.0))
    dbl = ppa.solve_double(A, ppa.SolveConfig(m=50, k=20, nev=15, double_d1=1, double_d2=10,
                                              seed=3))
    one = ppa.solve(A, ppa.SolveConfig(m=50, k=20, nev=15, degree=10, seed=3))
    assert dbl["converged"] and one["converged"] and dbl["cycles"] == one["cycles"]
    assert np.allclose(np.sort(dbl["eigenvalues"].real), np.sort(one["eigenvalues"].real),
                       rtol=1e-8)


@pytest.mark.gpu
def test_example4_two_vector_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    lam = np.arange(1.0, 1001.0)
    A = ppa.make_diagonal(lam)
    b1, b2 = _example4_starts(1)
    two = ppa.build_two_vector_poly(A, cuda.tensor(b1, device="cuda"),
                                    cuda.tensor(b2, device="cuda"), 10)
    otwo = O.build_two_vector_poly(O.diagonal_operator(lam), b1, b2, 10)
    assert np.max(np.abs(two - otwo) / np.abs(otwo)) < 1e-8
    r = ppa.solve(ppa.make_poly_complement_operator(A, two),
                  ppa.SolveConfig(m=50, k=20, nev=15, degree=0, seed=3, max_cycles=50))
    assert r["converged"] and r["cycles"] <= 2
    nu = np.sort(np.abs([1.0 - O.eval_poly(two, x) for x in lam]))
    assert np.allclose(np.sort(np.abs(r["eigenvalues"])), nu[:15], rtol=1e-8)


@pytest.mark.gpu
def test_damping_halves_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    d = np.concatenate([np.linspace(1.0, 1.001, 100), np.linspace(2.0, 3.0, 100)])
    cfg = ppa.SolveConfig(m=50, k=20, nev=15, degree=40, seed=7, damping="auto_heuristic",
                          max_cycles=30)
    r = ppa.solve(ppa.make_diagonal(d), cfg)
    o = O.solve(O.diagonal_operator(d), 50, 20, 15, degree=40, seed=7, damping=1, max_cycles=30)
    assert r["converged"] and 1 <= r["composite_degree"] < 40
    assert r["composite_degree"] == o["composite_degree"]
    assert r["discarded_probes"] == o["discarded"]
