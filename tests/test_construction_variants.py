"""SURVEY §8f "next" rows: polynomial-construction variants (two start vectors,
damped starts, the damping heuristic; PAPER.md sections 5-6) and Matrix Market
ingest.  Oracle pins from SPEC.md's known-answer examples (CPU) and GPU parity
through the C-ABI."""
import os

import numpy as np
import pytest

from oracle import oracle as O

MM_IDENTITY = """%%MatrixMarket matrix coordinate real general
% 2x2 identity
2 2 2
1 1 1.0
2 2 1.0
"""
MM_SYM = """%%MatrixMarket matrix coordinate real symmetric
3 3 4
1 1 4.0
2 1 -1.0
3 2 -2.5
3 3 2.0
"""


# ------------------------------------------------------------ oracle pins --
def test_block2_kat():
    # A = diag[1,2], v = [1,0,0,1] -> [1,0,0,2]; +2 mvps per apply
    B = O.block2_operator(O.diagonal_operator([1.0, 2.0]))
    cost = np.zeros(3)
    assert np.array_equal(B.apply([1.0, 0.0, 0.0, 1.0], cost), [1.0, 0.0, 0.0, 2.0])
    assert cost[0] == 2


def test_shifted_kat():
    # mu = 0 identical; diag[1,2,3], mu = 2 -> eigenvalues {-1,0,1}
    A = O.diagonal_operator([1.0, 2.0, 3.0])
    x = np.array([0.3, -1.2, 2.5])
    assert np.array_equal(O.shifted_operator(A, 0.0).apply(x), A.apply(x))
    assert np.allclose(O.shifted_operator(A, 2.0).apply(x), np.array([-1.0, 0.0, 1.0]) * x)


def test_two_vector_kats():
    # b1 = b2 -> the single-vector polynomial of b1
    d = np.linspace(1.0, 50.0, 200)
    A = O.diagonal_operator(d)
    b = O.normal_vector(200, 4, 2)
    r2 = O.build_two_vector_poly(A, b, b, 6)
    r1, _ = O.build_gmres_poly(A, b, 6)
    assert np.allclose(np.sort_complex(r2), np.sort_complex(r1), rtol=1e-9)
    # SPEC.md:90 (n >= m+1 form): diag[1,2,3], b1 = e1, b2 = e2, d = 2 -> roots {1,2}
    A3 = O.diagonal_operator([1.0, 2.0, 3.0])
    r = O.build_two_vector_poly(A3, [1.0, 0, 0], [0, 1.0, 0], 2)
    assert np.allclose(np.sort(r.real), [1.0, 2.0], rtol=1e-12)
    with pytest.raises(ValueError, match="zero starting vector"):
        O.build_two_vector_poly(A3, [0.0, 0, 0], [0, 1.0, 0], 2)


def test_damped_start_kats():
    # alpha = 0, power 1 -> Ab normalised
    d = np.array([1.0, 2.0, 3.0, 4.0])
    A = O.diagonal_operator(d)
    b = np.array([1.0, -1.0, 0.5, 2.0])
    w = O.damped_start(A, b, 0.0, 1)
    assert np.allclose(w, d * b / np.linalg.norm(d * b), rtol=1e-15)
    w2 = O.damped_start(A, b, 0.0, 2)
    assert np.allclose(w2, d * d * b / np.linalg.norm(d * d * b), rtol=1e-15)
    w3 = O.damped_start(A, b, 5.0, 1)
    t = d * b + 5.0 * b
    assert np.allclose(w3, t / np.linalg.norm(t), rtol=1e-15)
    with pytest.raises(ValueError, match="power"):
        O.damped_start(A, b, 0.0, 3)


def test_check_ideal_order_kats():
    # the Example 6 failure (values 13-15 non-monotone) -> false
    mu = list(range(1, 13)) + [68.83, 67.62, 68.72, 71.74, 67.26, 67.86, 84.61, 72.80]
    assert not O.check_ideal_order(mu, 15)
    # clean buffer -> true
    assert O.check_ideal_order([1, 2, 3, 4, 5, 10, 11, 12, 13, 14, 15], 5)
    # nev = k -> monotonicity only
    assert O.check_ideal_order([1, 2, 3], 3)
    assert not O.check_ideal_order([1, 3, 2], 3)


def test_matrix_market_reader(tmp_path):
    p = tmp_path / "eye.mtx"
    p.write_text(MM_IDENTITY)
    rp, ci, v = O.read_matrix_market(p).arrays()
    assert list(rp) == [0, 1, 2] and list(ci) == [0, 1] and list(v) == [1.0, 1.0]
    s = tmp_path / "sym.mtx"
    s.write_text(MM_SYM)
    rp, ci, v = O.read_matrix_market(s).arrays()
    D = np.zeros((3, 3))
    for i in range(3):
        D[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    assert np.array_equal(D, [[4.0, -1.0, 0.0], [-1.0, 0.0, -2.5], [0.0, -2.5, 2.0]])
    bad = {"pattern.mtx": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n",
           "rect.mtx": "%%MatrixMarket matrix coordinate real general\n2 3 0\n",
           "oor.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
           "trunc.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
           "hdr.mtx": "%%MatrixMarket matrix array real general\n2 2\n"}
    msgs = {"pattern.mtx": "unsupported field", "rect.mtx": "square", "oor.mtx": "out of range",
            "trunc.mtx": "truncated", "hdr.mtx": "malformed header"}
    for name, txt in bad.items():
        f = tmp_path / name
        f.write_text(txt)
        with pytest.raises(Exception, match=msgs[name]):
            O.read_matrix_market(f)


def test_example6_damping_oracle():
    # PAPER.md 6.2-6.3 / SPEC.md:175 (scaled trial): diag[1..10000], Arnoldi(50,20),
    # d = 50: the undamped polynomial is overenthusiastic; the heuristic damps it
    A = O.diagonal_operator(np.arange(1.0, 10001.0))
    ref = np.arange(1.0, 16.0)
    damp = O.solve(A, 50, 20, 15, degree=50, seed=7, damping=1, max_cycles=40)
    assert damp["converged"]
    assert np.allclose(np.sort(damp["eigenvalues"].real), ref, rtol=1e-8)
    forced = O.solve(A, 50, 20, 15, degree=50, seed=7, damping=2, damping_power=1, max_cycles=40)
    assert forced["converged"]
    assert np.allclose(np.sort(forced["eigenvalues"].real), ref, rtol=1e-8)


# ----------------------------------------------------------------- GPU parity --
@pytest.mark.gpu
@pytest.mark.parametrize("gen", [lambda M: M.convection_diffusion(30),   # diagonal layout
                                 lambda M: M.bidiagonal(900),           # SELL-32
                                 lambda M: M.random_poisson(5000, 8.0, 3)])  # packed SELL
def test_block2_shifted_gpu(cuda, gen):
    import paper_1806_08020_b200 as ppa

    P = gen(ppa.CsrMatrix)
    Q = gen(O.Csr)
    n = P.n
    x = np.concatenate([O.normal_vector(n, 1, 1), O.normal_vector(n, 2, 1)])
    B = ppa.make_block2(ppa.make_csr_operator(P))
    assert B.dim() == 2 * n and B.mvps_per_apply() == 2 and B.kind() == "block2"
    y = cuda.empty(2 * n, dtype=cuda.float64, device="cuda")
    rec = B.apply(cuda.tensor(x, device="cuda"), y)
    assert rec.mvps == 2
    assert np.array_equal(y.cpu().numpy(), O.block2_operator(O.csr_operator(Q)).apply(x))
    S = ppa.make_shifted(ppa.make_csr_operator(P), 123.5)
    ys = cuda.empty(n, dtype=cuda.float64, device="cuda")
    rec = S.apply(cuda.tensor(x[:n], device="cuda"), ys)
    assert (rec.mvps, rec.vops) == (1, 1)
    assert np.array_equal(ys.cpu().numpy(), O.shifted_operator(O.csr_operator(Q), 123.5).apply(x[:n]))


@pytest.mark.gpu
def test_two_vector_and_damped_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    P = ppa.CsrMatrix.laplacian_3d(12)
    Q = O.Csr.laplacian_3d(12)
    n = P.n
    b1, b2 = O.normal_vector(n, 3, 2), O.normal_vector(n, 4, 2)
    A = ppa.make_csr_operator(P)
    rec = ppa.CostRecord()
    roots = ppa.build_two_vector_poly(A, cuda.tensor(b1, device="cuda"),
                                      cuda.tensor(b2, device="cuda"), 10, rec)
    cost = np.zeros(3)
    oroots = O.build_two_vector_poly(O.csr_operator(Q), b1, b2, 10, cost)
    assert np.max(np.abs(roots - oroots) / np.abs(oroots)) < 1e-8
    assert (rec.mvps, rec.dots, rec.vops) == tuple(int(c) for c in cost)
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    for alpha, power in ((0.0, 1), (2.5e3, 1), (0.0, 2)):
        rec = ppa.CostRecord()
        ppa.damped_start(A, cuda.tensor(b1, device="cuda"), alpha, power, out, rec)
        cost = np.zeros(3)
        ref = O.damped_start(O.csr_operator(Q), b1, alpha, power, cost)
        got = out.cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-14
        assert (rec.mvps, rec.dots, rec.vops) == tuple(int(c) for c in cost)


@pytest.mark.gpu
def test_ideal_order_and_damping_heuristic_gpu(cuda):
    import paper_1806_08020_b200 as ppa

    mu = list(range(1, 13)) + [68.83, 67.62, 68.72, 71.74, 67.26, 67.86, 84.61, 72.80]
    assert not ppa.check_ideal_order(mu, 15)
    assert ppa.check_ideal_order([1, 2, 3, 4, 5, 10, 11, 12], 5)
    A = ppa.make_diagonal(np.arange(1.0, 10001.0))
    cfg = ppa.SolveConfig(m=50, k=20, nev=15, degree=50, seed=7, damping="auto_heuristic",
                          max_cycles=40)
    r = ppa.solve(A, cfg)
    o = O.solve(O.diagonal_operator(np.arange(1.0, 10001.0)), 50, 20, 15, degree=50, seed=7,
                damping=1, max_cycles=40)
    assert r["converged"] and o["converged"]
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1.0, 16.0), rtol=1e-8)
    assert r["discarded_probes"] == o["discarded"]
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]
    roots = ppa.damping_heuristic(A, cfg)
    assert len(roots) >= 1


@pytest.mark.gpu
def test_matrix_market_product_reader(cuda, tmp_path):
    import paper_1806_08020_b200 as ppa

    s = tmp_path / "sym.mtx"
    s.write_text(MM_SYM)
    P = ppa.read_matrix_market(s)
    Q = O.read_matrix_market(s)
    for a, b in zip(P.arrays(), Q.arrays()):
        assert np.array_equal(a, b)
    with pytest.raises(RuntimeError, match="unsupported field"):
        f = tmp_path / "pat.mtx"
        f.write_text("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n")
        ppa.read_matrix_market(f)
