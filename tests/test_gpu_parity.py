"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact where the arithmetic allows (SpMV and the fused
polynomial factors reproduce the reference's operation order without FMA);
within the BASELINE tolerances elsewhere (pi(A)v 1e-12 relative 2-norm,
eigenvalues 1e-8 relative, mvps within 5%)."""
import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def dev(torch, x):
    return torch.tensor(np.asarray(x, dtype=np.float64), device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


MATRICES = [
    ("bidiag", lambda M: M.bidiagonal(777)),
    ("convdiff_ref", lambda M: M.convection_diffusion(37)),
    ("convdiff_const", lambda M: M.convection_diffusion_const(45, 0.5)),
    ("laplace3d", lambda M: M.laplacian_3d(17)),
    ("random_poisson", lambda M: M.random_poisson(20000, 16.0, 7)),
]


@pytest.mark.parametrize("name,gen", MATRICES)
def test_spmv_bit_exact(cuda, name, gen):
    P = gen(ppa.CsrMatrix)
    Q = gen(O.Csr)
    assert P.fingerprint() == Q.info()[2]
    A = ppa.make_csr_operator(P)
    Ao = O.csr_operator(Q)
    n = P.n
    x = O.normal_vector(n, 11, 9)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    rec = A.apply(dev(cuda, x), y)
    assert rec.mvps == 1
    assert np.array_equal(host(y), Ao.apply(x))


@pytest.mark.parametrize("name,gen", MATRICES)
@pytest.mark.parametrize("layout", ["csr_rowblock", "sell_unsorted_only", "sell_unpacked",
                                    "sell_packed"])
def test_spmv_other_layouts_bit_exact(cuda, monkeypatch, name, gen, layout):
    # the CSR row-block kernel (PPA_DISABLE_SELL), SELL without sigma sorting
    # (PPA_DISABLE_SIGMA: irregular rows fall back to the row-block path) and
    # SELL-32 without the packed / diagonal-coded streams, packed SELL-32
    # without the diagonal-coded one
    env = {"csr_rowblock": ["PPA_DISABLE_SELL"], "sell_unsorted_only": ["PPA_DISABLE_SIGMA"],
           "sell_unpacked": ["PPA_DISABLE_PACKED", "PPA_DISABLE_DIA"],
           "sell_packed": ["PPA_DISABLE_DIA"]}[layout]
    for e in env:
        monkeypatch.setenv(e, "1")
    P, Q = gen(ppa.CsrMatrix), gen(O.Csr)
    A = ppa.make_csr_operator(P)
    x = O.normal_vector(P.n, 4, 9)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    A.apply(dev(cuda, x), y)
    assert np.array_equal(host(y), O.csr_operator(Q).apply(x))
    roots = _roots_mixed()
    out = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, x), out)
    assert np.array_equal(host(out), O.apply_poly(roots, O.csr_operator(Q), x))


EXPECTED_LAYOUT = {
    # bidiagonal a_ii = i: 777 distinct values, width 2 -> packing would grow the stream
    "bidiag": ("sell32", 0),
    "convdiff_ref": ("dia_coded", None),
    "convdiff_const": ("dia_coded", 4),  # C, E, W, N = S
    "laplace3d": ("dia_coded", 2),
    # n = 20000: random offsets still fit int16; > 256 values -> fp64 stream
    "random_poisson": ("sell32_packed", 0),
}


@pytest.mark.parametrize("name,gen", MATRICES)
def test_layout_selection(cuda, name, gen):
    lay = ppa.make_csr_operator(gen(ppa.CsrMatrix)).layout()
    want, nd = EXPECTED_LAYOUT[name]
    assert lay["layout"] == want
    if nd is not None:
        assert lay["dict_size"] == nd


@pytest.mark.parametrize("cap,want", [("auto", "dia_coded"), ("csr", "csr"), ("sell32", "sell32"),
                                      ("sell32_packed", "sell32_packed"),
                                      ("dia_coded", "dia_coded")])
def test_layout_cap_bit_exact(cuda, cap, want):
    # ppa_csr_operator_layout: every cap computes the same bits
    P, Q = ppa.CsrMatrix.laplacian_3d(19), O.Csr.laplacian_3d(19)
    A = ppa.make_csr_operator(P, cap)
    assert A.layout()["layout"] == want
    x = O.normal_vector(P.n, 8, 1)
    roots = _roots_mixed()
    out = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, x), out)
    assert np.array_equal(host(out), O.apply_poly(roots, O.csr_operator(Q), x))


def _banded(n, offsets, vals, irregular=()):
    """Constant-diagonal band matrix; rows in `irregular` get a perturbed value."""
    rows, cols, vv = [], [], []
    for i in range(n):
        for o, v in zip(offsets, vals):
            j = i + o
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vv.append(v * (1.5 if i in irregular else 1.0))
    return rows, cols, vv


@pytest.mark.parametrize("offsets", [
    (-1, 0, 1),                                        # 3 diagonals: one code word
    (-41, -40, -39, -1, 0, 1, 39, 40, 41),             # 9-point: four code words
    tuple(range(-8, 9)),                               # 17 diagonals: coded form only
])
def test_dia_diagonal_counts_bit_exact(cuda, offsets):
    n = 6000
    vals = [float(k + 2) * (-1) ** k for k in range(len(offsets))]
    rows, cols, vv = _banded(n, offsets, vals, irregular={5, 1234, 4001})
    P = ppa.CsrMatrix.from_triplets(n, rows, cols, vv)
    Q = O.Csr.from_triplets(n, rows, cols, vv)
    A = ppa.make_csr_operator(P)
    assert A.layout()["layout"] == "dia_coded"
    x = O.normal_vector(n, 3, 3)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    A.apply(dev(cuda, x), y)
    assert np.array_equal(host(y), O.csr_operator(Q).apply(x))
    roots = _roots_mixed()
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, x), out)
    assert np.array_equal(host(out), O.apply_poly(roots, O.csr_operator(Q), x))
    # multi-RHS
    ld = (n + 31) // 32 * 32
    Y = np.zeros((3, ld))
    for j in range(3):
        Y[j, :n] = O.normal_vector(n, 40 + j, 1)
    AYd = cuda.zeros(3 * ld, dtype=cuda.float64, device="cuda")
    ppa.spmm(A, dev(cuda, Y.ravel()), ld, 3, AYd, ld)
    AY = host(AYd).reshape(3, ld)
    for j in range(3):
        assert np.array_equal(AY[j, :n], O.csr_operator(Q).apply(Y[j, :n]))


def _banded_csr(n, offsets, vals, irregular=()):
    """_banded as CSR arrays, vectorised (multi-million-row cases)."""
    offs = np.asarray(offsets)
    cols = np.arange(n)[:, None] + offs[None, :]
    keep = (cols >= 0) & (cols < n)
    v = np.broadcast_to(np.asarray(vals, dtype=np.float64), cols.shape).copy()
    v[list(irregular)] *= 1.5
    rp = np.concatenate([[0], np.cumsum(keep.sum(axis=1))]).astype(np.int32)
    return rp, cols[keep].astype(np.int32), v[keep]


@pytest.mark.parametrize("n,offsets", [
    (300 * 13 + 7, (-300, -1, 0, 1, 300)),               # centre in the middle, ragged tail
    (300 * 12, (-300, -1, 1, 300)),                      # even count: no centre reuse
    (256 * 9 + 100, (-256, -2, -1, 7, 256)),             # odd count, middle is not offset 0
    (400 * 10, (-400, -20, -1, 0, 1, 20, 400)),          # 7-point, 3-D-like
    (2048 * 1200 + 77, (-2048, -1, 0, 1, 2048)),         # enough warps for 8 planes per thread
])
def test_dia_march_bit_exact(cuda, n, offsets):
    # the marching sweep (outer diagonals +-D, D >= 256): SpMV, pi(A)v with
    # real and pair roots, and the complement, against the oracle
    vals = [float(k + 2) * (-1) ** k for k in range(len(offsets))]
    rp, ci, vv = _banded_csr(n, offsets, vals, irregular=[3, n // 2, n - 5])
    P = ppa.CsrMatrix.from_arrays(n, rp, ci, vv)
    Q = O.Csr.from_arrays(n, rp, ci, vv)
    A = ppa.make_csr_operator(P)
    assert A.layout()["layout"] == "dia_coded"
    x = O.normal_vector(n, 6, 3)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    A.apply(dev(cuda, x), y)
    assert np.array_equal(host(y), O.csr_operator(Q).apply(x))
    roots = _roots_mixed()
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, x), out)
    assert np.array_equal(host(out), O.apply_poly(roots, O.csr_operator(Q), x))
    T = ppa.make_poly_complement_operator(A, roots)
    T.apply(dev(cuda, x), out)
    assert np.array_equal(host(out), O.poly_operator(O.csr_operator(Q), roots, complement=True).apply(x))


def _edge_matrices():
    rng = np.random.default_rng(11)
    out = {}
    # ragged: every third row empty, the rest 1-9 entries near the diagonal
    n = 3000
    rows, cols, vals = [], [], []
    for i in range(n):
        if i % 3 == 0:
            continue
        for o in sorted(set(rng.integers(-40, 41, 1 + i % 9).tolist())):
            if 0 <= i + o < n:
                rows.append(i)
                cols.append(i + o)
                vals.append(float(rng.choice([-1.0, 2.5, 0.0, -0.0])))  # explicit zeros
    out["ragged_zeros"] = (n, rows, cols, vals)
    # one row, one entry
    out["n1"] = (1, [0], [0], [3.0])
    # last rows empty, first row dense-ish
    n = 700
    rows, cols, vals = [], [], []
    for j in range(0, n, 7):
        rows.append(0)
        cols.append(j)
        vals.append(1.0 + j)
    for i in range(1, n - 40):
        rows += [i, i]
        cols += [i - 1, i]
        vals += [-1.0, 2.0]
    out["tail_empty"] = (n, rows, cols, vals)
    out["all_empty"] = (40, [], [], [])  # nnz = 0: y = 0 (or the epilogue of 0)
    return out


EDGE = _edge_matrices()


@pytest.mark.parametrize("cap", ["auto", "csr", "sell32", "sell32_packed", "dia_coded"])
@pytest.mark.parametrize("name", sorted(EDGE))
def test_edge_matrices_every_layout(cuda, cap, name):
    n, rows, cols, vals = EDGE[name]
    P = ppa.CsrMatrix.from_triplets(n, rows, cols, vals)
    Q = O.Csr.from_triplets(n, rows, cols, vals)
    A = ppa.make_csr_operator(P, cap)
    x = O.normal_vector(n, 5, 5)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    A.apply(dev(cuda, x), y)
    assert np.array_equal(host(y), O.csr_operator(Q).apply(x))
    roots = _roots_mixed()
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, x), out)
    assert np.array_equal(host(out), O.apply_poly(roots, O.csr_operator(Q), x))


def test_empty_dimension_operator(cuda):
    # n = 0 is a valid CsrMatrix (src/operators.cpp:12-37): a no-op operator
    P = ppa.CsrMatrix.from_arrays(0, [0], [], [])
    A = ppa.make_csr_operator(P)
    assert A.dim() == 0
    x = cuda.empty(1, dtype=cuda.float64, device="cuda")
    y = cuda.empty(1, dtype=cuda.float64, device="cuda")
    rec = A.apply(x, y)
    assert rec.mvps == 1


def test_packed_fp64_values_and_perm(cuda):
    # packed stream without a value table (> 256 distinct values), sigma-sorted
    # rows of very different lengths, offsets near the int16 limit
    n = 70000
    rng = np.random.default_rng(5)
    rows, cols, vals = [], [], []
    for i in range(n):
        L = 9 + (i * 7919) % 13
        off = np.unique(rng.integers(-32767, 32768, L))
        c = np.clip(i + off, 0, n - 1)
        c = np.unique(c)
        rows += [i] * len(c)
        cols += list(c)
        vals += list(rng.standard_normal(len(c)))
    P = ppa.CsrMatrix.from_triplets(n, rows, cols, vals)
    Q = O.Csr.from_triplets(n, rows, cols, vals)
    A = ppa.make_csr_operator(P)
    lay = A.layout()
    assert lay["layout"] == "sell32_packed" and lay["dict_size"] == 0 and lay["sigma"] > 1
    x = O.normal_vector(n, 2, 2)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    A.apply(dev(cuda, x), y)
    assert np.array_equal(host(y), O.csr_operator(Q).apply(x))
    roots = _roots_mixed()
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, x), out)
    assert np.array_equal(host(out), O.apply_poly(roots, O.csr_operator(Q), x))


def test_csr_matrix_multiply_uncounted(cuda):
    # CsrMatrix::multiply (inc/operators.hpp:27-28): plain y = A x
    P, Q = ppa.CsrMatrix.convection_diffusion(33), O.Csr.convection_diffusion(33)
    x = O.normal_vector(P.n, 1, 2)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    P.multiply(dev(cuda, x), y)
    assert np.array_equal(host(y), O.csr_operator(Q).apply(x))


def test_spmv_long_rows(cuda):
    # rows longer than one row block (2048 nnz) take the block-reduction path
    n = 6000
    rows, cols, vals = [], [], []
    rng = np.random.default_rng(3)
    for i in range(n):
        L = 5000 if i in (17, 4000) else 3
        cs = np.unique(rng.integers(0, n, L))
        rows += [i] * len(cs)
        cols += list(cs)
        vals += list(rng.standard_normal(len(cs)))
    P = ppa.CsrMatrix.from_triplets(n, rows, cols, vals)
    Q = O.Csr.from_triplets(n, rows, cols, vals)
    x = O.normal_vector(n, 1, 1)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.make_csr_operator(P).apply(dev(cuda, x), y)
    ref = O.csr_operator(Q).apply(x)
    assert rel(host(y), ref) < 1e-14


def _roots_real(k, lo=1.0, hi=3000.0):
    return O.leja_order(np.linspace(lo, hi, k))


def _roots_mixed():
    r = [4000.0, 2500 + 300j, 2500 - 300j, 900.0, 120 + 40j, 120 - 40j, 15.0, 3000.0]
    return O.leja_order(r)


@pytest.mark.parametrize("kind", ["real", "mixed", "pairs_only", "single_pair", "empty"])
def test_apply_poly_bit_exact(cuda, kind):
    P = ppa.CsrMatrix.convection_diffusion(40)
    Q = O.Csr.convection_diffusion(40)
    roots = {"real": _roots_real(12), "mixed": _roots_mixed(),
             "pairs_only": [300 + 20j, 300 - 20j, 50 + 5j, 50 - 5j],
             "single_pair": [300 + 20j, 300 - 20j], "empty": []}[kind]
    A = ppa.make_csr_operator(P)
    Ao = O.csr_operator(Q)
    n = P.n
    v = O.normal_vector(n, 5, 2)
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    rec = ppa.apply_poly(roots, A, dev(cuda, v), out)
    cost = np.zeros(3)
    ref = O.apply_poly(roots, Ao, v, cost)
    assert np.array_equal(host(out), ref), rel(host(out), ref)
    assert (rec.mvps, rec.vops) == (int(cost[0]), int(cost[2]))


@pytest.mark.parametrize("kind", ["real_even", "real_odd", "mixed", "pairs_only"])
@pytest.mark.parametrize("complement", [False, True])
def test_large_chains_bit_exact(cuda, kind, complement):
    # n >= 65536 chains (two-factor passes on the stencils, the generic
    # pair path on the reference's jump-coefficient matrix) equal the oracle
    # bit for bit, and repeated applies stay exact
    gens = {"real_even": lambda M: M.laplacian_3d(48), "real_odd": lambda M: M.laplacian_3d(48),
            "mixed": lambda M: M.convection_diffusion(300),
            "pairs_only": lambda M: M.convection_diffusion_const(260, 0.5)}
    roots = {"real_even": _roots_real(10, 10.0, 60000.0), "real_odd": _roots_real(9, 10.0, 60000.0),
             "mixed": O.leja_order([4.5e6, 2e6 + 3e5j, 2e6 - 3e5j, 9e5, 1.2e5 + 4e4j,
                                    1.2e5 - 4e4j, 1.5e4, 3e6, 6e5]),
             "pairs_only": [3e5 + 2e4j, 3e5 - 2e4j, 5e4 + 5e3j, 5e4 - 5e3j]}[kind]
    P, Q = gens[kind](ppa.CsrMatrix), gens[kind](O.Csr)
    assert P.n >= 65536
    mk = ppa.make_poly_complement_operator if complement else ppa.make_poly_operator
    op = mk(ppa.make_csr_operator(P), roots)
    opo = O.poly_operator(O.csr_operator(Q), roots, complement)
    x = O.normal_vector(P.n, 6, 6)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    rec = op.apply(dev(cuda, x), y)
    cost = np.zeros(3)
    ref = opo.apply(x, cost)
    assert np.array_equal(host(y), ref), rel(host(y), ref)
    assert (rec.mvps, rec.vops) == (int(cost[0]), int(cost[2]))
    op.apply(dev(cuda, x), y)
    assert np.array_equal(host(y), ref)


def test_apply_poly_eigvec_matches_eval(cuda):
    # SPEC.md gmres_poly invariant: on eigenvectors of a diagonal A, apply = eval
    d = np.arange(1.0, 201.0)
    A = ppa.make_diagonal(d)
    roots = O.leja_order([150.0, 60 + 10j, 60 - 10j, 7.0])
    out = cuda.empty(200, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, np.ones(200)), out)
    want = np.array([ppa.eval_poly(roots, z).real for z in d])
    assert np.allclose(host(out), want, rtol=1e-13, atol=1e-13)


def test_apply_poly_malformed_pair_raises(cuda):
    A = ppa.make_diagonal([1.0, 2.0, 3.0])
    out = cuda.empty(3, dtype=cuda.float64, device="cuda")
    with pytest.raises(ppa.LogicError, match="without adjacent conjugate"):
        ppa.apply_poly([2 + 1j, 5.0, 2 - 1j], A, dev(cuda, np.ones(3)), out)


@pytest.mark.parametrize("complement", [False, True])
def test_poly_operator_and_complement(cuda, complement):
    P = ppa.CsrMatrix.laplacian_3d(12)
    Q = O.Csr.laplacian_3d(12)
    roots = _roots_mixed()
    op = (ppa.make_poly_complement_operator if complement else ppa.make_poly_operator)(
        ppa.make_csr_operator(P), roots)
    opo = O.poly_operator(O.csr_operator(Q), roots, complement)
    n = P.n
    assert op.mvps_per_apply() == len(roots)
    assert op.kind() == ("composite" if complement else "poly")
    x = O.normal_vector(n, 3, 3)
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    rec = op.apply(dev(cuda, x), y)
    cost = np.zeros(3)
    ref = opo.apply(x, cost)
    assert np.array_equal(host(y), ref)
    assert (rec.mvps, rec.vops) == (int(cost[0]), int(cost[2]))


@pytest.mark.parametrize("inner_kind", ["real", "mixed"])
def test_nested_double_polynomial(cuda, inner_kind):
    # pi2(tau(A)), tau = I - pi1(A) over CSR: each outer factor's axpy is
    # folded into the last inner launch (src/gmres_poly.cpp:129-143 over the
    # tau operator of src/gmres_poly.cpp:302-311); bit-identical to the
    # oracle's generic sequence, with its counters.
    P = ppa.CsrMatrix.convection_diffusion_const(30, 0.5)
    Q = O.Csr.convection_diffusion_const(30, 0.5)
    r1 = _roots_real(5, 100.0, 7000.0) if inner_kind == "real" else O.leja_order(
        [150.0, 3000.0 + 400.0j, 3000.0 - 400.0j, 6500.0])
    r2 = O.leja_order([0.9, 0.5 + 0.1j, 0.5 - 0.1j, 0.2])
    tau = ppa.make_poly_complement_operator(ppa.make_csr_operator(P), r1)
    op = ppa.make_poly_operator(tau, r2)
    opo = O.poly_operator(O.poly_operator(O.csr_operator(Q), r1, True), r2)
    assert op.mvps_per_apply() == len(r1) * len(r2)
    x = O.normal_vector(P.n, 8, 8)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    rec = op.apply(dev(cuda, x), y)
    cost = np.zeros(3)
    ref = opo.apply(x, cost)
    assert np.array_equal(host(y), ref)
    assert (rec.mvps, rec.vops) == (int(cost[0]), int(cost[2]))


def test_apply_host_e2e(cuda):
    P = ppa.CsrMatrix.laplacian_3d(10)
    roots = _roots_real(6, 10.0, 1100.0)
    op = ppa.make_poly_operator(ppa.make_csr_operator(P), roots)
    x = O.normal_vector(P.n, 2, 2)
    y = op.apply_host(x)
    ref = O.apply_poly(roots, O.csr_operator(O.Csr.laplacian_3d(10)), x)
    assert np.array_equal(y, ref)
    # batched host API: H2D / compute / D2H overlapped across vectors
    X = np.stack([O.normal_vector(P.n, 2, s) for s in range(5)])
    rec = ppa.CostRecord()
    Y = op.apply_host_batch(X, rec=rec)
    assert rec.mvps == 5 * len(roots)
    Ao = O.csr_operator(O.Csr.laplacian_3d(10))
    for i in range(5):
        assert np.array_equal(Y[i], O.apply_poly(roots, Ao, X[i]))
    XT = cuda.from_numpy(X).pin_memory()
    YT = cuda.empty_like(XT).pin_memory()
    op.apply_host_batch(XT, YT)
    assert np.array_equal(YT.numpy(), Y)


@pytest.mark.parametrize("gen,deg", [(lambda M: M.laplacian_3d(14), 20),
                                     (lambda M: M.convection_diffusion(30), 15),
                                     (lambda M: M.random_poisson(3000, 16.0, 2), 12)])
def test_build_gmres_poly_vs_oracle(cuda, gen, deg):
    P, Q = gen(ppa.CsrMatrix), gen(O.Csr)
    n = P.n
    b = O.normal_vector(n, 1, 2)
    cost = np.zeros(3)
    oroots, otrunc = O.build_gmres_poly(O.csr_operator(Q), b, deg, cost)
    for ortho in ("cgs2", "dcgs2"):
        rec = ppa.CostRecord()
        roots, trunc = ppa.build_gmres_poly(ppa.make_csr_operator(P), dev(cuda, b), deg, rec,
                                            orthogonalization=ortho)
        assert trunc == otrunc and len(roots) == len(oroots)
        # same Leja permutation, roots equal to roundoff (CGS2 / DCGS2 vs MGS2)
        assert np.max(np.abs(roots - oroots) / np.abs(oroots)) < 1e-8, ortho
        assert (rec.mvps, rec.dots, rec.vops) == tuple(int(c) for c in cost)
    # minimum-residual property: ||pi(A) b|| equals the GMRES(d) residual
    A = ppa.make_csr_operator(P)
    out = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, dev(cuda, b), out)
    Ad = _dense(P)
    beta = np.linalg.norm(b)
    V = np.zeros((n, deg + 1))
    Hh = np.zeros((deg + 1, deg))
    V[:, 0] = b / beta
    for j in range(deg):
        w = Ad @ V[:, j]
        for _ in range(2):
            c = V[:, :j + 1].T @ w
            w -= V[:, :j + 1] @ c
            Hh[:j + 1, j] += c
        Hh[j + 1, j] = np.linalg.norm(w)
        V[:, j + 1] = w / Hh[j + 1, j]
    e1 = np.zeros(deg + 1)
    e1[0] = beta
    y = np.linalg.lstsq(Hh, e1, rcond=None)[0]
    gm = np.linalg.norm(e1 - Hh @ y)
    assert abs(np.linalg.norm(host(out)) - gm) / gm < 1e-6


@pytest.fixture(params=["cgs2", "dcgs2"])
def ortho(request):
    """Run a test under classic CGS2 and under delayed CGS2 (arnoldi.cpp)."""
    return request.param


def test_arnoldi_relation_and_orthonormality(cuda, ortho):
    P = ppa.CsrMatrix.convection_diffusion(32)
    n = P.n
    A = ppa.make_csr_operator(P)
    m = 40
    v0 = O.normal_vector(n, 3, 3)
    rec = ppa.CostRecord()
    st = ppa.arnoldi_init(dev(cuda, v0), n, m, rec)
    st.set_orthogonalization(ortho)
    st.extend(A, m, rec)
    assert st.cur_dim == m and not st.breakdown
    Vh = _read_V(cuda, st, n, m + 1)
    H = st.H
    E = Vh.T @ Vh - np.eye(m + 1)
    assert np.linalg.norm(E) <= 1e-10
    Ad = _dense(P)
    R = Ad @ Vh[:, :m] - Vh @ H
    assert np.linalg.norm(R) <= 1e-9 * max(1.0, np.linalg.norm(H))
    # counters: MGS2 charges
    assert rec.mvps == m
    assert rec.dots == 1 + sum(2 * (j + 1) + 1 for j in range(m))
    # H matches the oracle's MGS2 Hessenberg to roundoff
    ref = O.arnoldi(O.csr_operator(O.Csr.convection_diffusion(32)), v0, m)
    assert np.max(np.abs(H - ref["H"])) <= 1e-9 * np.abs(ref["H"]).max()


def _dense(P):
    n = P.n
    rp, ci, v = P.arrays()
    D = np.zeros((n, n))
    for i in range(n):
        D[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return D


def _read_V(torch, st, n, cols):
    ld = st.ld
    buf = torch.empty(cols * ld, dtype=torch.float64, device="cuda")
    # device-to-device copy via the C-ABI combine kernel with G = I
    G = dev(torch, np.eye(cols).T.ravel())
    ppa.ts_combine(st.V_ptr, ld, n, cols, G, cols, buf, ld)
    torch.cuda.synchronize()
    return host(buf).reshape(cols, ld)[:, :n].T.copy()


def test_arnoldi_m100(cuda, ortho):
    # the largest basis the north star keeps on the host side (m <= 100):
    # widest TMA tiles (c up to 100) in every CGS kernel
    P = ppa.CsrMatrix.convection_diffusion(45)
    n = P.n
    A = ppa.make_csr_operator(P)
    m = 100
    rec = ppa.CostRecord()
    st = ppa.arnoldi_init(dev(cuda, O.normal_vector(n, 9, 3)), n, m, rec)
    st.set_orthogonalization(ortho)
    st.extend(A, m, rec)
    assert st.cur_dim == m and not st.breakdown
    Vh = _read_V(cuda, st, n, m + 1)
    assert np.linalg.norm(Vh.T @ Vh - np.eye(m + 1)) <= 1e-10
    R = _dense(P) @ Vh[:, :m] - Vh @ st.H
    assert np.linalg.norm(R) <= 1e-9 * max(1.0, np.linalg.norm(st.H))


def test_breakdown_diag_e1(cuda, ortho):
    # diag[1..6] with e1 breaks down at dimension 1
    A = ppa.make_diagonal(np.arange(1.0, 7.0))
    e1 = np.zeros(6)
    e1[0] = 1.0
    rec = ppa.CostRecord()
    st = ppa.arnoldi_init(dev(cuda, e1), 6, 3, rec)
    st.set_orthogonalization(ortho)
    st.extend(A, 3, rec)
    assert st.breakdown and st.cur_dim == 1 and st.H[1, 0] == 0.0
    # counters as the reference's MGS2: one application, no scaling charge
    assert rec.mvps == 1 and rec.dots == 1 + 3


def test_thick_restart_preserves_pairs(cuda, ortho):
    # retained pairs keep value and residual across a restart
    d = np.arange(1.0, 101.0)
    A = ppa.make_diagonal(d)
    v0 = O.normal_vector(100, 4, 3)
    st = ppa.arnoldi_init(dev(cuda, v0), 100, 20)
    st.set_orthogonalization(ortho)
    st.extend(A, 20)
    vals, res = st.ritz_pairs(ppa.SMALLEST_MAGNITUDE)
    kk = st.thick_restart(8, ppa.SMALLEST_MAGNITUDE)
    assert kk == 8 and st.cur_dim == 8
    H = st.H
    ev = np.sort(np.linalg.eigvals(H[:8, :8]).real)
    assert np.allclose(ev, np.sort(vals[:8].real), rtol=1e-10, atol=1e-10)
    # orthonormality after compression
    Vh = _read_V(cuda, st, 100, 9)
    assert np.linalg.norm(Vh.T @ Vh - np.eye(9)) < 1e-10
    st.extend(A, 20)
    Vh = _read_V(cuda, st, 100, 21)
    R = np.diag(d) @ Vh[:, :20] - Vh @ st.H
    assert np.linalg.norm(R) <= 1e-9 * max(1.0, np.linalg.norm(st.H))


def test_extend_after_restart_nonsymmetric(cuda, ortho):
    # after thick_restart H's leading block is full, not Hessenberg
    # (src/arnoldi.cpp:326-333); the next extend must keep the Arnoldi
    # relation A V_m = V_{m+1} H to roundoff under either orthogonalisation
    P = ppa.CsrMatrix.convection_diffusion(30)
    n = P.n
    A = ppa.make_csr_operator(P)
    m, k = 30, 12
    st = ppa.arnoldi_init(dev(cuda, O.normal_vector(n, 6, 3)), n, m)
    st.set_orthogonalization(ortho)
    Ad = _dense(P)
    for cycle in range(3):
        st.extend(A, m)
        assert st.cur_dim == m and not st.breakdown
        Vh = _read_V(cuda, st, n, m + 1)
        H = st.H
        assert np.linalg.norm(Vh.T @ Vh - np.eye(m + 1)) <= 1e-10
        R = Ad @ Vh[:, :m] - Vh @ H
        assert np.linalg.norm(R) <= 1e-9 * max(1.0, np.linalg.norm(H)), (cycle, np.linalg.norm(R))
        kk = st.thick_restart(k, ppa.SMALLEST_MAGNITUDE)
        # the restarted block is genuinely non-Hessenberg for this matrix
        assert np.abs(np.tril(st.H[:kk + 1, :kk], -2)).max() > 1e-6 * np.abs(st.H).max()


def test_breakdown_late_invariant_subspace(cuda, ortho):
    # breakdown at step 4 (invariant subspace of dimension 4): DCGS2 finds it
    # one step late and must un-charge the extra application
    d = np.arange(1.0, 301.0)
    v0 = np.zeros(300)
    v0[[3, 50, 120, 299]] = [1.0, 2.0, -1.0, 0.5]
    A = ppa.make_diagonal(d)
    rec = ppa.CostRecord()
    st = ppa.arnoldi_init(dev(cuda, v0), 300, 10, rec)
    st.set_orthogonalization(ortho)
    st.extend(A, 10, rec)
    assert st.breakdown and st.cur_dim == 4
    assert rec.mvps == 4
    assert rec.dots == 1 + sum(2 * (j + 1) + 1 for j in range(4))
    assert rec.vops == 2 + sum(4 * (j + 1) + 2 for j in range(3)) + 4 * 4 + 1
    ev = np.sort(np.linalg.eigvals(st.H[:4, :4]).real)
    assert np.allclose(ev, [4.0, 51.0, 121.0, 300.0], rtol=1e-10)


def test_poly_solve_both_orthogonalisations(cuda, ortho):
    # the polynomial-preconditioned solve on a nonsymmetric matrix agrees with
    # the oracle under either orthogonalisation
    P = ppa.CsrMatrix.convection_diffusion(40)
    A = ppa.make_csr_operator(P)
    cfg = ppa.SolveConfig(m=40, k=20, nev=8, degree=12, seed=5, max_cycles=60,
                          orthogonalization=ortho)
    r = ppa.solve(A, cfg)
    o = O.solve(O.csr_operator(O.Csr.convection_diffusion(40)), 40, 20, 8, degree=12, seed=5,
                max_cycles=60)
    assert r["converged"] and o["converged"]
    assert np.all(r["residuals"] <= r["rtol"])
    got, ref = np.sort_complex(r["eigenvalues"]), np.sort_complex(o["eigenvalues"])
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-8
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]


def test_solve_config1_vs_oracle(cuda):
    P = ppa.CsrMatrix.config(1)
    A = ppa.make_csr_operator(P)
    cfg = ppa.config_solve_config(1)
    r = ppa.solve(A, cfg)
    o = O.solve(O.csr_operator(O.Csr.config(1)), m=30, k=15, nev=10, degree=10, seed=1)
    assert r["converged"] and o["converged"]
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1.0, 11.0), rtol=1e-8)
    assert np.max(np.abs(np.sort(r["eigenvalues"].real) - np.sort(o["eigenvalues"].real))
                  / np.arange(1.0, 11.0)) < 1e-8
    assert np.all(r["residuals"] <= r["rtol"])
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]
    assert np.allclose(r["poly"], o["poly"], rtol=1e-8)


def test_solve_diag1000_one_cycle(cuda):
    # SPEC.md:374 / PAPER Example 4: diag[1..1000], Arnoldi(50,20), d=10, nev=15
    A = ppa.make_diagonal(np.arange(1.0, 1001.0))
    r = ppa.solve(A, ppa.SolveConfig(m=50, k=20, nev=15, degree=10, seed=1))
    assert r["converged"] and r["cycles"] <= 2
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1.0, 16.0), rtol=1e-8)


def test_solve_double_small_vs_oracle(cuda):
    P = ppa.CsrMatrix.convection_diffusion_const(60, 0.5)
    Q = O.Csr.convection_diffusion_const(60, 0.5)
    cfg = ppa.SolveConfig(m=30, k=15, nev=8, double_d1=5, double_d2=6, seed=3, max_cycles=40)
    r = ppa.solve_double(ppa.make_csr_operator(P), cfg)
    o = O.solve(O.csr_operator(Q), m=30, k=15, nev=8, double=(5, 6), seed=3, max_cycles=40)
    assert r["converged"] and o["converged"]
    assert r["composite_degree"] == o["composite_degree"] == 30
    assert np.allclose(r["inner_poly"], o["inner_poly"], rtol=1e-8)
    assert np.all(r["residuals"] <= r["rtol"])
    # Constant-Peclet convection-diffusion is similar to a symmetric matrix only
    # through a diagonal scaling with cond ~ 3^((N-1)/2) (1e14 at N = 60): Ritz
    # values certified by tiny residuals sit in the pseudospectrum, where a
    # residual r moves them by up to kappa * r.  CPU (MGS2) and GPU (CGS2)
    # roundoff therefore give different, equally valid, certified pairs
    # (DESIGN.md "Non-normal configs"); compare loosely.
    a, b = np.sort(r["eigenvalues"].real), np.sort(o["eigenvalues"].real)
    assert np.max(np.abs(a - b) / np.abs(b)) < 1e-4
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]


@pytest.mark.parametrize("name,gen", MATRICES)
@pytest.mark.parametrize("p", [1, 5, 8, 13])
def test_spmm_columns_bit_exact(cuda, name, gen, p):
    # multi-RHS SpMM of the convergence check: every column equals the oracle SpMV
    P, Q = gen(ppa.CsrMatrix), gen(O.Csr)
    A = ppa.make_csr_operator(P)
    n = P.n
    ld = (n + 31) // 32 * 32
    Y = np.zeros((p, ld))
    for j in range(p):
        Y[j, :n] = O.normal_vector(n, 30 + j, 7)
    Yd = dev(cuda, Y.ravel())
    AYd = cuda.zeros(p * ld, dtype=cuda.float64, device="cuda")
    ppa.spmm(A, Yd, ld, p, AYd, ld)
    AY = host(AYd).reshape(p, ld)
    Ao = O.csr_operator(Q)
    for j in range(p):
        assert np.array_equal(AY[j, :n], Ao.apply(Y[j, :n]))


@pytest.mark.parametrize("d,p,inplace", [(5, 1, False), (40, 15, False), (40, 20, True),
                                         (41, 21, True), (7, 7, True), (60, 45, True),
                                         (60, 45, False), (129, 33, False), (33, 30, True)])
def test_ts_combine_shapes(cuda, d, p, inplace):
    # V*G (thick restart in place, Ritz vectors out of place): every
    # accumulator bucket, the >32-column passes and the wide in-place path,
    # against the host product (fma-chain roundoff: 1e-13 relative per term)
    n = 3001
    ld = (n + 31) // 32 * 32
    rng = np.random.default_rng(d * 100 + p)
    Vh = np.zeros((d + 1, ld))
    Vh[:, :n] = rng.standard_normal((d + 1, n))
    Gh = rng.standard_normal((p, d))  # column-major d x p
    V = cuda.tensor(Vh.ravel(), device="cuda")
    if inplace:
        ppa.ts_combine(V, ld, n, d, cuda.tensor(Gh.ravel(), device="cuda"), p, V, ld)
        got = host(V).reshape(d + 1, ld)[:p, :n]
    else:
        Out = cuda.zeros(p * ld, dtype=cuda.float64, device="cuda")
        ppa.ts_combine(V, ld, n, d, cuda.tensor(Gh.ravel(), device="cuda"), p, Out, ld)
        got = host(Out).reshape(p, ld)[:, :n]
    ref = Gh @ Vh[:d, :n]
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref)) * d
    if inplace:  # columns p..d untouched
        assert np.array_equal(host(V).reshape(d + 1, ld)[p:, :n], Vh[p:, :n])


@pytest.mark.parametrize("d,p,inplace,n", [(40, 20, True, 4099), (40, 15, False, 3001),
                                           (41, 21, True, 128), (7, 3, False, 1000),
                                           (96, 32, True, 2177), (60, 45, True, 1500),
                                           (30, 20, False, 257)])
def test_ts_combine_tma_equals_register_kernel(cuda, monkeypatch, d, p, inplace, n):
    # the TMA-fed V*G (cgs.cu k_combine_tma) and the register kernel
    # (tallskinny.cu) sum each output over j in the same order with fma:
    # identical bits, in place and out of place, ragged last tiles
    ld = (n + 31) // 32 * 32
    rng = np.random.default_rng(d * 7 + p + n)
    Vh = np.zeros((d + 1, ld))
    Vh[:, :n] = rng.standard_normal((d + 1, n))
    Gh = rng.standard_normal((p, d))
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("PPA_COMBINE_TMA", flag)
        V = cuda.tensor(Vh.ravel(), device="cuda")
        G = cuda.tensor(Gh.ravel(), device="cuda")
        if inplace:
            ppa.ts_combine(V, ld, n, d, G, p, V, ld)
            outs.append(host(V).reshape(d + 1, ld)[:, :n])
        else:
            Out = cuda.zeros(p * ld, dtype=cuda.float64, device="cuda")
            ppa.ts_combine(V, ld, n, d, G, p, Out, ld)
            outs.append(host(Out).reshape(p, ld)[:, :n])
    assert np.array_equal(outs[0], outs[1])
    ref = Gh @ Vh[:d, :n]
    assert np.max(np.abs(outs[0][:p] - ref)) <= 1e-13 * np.max(np.abs(ref)) * d
