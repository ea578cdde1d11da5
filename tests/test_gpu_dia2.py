"""Two polynomial factors per pass over stencil matrices (kernels/spmv_dia2.cu):
the temporally blocked pass must reproduce the factor chain of
src/gmres_poly.cpp:129-143 (and the complement of 306-308) bit for bit, with
the reference's counters, on every geometry it accepts; matrices it does not
accept must fall back to the single-factor launches."""
import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def dev(torch, x):
    return torch.tensor(np.asarray(x, dtype=np.float64), device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def _banded(n, offsets, vals, scaled=()):
    offs = np.asarray(offsets)
    cols = np.arange(n)[:, None] + offs[None, :]
    keep = (cols >= 0) & (cols < n)
    v = np.broadcast_to(np.asarray(vals, dtype=np.float64), cols.shape).copy()
    v[list(scaled)] *= 1.5
    rp = np.concatenate([[0], np.cumsum(keep.sum(axis=1))]).astype(np.int32)
    return rp, cols[keep].astype(np.int32), v[keep]


ROOTS = {
    "real_even": O.leja_order(np.linspace(10.0, 60000.0, 10)),
    "real_odd": O.leja_order(np.linspace(10.0, 60000.0, 9)),
    "mixed": O.leja_order([4.5e4, 2e4 + 3e3j, 2e4 - 3e3j, 9e3, 1.2e3 + 4e2j, 1.2e3 - 4e2j,
                           150.0, 3e4, 6e3]),
    "pairs_only": [3e4 + 2e3j, 3e4 - 2e3j, 5e3 + 5e2j, 5e3 - 5e2j],
    "single_real": [700.0],
}


def _check(cuda, P, Q, roots, complement, seed=4):
    mk = ppa.make_poly_complement_operator if complement else ppa.make_poly_operator
    op = mk(ppa.make_csr_operator(P), roots)
    opo = O.poly_operator(O.csr_operator(Q), roots, complement)
    x = O.normal_vector(P.n, seed, seed)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    rec = op.apply(dev(cuda, x), y)
    cost = np.zeros(3)
    ref = opo.apply(x, cost)
    got = host(y)
    assert np.array_equal(got, ref), np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert (rec.mvps, rec.vops) == (int(cost[0]), int(cost[2]))
    return op, x, ref


GEOMETRIES = [
    (300 * 13 + 8, (-300, -1, 0, 1, 300)),                 # 2-D 5-point, ragged last plane
    (256 * 9 + 100, (-256, -7, 0, 2, 256)),                # asymmetric in-plane offsets
    (300 * 12, (-300, 0, 300)),                            # 3-point
    (576 * 30, (-576, -24, -1, 0, 1, 24, 576)),            # 3-D 7-point (24^3-like)
    (1000 * 8, (-1000, -250, 0, 250, 1000)),               # in-plane offset D/4 (largest accepted)
    (64 * 40, (-64, -1, 0, 1, 64)),                        # smallest plane
    (2048 * 300 + 512, (-2048, -1, 0, 1, 2048)),           # many planes, partial last plane
    (25600 * 8, (-25600, -160, -1, 0, 1, 160, 25600)),     # config-3 plane, few planes
    (100 * 50, (-100, -10, -3, 0, 2, 5, 100)),             # 7 diagonals, irregular spacing
    (4096 * 10 + 64, (-4096, -64, -1, 0, 1, 64, 4096)),    # lines of 64: warp-shifted tiles
    (25600 * 6 + 2, (-25600, -160, -1, 0, 1, 160, 25600)), # last plane of 2 rows: the
                                                           # presence copies reach n + 4D + Dm
]


@pytest.mark.parametrize("n,offsets", GEOMETRIES)
@pytest.mark.parametrize("kind", ["real_even", "mixed"])
@pytest.mark.parametrize("complement", [False, True])
def test_dia2_geometries_bit_exact(cuda, n, offsets, kind, complement):
    vals = [float(k + 2) * (-1) ** k for k in range(len(offsets))]
    rp, ci, vv = _banded(n, offsets, vals)
    P = ppa.CsrMatrix.from_arrays(n, rp, ci, vv)
    Q = O.Csr.from_arrays(n, rp, ci, vv)
    lay = ppa.make_csr_operator(P).layout()
    assert lay["layout"] == "dia_coded" and lay["two_factor_pass"], lay
    _check(cuda, P, Q, ROOTS[kind], complement)


STENCILS = [
    ("laplace3d_24", lambda M: M.laplacian_3d(24)),
    ("laplace3d_40", lambda M: M.laplacian_3d(40)),
    ("laplace3d_64", lambda M: M.laplacian_3d(64)),       # lines of 64: warp-shifted tiles
    ("convdiff_300", lambda M: M.convection_diffusion_const(300, 0.5)),
]


@pytest.mark.parametrize("name,gen", STENCILS)
@pytest.mark.parametrize("kind", sorted(ROOTS))
@pytest.mark.parametrize("complement", [False, True])
def test_dia2_stencils_bit_exact(cuda, name, gen, kind, complement):
    P, Q = gen(ppa.CsrMatrix), gen(O.Csr)
    assert ppa.make_csr_operator(P).layout()["two_factor_pass"]
    _check(cuda, P, Q, ROOTS[kind], complement)


def test_dia2_matches_single_factor_chain(cuda, monkeypatch):
    # the fused and the single-factor chains agree on a long polynomial
    P = ppa.CsrMatrix.laplacian_3d(40)
    roots = O.leja_order(np.linspace(5.0, 2.0e4, 31))
    x = dev(cuda, O.normal_vector(P.n, 9, 9))
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PPA_DISABLE_DIA2", flag)
        A = ppa.make_csr_operator(P)
        assert A.layout()["two_factor_pass"] == (flag == "0")
        y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
        ppa.apply_poly(roots, A, x, y)
        outs.append(host(y))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("why", ["scaled_row", "odd_n", "odd_plane", "wide_middle", "few_planes",
                                 "even_count", "no_centre", "eight"])
def test_dia2_not_applicable_falls_back(cuda, why):
    n, offsets, scaled = {
        "even_count": (300 * 12, (-300, -1, 1, 300), []),
        "no_centre": (256 * 9 + 100, (-256, -2, -1, 7, 256), []),
        "eight": (100 * 50, (-100, -10, -3, -1, 0, 2, 5, 100), []),
        "scaled_row": (300 * 12, (-300, -1, 0, 1, 300), [5, 1000]),   # values off the default
        "odd_n": (300 * 12 + 1, (-300, -1, 0, 1, 300), []),
        "odd_plane": (301 * 12, (-301, -1, 0, 1, 301), []),
        "wide_middle": (400 * 12, (-400, -101, 0, 101, 400), []),     # 4 * 101 > 400
        "few_planes": (300 * 3, (-300, -1, 0, 1, 300), []),
    }[why]
    vals = [float(k + 2) * (-1) ** k for k in range(len(offsets))]
    rp, ci, vv = _banded(n, offsets, vals, scaled)
    P = ppa.CsrMatrix.from_arrays(n, rp, ci, vv)
    Q = O.Csr.from_arrays(n, rp, ci, vv)
    lay = ppa.make_csr_operator(P).layout()
    assert lay["layout"] == "dia_coded" and not lay["two_factor_pass"], lay
    _check(cuda, P, Q, ROOTS["mixed"], False)


def test_dia2_misaligned_vectors(cuda):
    # a chain whose input is not 16-byte aligned runs the single-factor
    # launches (the bulk copies need aligned sources); same bits
    P = ppa.CsrMatrix.laplacian_3d(24)
    Q = O.Csr.laplacian_3d(24)
    roots = ROOTS["real_even"]
    x = O.normal_vector(P.n, 2, 2)
    buf = cuda.zeros(P.n + 1, dtype=cuda.float64, device="cuda")
    buf[1:] = dev(cuda, x)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, ppa.make_csr_operator(P), buf[1:], y)
    assert np.array_equal(host(y), O.apply_poly(roots, O.csr_operator(Q), x))


@pytest.mark.parametrize("inner_kind", ["real_even", "real_odd", "mixed"])
def test_dia2_nested_double_polynomial(cuda, inner_kind):
    # phi(tau(A)): inner passes fused, the outer fold on a single launch
    P = ppa.CsrMatrix.convection_diffusion_const(300, 0.5)
    Q = O.Csr.convection_diffusion_const(300, 0.5)
    r1 = ROOTS[inner_kind]
    r2 = O.leja_order([0.9, 0.5 + 0.1j, 0.5 - 0.1j, 0.2])
    tau = ppa.make_poly_complement_operator(ppa.make_csr_operator(P), r1)
    op = ppa.make_poly_operator(tau, r2)
    opo = O.poly_operator(O.poly_operator(O.csr_operator(Q), r1, True), r2)
    x = O.normal_vector(P.n, 8, 8)
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    rec = op.apply(dev(cuda, x), y)
    cost = np.zeros(3)
    ref = opo.apply(x, cost)
    assert np.array_equal(host(y), ref)
    assert (rec.mvps, rec.vops) == (int(cost[0]), int(cost[2]))


def test_dia2_repeated_applies_and_graphs(cuda, monkeypatch):
    # repeated applies (ring barriers start fresh per launch) and the
    # CUDA-graph chain recording give the same bits
    P = ppa.CsrMatrix.laplacian_3d(40)
    Q = O.Csr.laplacian_3d(40)
    roots = ROOTS["mixed"]
    ref = O.poly_operator(O.csr_operator(Q), roots).apply(O.normal_vector(P.n, 3, 3))
    for graphs in ("0", "1"):
        monkeypatch.setenv("PPA_CHAIN_GRAPHS", graphs)
        op = ppa.make_poly_operator(ppa.make_csr_operator(P), roots)
        x = dev(cuda, O.normal_vector(P.n, 3, 3))
        y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
        for _ in range(3):
            op.apply(x, y)
            assert np.array_equal(host(y), ref)


def _fuzz_case(seed):
    rng = np.random.default_rng(1000 + seed)
    nd = int(rng.choice([3, 5, 7]))
    D = int(rng.choice([64, 96, 130, 256, 400, 1000, 2048]))
    side = (nd - 3) // 2  # in-plane offsets on each side of the centre
    dm_cap = max(2, D // 4)

    def draw():
        vals = set()
        if side and rng.integers(0, 2):
            vals.add(1)  # the +-1 neighbours of 2-D/3-D stencils (immediate offsets)
        while len(vals) < side:
            vals.add(int(rng.integers(1, dm_cap + 1)))
        return sorted(vals)

    neg, pos = draw(), draw()
    offsets = [-D] + [-v for v in reversed(neg)] + [0] + pos + [D]
    planes = int(rng.integers(4, 40))
    n = D * planes + int(rng.integers(0, D))
    n += n & 1
    vals = [float(v) for v in rng.choice([-1.0, 2.5, -0.75, 4.0, 0.5, -3.0], size=nd)]
    kind = str(rng.choice(["real_even", "real_odd", "mixed", "pairs_only"]))
    return n, tuple(offsets), vals, kind, bool(rng.integers(0, 2))


@pytest.mark.parametrize("seed", range(40))
def test_dia2_fuzz_bit_exact(cuda, seed):
    # seeded stencil geometries (plane widths, in-plane offsets up to D/4,
    # 3/5/7 points, ragged last planes, values per diagonal) and root mixes:
    # the two-factor pass must reproduce the oracle bit for bit
    n, offsets, vals, kind, complement = _fuzz_case(seed)
    rp, ci, vv = _banded(n, offsets, vals)
    P = ppa.CsrMatrix.from_arrays(n, rp, ci, vv)
    Q = O.Csr.from_arrays(n, rp, ci, vv)
    lay = ppa.make_csr_operator(P).layout()
    assert lay["layout"] == "dia_coded" and lay["two_factor_pass"], (n, offsets, lay)
    _check(cuda, P, Q, ROOTS[kind], complement, seed=seed)


# ---- box-grid form (kernels/spmv_grid2.cu) --------------------------------
def _box(nx, ny, nz, vals):
    """7-point (ny > 1) or 5-point (ny == 1) stencil on an nx x ny x nz box,
    cut at the faces, one value per diagonal (columns in increasing order)."""
    if ny > 1:
        offs = [(-1, 0, 0, 2), (0, -1, 0, 1), (0, 0, -1, 0), (0, 0, 0, None), (0, 0, 1, 0),
                (0, 1, 0, 1), (1, 0, 0, 2)]
    else:
        offs = [(-1, 0, 0, 2), (0, 0, -1, 0), (0, 0, 0, None), (0, 0, 1, 0), (1, 0, 0, 2)]
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    z, y, x = z.ravel(), y.ravel(), x.ravel()
    n = nx * ny * nz
    cols, keeps = [], []
    for dz, dy, dx, _ in offs:
        zz, yy, xx = z + dz, y + dy, x + dx
        keeps.append((zz >= 0) & (zz < nz) & (yy >= 0) & (yy < ny) & (xx >= 0) & (xx < nx))
        cols.append((zz * ny + yy) * nx + xx)
    C = np.stack(cols, axis=1)
    K = np.stack(keeps, axis=1)
    V = np.broadcast_to(np.asarray(vals, dtype=np.float64), C.shape)
    rp = np.concatenate([[0], np.cumsum(K.sum(axis=1))]).astype(np.int32)
    return n, rp, C[K].astype(np.int32), V[K].copy()


BOXES = [
    (160, 160, 6),     # config-3 planes, fewer planes than chunks
    (30, 50, 20),      # lines shorter than a warp, odd tile splits
    (200, 7, 30),      # few lines per plane
    (8, 100, 50),      # one partial warp per line
    (96, 96, 96),
    (252, 40, 12),     # widest line the 3-D form takes
    (1000, 1, 40),     # 2-D: several x tiles
    (2048, 1, 64),
    (64, 1, 700),      # 2-D, narrow lines, many chunks
    (130, 1, 9),
]


@pytest.mark.parametrize("box", BOXES)
@pytest.mark.parametrize("kind", ["real_even", "real_odd", "mixed", "pairs_only"])
@pytest.mark.parametrize("complement", [False, True])
def test_grid2_boxes_bit_exact(cuda, box, kind, complement):
    nx, ny, nz = box
    nd = 7 if ny > 1 else 5
    vals = [float(v) for v in np.random.default_rng(nx * ny + nz).choice(
        [-1.0, 2.5, -0.75, 4.0, 0.5, -3.0, 6.0], size=nd)]
    n, rp, ci, vv = _box(nx, ny, nz, vals)
    P = ppa.CsrMatrix.from_arrays(n, rp, ci, vv)
    Q = O.Csr.from_arrays(n, rp, ci, vv)
    lay = ppa.make_csr_operator(P).layout()
    assert lay["grid"] == (nx, ny, nz) and lay["grid_pass"] and lay["two_factor_pass"], lay
    _check(cuda, P, Q, ROOTS[kind], complement, seed=nx + nz)


def test_grid2_configs_detected(cuda):
    # configs 2, 3 and 5 are box grids; the reference's jump-coefficient
    # convection-diffusion is not (two values on one diagonal)
    for k, g in ((2, (1000, 1, 1000)), (3, (160, 160, 160)), (5, (2048, 1, 2048))):
        lay = ppa.make_csr_operator(ppa.CsrMatrix.config(k)).layout()
        assert lay["grid"] == g and lay["grid_pass"], (k, lay)
        # the pass's row evaluations (ppa_csr_grid_work, the bench's FP64
        # roofline): level 2 once per row, level 1 on the tiles plus halo
        l1, l2 = lay["grid_rows_per_pass"]
        n = g[0] * g[1] * g[2]
        assert l2 == n and n <= l1 < 1.6 * n, (k, l1, l2)
    assert ppa.make_csr_operator(ppa.CsrMatrix.convection_diffusion(64)).layout()["grid"] is None


def test_grid2_matches_presence_form(cuda, monkeypatch):
    # the box-grid form and the presence-byte form of the pass agree bit for bit
    P = ppa.CsrMatrix.laplacian_3d(48)
    roots = ROOTS["mixed"]
    x = dev(cuda, O.normal_vector(P.n, 5, 5))
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PPA_DISABLE_GRID2", flag)
        A = ppa.make_csr_operator(P)
        assert A.layout()["grid_pass"] == (flag == "0") and A.layout()["two_factor_pass"]
        y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
        ppa.apply_poly(roots, A, x, y)
        outs.append(host(y))
    assert np.array_equal(outs[0], outs[1])


def _grid_fuzz_case(seed):
    # the diagonal layout keeps its regular-row (and so presence / box-grid)
    # form only when at least half the rows are interior rows: draw shapes
    # until that holds
    rng = np.random.default_rng(5000 + seed)
    while True:
        if rng.integers(0, 2):
            nx = int(rng.choice([4, 10, 32, 46, 64, 96, 130, 160, 250]))
            ny = int(rng.integers(2, 60))
            nz = int(rng.integers(3, 40))
            interior = max(nx - 2, 0) * max(ny - 2, 0) * max(nz - 2, 0) / (nx * ny * nz)
        else:
            nx = int(rng.choice([8, 66, 300, 514, 1000, 1500, 2048]))
            ny = 1
            nz = int(rng.integers(3, 200))
            interior = max(nx - 2, 0) * max(nz - 2, 0) / (nx * nz)
        if interior >= 0.55:
            break
    nd = 7 if ny > 1 else 5
    vals = [float(v) for v in rng.choice([-1.0, 2.5, -0.75, 4.0, 0.5, -3.0, 6.0], size=nd)]
    kind = str(rng.choice(["real_even", "real_odd", "mixed", "pairs_only", "single_real"]))
    return (nx, ny, nz), vals, kind, bool(rng.integers(0, 2))


@pytest.mark.parametrize("seed", range(24))
def test_grid2_fuzz_bit_exact(cuda, seed):
    # seeded box shapes (3-D lines of 4-250 columns, 2-D lines up to 2048,
    # few and many planes), values per diagonal and root mixes: the
    # box-grid pass equals the oracle bit for bit
    box, vals, kind, complement = _grid_fuzz_case(seed)
    n, rp, ci, vv = _box(*box, vals)
    P = ppa.CsrMatrix.from_arrays(n, rp, ci, vv)
    Q = O.Csr.from_arrays(n, rp, ci, vv)
    lay = ppa.make_csr_operator(P).layout()
    assert lay["grid"] == box and lay["grid_pass"], (box, lay)
    _check(cuda, P, Q, ROOTS[kind], complement, seed=seed)
