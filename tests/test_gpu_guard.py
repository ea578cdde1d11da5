"""Guard-band checks of the device kernels (compute-sanitizer is not available on
the GPU pool, so this is the suite's own memcheck).

Every vector a kernel reads sits inside a larger buffer whose bands are NaN:
a read past either end that reaches the arithmetic poisons the result, which
is compared bit for bit with the same call on plain buffers.  Every vector a
kernel writes sits inside a buffer of sentinel words that must survive.  Sizes
are ragged on purpose (not multiples of the 32-row slices, the 128-row TMA
tiles or the box-grid tile shapes)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BAND = 4096  # doubles each side (32 KB: wider than any tile's overshoot)
SENTINEL = 0x7FF8DEADBEEF1234  # a quiet NaN with a payload


class Guarded:
    """n doubles inside a sentinel-filled buffer."""

    def __init__(self, torch, n, fill=None):
        self.torch = torch
        self.n = n
        self.buf = torch.full((n + 2 * BAND,), SENTINEL, dtype=torch.int64, device="cuda")
        self.v = self.buf[BAND:BAND + n].view(torch.float64)
        if fill is not None:
            self.v.copy_(fill)

    def intact(self):
        lo = self.buf[:BAND]
        hi = self.buf[BAND + self.n:]
        return bool((lo == SENTINEL).all().item()) and bool((hi == SENTINEL).all().item())


def _mats(ppa):
    return [
        ("bidiag-2999", ppa.CsrMatrix.bidiagonal(2999)),
        ("convdiff2d-70", ppa.CsrMatrix.convection_diffusion_const(70)),
        ("convdiff2d-257", ppa.CsrMatrix.convection_diffusion_const(258)),
        ("laplace3d-22", ppa.CsrMatrix.laplacian_3d(22)),
        ("laplace3d-34", ppa.CsrMatrix.laplacian_3d(34)),
        ("poisson-6001", ppa.CsrMatrix.random_poisson(6001, 16.0, 4)),
    ]


def _vec(torch, ppa, n, seed):
    return torch.tensor(ppa.normal_vector(n, seed, ppa.STREAM_ARNOLDI), device="cuda")


@pytest.mark.parametrize("layout", ["auto", "csr", "sell32", "sell32_packed", "dia_coded"])
def test_spmv_and_factor_chain_stay_in_bounds(cuda, layout):
    import paper_1806_08020_b200 as ppa

    torch = cuda
    roots = ppa.leja_order(np.array([9000.0, 4000 + 900j, 4000 - 900j, 1500.0, 300.0, 40.0,
                                     7.0]))
    for name, m in _mats(ppa):
        n = m.n
        A = ppa.make_csr_operator(m, layout)
        x = _vec(torch, ppa, n, 1)
        y0 = torch.empty(n, dtype=torch.float64, device="cuda")
        p0 = torch.empty(n, dtype=torch.float64, device="cuda")
        ppa.spmv(A, x, y0)
        ppa.apply_poly(roots, A, x, p0)
        gx, gy, gp = Guarded(torch, n, x), Guarded(torch, n), Guarded(torch, n)
        ppa.spmv(A, gx.v, gy.v)
        ppa.apply_poly(roots, A, gx.v, gp.v)
        torch.cuda.synchronize()
        assert torch.equal(gy.v, y0), (name, layout, "spmv read past x")
        assert torch.equal(gp.v, p0), (name, layout, "factor chain read past x")
        assert gx.intact() and gy.intact() and gp.intact(), (name, layout, "write out of bounds")


@pytest.mark.parametrize("complement", [False, True])
def test_poly_operators_stay_in_bounds(cuda, complement):
    # two-factor passes (box-grid and presence forms) with the complement
    # epilogue, odd and even factor counts
    import paper_1806_08020_b200 as ppa

    torch = cuda
    mk = ppa.make_poly_complement_operator if complement else ppa.make_poly_operator
    for nroots in (4, 7):
        rr = np.array([9000.0, 4000 + 900j, 4000 - 900j, 1500.0, 300.0, 40.0, 7.0])[:nroots]
        roots = ppa.leja_order(rr)
        for name, m in _mats(ppa):
            n = m.n
            op = mk(ppa.make_csr_operator(m), roots)
            x = _vec(torch, ppa, n, 2)
            y0 = torch.empty(n, dtype=torch.float64, device="cuda")
            op.apply(x, y0)
            gx, gy = Guarded(torch, n, x), Guarded(torch, n)
            op.apply(gx.v, gy.v)
            torch.cuda.synchronize()
            assert torch.equal(gy.v, y0), (name, nroots, complement)
            assert gx.intact() and gy.intact(), (name, nroots, complement)


def test_spmm_stays_in_bounds(cuda):
    import paper_1806_08020_b200 as ppa

    torch = cuda
    for name, m in _mats(ppa):
        n, p = m.n, 5
        ld = (n + 31) // 32 * 32
        A = ppa.make_csr_operator(m)
        Y = Guarded(torch, p * ld)
        Y.v.zero_()
        for j in range(p):
            Y.v[j * ld:j * ld + n] = _vec(torch, ppa, n, 10 + j)
        AY = Guarded(torch, p * ld)
        AY.v.fill_(-7.0)
        ppa.spmm(A, Y.v, ld, p, AY.v, ld)
        y1 = torch.empty(n, dtype=torch.float64, device="cuda")
        for j in range(p):
            ppa.spmv(A, Y.v[j * ld:j * ld + n], y1)
            torch.cuda.synchronize()
            assert torch.equal(AY.v[j * ld:j * ld + n], y1), (name, j)
            # the padding rows between columns are not written
            assert bool((AY.v[j * ld + n:(j + 1) * ld] == -7.0).all().item()), (name, j)
        assert Y.intact() and AY.intact(), name


@pytest.mark.parametrize("n,c", [(3001, 1), (3001, 4), (4099, 9), (2177, 24), (5000, 51),
                                 (129, 100)])
def test_cgs2_step_stays_in_bounds(cuda, n, c):
    # the three TMA-pipelined sweeps over a basis with a ragged last tile:
    # V[:, c] is written, V[:, :c] and the rows past n are not
    import paper_1806_08020_b200 as ppa

    torch = cuda
    ld = (n + 31) // 32 * 32
    rng = np.random.default_rng(n + c)
    Q, _ = np.linalg.qr(rng.standard_normal((n, c)))
    Vh = np.zeros((c + 1, ld))
    Vh[:c, :n] = Q.T
    wh = rng.standard_normal(n)

    def run(V, w):
        Hc = torch.zeros(c + 2, dtype=torch.float64, device="cuda")
        flag = torch.zeros(2, dtype=torch.int32, device="cuda")
        ppa.cgs2_step(V, ld, n, c, w, Hc, flag)
        torch.cuda.synchronize()
        return Hc

    V0 = torch.tensor(Vh.ravel(), device="cuda")
    w0 = torch.tensor(wh, device="cuda")
    H0 = run(V0, w0)
    gV = Guarded(torch, (c + 1) * ld, torch.tensor(Vh.ravel(), device="cuda"))
    gw = Guarded(torch, n, torch.tensor(wh, device="cuda"))
    H1 = run(gV.v, gw.v)
    assert torch.equal(H0, H1)
    assert torch.equal(gV.v, V0)
    assert gV.intact() and gw.intact()
    got = gV.v.cpu().numpy().reshape(c + 1, ld)
    assert np.array_equal(got[:c], Vh[:c]), "basis columns changed"
    assert not got[c, n:].any(), "rows past n written"
    # the new column is orthonormal to the basis
    q = got[c, :n]
    assert abs(np.linalg.norm(q) - 1.0) < 1e-12 and np.max(np.abs(Q.T @ q)) < 1e-12


@pytest.mark.parametrize("d,p,inplace,n", [(40, 20, True, 4099), (40, 15, False, 3001),
                                           (41, 21, True, 129), (7, 3, False, 1000),
                                           (60, 45, True, 1500)])
def test_ts_combine_stays_in_bounds(cuda, d, p, inplace, n):
    import paper_1806_08020_b200 as ppa

    torch = cuda
    ld = (n + 31) // 32 * 32
    rng = np.random.default_rng(d * 7 + p + n)
    Vh = np.zeros((d + 1, ld))
    Vh[:, :n] = rng.standard_normal((d + 1, n))
    G = torch.tensor(rng.standard_normal((p, d)).ravel(), device="cuda")
    gV = Guarded(torch, (d + 1) * ld, torch.tensor(Vh.ravel(), device="cuda"))
    V0 = torch.tensor(Vh.ravel(), device="cuda")
    if inplace:
        ppa.ts_combine(V0, ld, n, d, G, p, V0, ld)
        ppa.ts_combine(gV.v, ld, n, d, G, p, gV.v, ld)
        torch.cuda.synchronize()
        assert torch.equal(gV.v, V0)
    else:
        O0 = torch.zeros(p * ld, dtype=torch.float64, device="cuda")
        gO = Guarded(torch, p * ld)
        gO.v.zero_()
        ppa.ts_combine(V0, ld, n, d, G, p, O0, ld)
        ppa.ts_combine(gV.v, ld, n, d, G, p, gO.v, ld)
        torch.cuda.synchronize()
        assert torch.equal(gO.v, O0)
        assert gO.intact()
    assert gV.intact()


def test_ritz_vector_outputs_stay_in_bounds(cuda):
    import paper_1806_08020_b200 as ppa

    torch = cuda
    m = ppa.CsrMatrix.convection_diffusion(45)
    n = m.n
    A = ppa.make_csr_operator(m)
    st = ppa.arnoldi_init(_vec(torch, ppa, n, 5), n, 14)
    st.extend(A, 14)
    yr, yi = Guarded(torch, n), Guarded(torch, n)
    for j in range(4):
        st.ritz_vector(j, yr.v, yi.v)
    torch.cuda.synchronize()
    assert yr.intact() and yi.intact()
    assert bool(torch.isfinite(yr.v).all().item())
