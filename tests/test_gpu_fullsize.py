"""Full-size parity at BASELINE config 3 (4,096,000 rows, 28.5M nnz) plus
the solver-level checks of every config.  The oracle runs here only where it
finishes in seconds (one pi(A)v with all host threads); slower oracle results
come from the committed fixtures in tests/golden/ (make_golden.py)."""
import json
import os

import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"fixture {name} not generated")
    return json.load(open(p))


def _c(d):
    return np.array(d["re"]) + 1j * np.array(d["im"])


def _canon_pairs(roots):
    """Leja order with each adjacent conjugate pair written +imag first: the two
    members of a pair have mathematically equal Leja scores, so roundoff picks
    which comes first, and the pair is applied as one real quadratic factor."""
    r = list(np.asarray(roots, dtype=np.complex128))
    i = 0
    while i < len(r) - 1:
        if abs(r[i].imag) > 1e-13 * abs(r[i]) and abs(r[i + 1] - np.conj(r[i])) <= 1e-6 * abs(r[i]):
            if r[i].imag < 0:
                r[i], r[i + 1] = r[i + 1], r[i]
            i += 2
        else:
            i += 1
    return np.array(r)


@pytest.fixture(scope="module")
def c3(cuda):
    P = ppa.CsrMatrix.config(3)
    return P, ppa.make_csr_operator(P)


def test_c3_model_bytes_and_default_layout(c3):
    # the north-star byte model of one SpMV, and the layout make_csr_operator
    # picks for config 3 (diagonal-coded, box-grid two-factor pass)
    P, A = c3
    assert A.model_bytes() == 12 * 28518400 + 4 * (4096000 + 1) + 16 * 4096000
    lay = A.layout()
    assert lay["layout"] == "dia_coded" and lay["grid"] == (160, 160, 160) and lay["grid_pass"]
    assert ppa.make_csr_operator(P, "sell32").layout()["layout"] == "sell32"


def test_c3_pi_av_bit_exact_full_size(cuda, c3):
    P, A = c3
    roots = _c(_golden("c3_poly.json")["roots"])
    v = ppa.normal_vector(P.n, 2, ppa.STREAM_ARNOLDI)
    out = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    rec = ppa.apply_poly(roots, A, cuda.tensor(v, device="cuda"), out)
    assert rec.mvps == len(roots)
    O.set_threads(os.cpu_count() or 1)
    ref = O.apply_poly(roots, O.csr_operator(O.Csr.config(3)), v)
    got = out.cpu().numpy()
    assert np.array_equal(got, ref), np.linalg.norm(got - ref) / np.linalg.norm(ref)


def test_c3_polynomial_matches_oracle(cuda, c3):
    P, A = c3
    g = _golden("c3_poly.json")
    b = cuda.tensor(ppa.normal_vector(P.n, 2, ppa.STREAM_POLY), device="cuda")
    rec = ppa.CostRecord()
    roots, trunc = ppa.build_gmres_poly(A, b, 50, rec)
    base = _c(g["base_roots"])
    assert not trunc and len(roots) == len(base) == 50
    # Same Leja permutation: every GPU root's nearest oracle root sits at the
    # same position.  Values agree to the conditioning of degree-50 harmonic
    # Ritz values under CGS2-vs-MGS2 roundoff (measured 9e-7 worst, 1e-9 typical).
    nearest = [int(np.argmin(np.abs(base - z))) for z in roots]
    assert nearest == list(range(50))
    assert np.max(np.abs(roots - base) / np.abs(base)) < 1e-5
    assert [rec.mvps, rec.dots, rec.vops] == [int(x) for x in g["cost"]]
    aug = ppa.add_stability_roots(roots, 50)
    assert len(aug) == len(_c(g["roots"]))
    # the two polynomials act alike on the start vector (the GMRES residual)
    out_g = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    out_o = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, b, out_g)
    ppa.apply_poly(base, A, b, out_o)
    ng, no = out_g.norm().item(), out_o.norm().item()
    assert abs(ng - no) / no < 1e-6
    assert (out_g - out_o).norm().item() / no < 1e-4


def _analytic_c3(k=40):
    N = 160
    h = 1.0 / (N + 1)
    s = 4 / h ** 2 * np.sin(np.arange(1, 8) * np.pi * h / 2) ** 2
    lam = np.sort((s[:, None, None] + s[None, :, None] + s[None, None, :]).ravel())
    return lam[:k]


def test_c3_solve_analytic_and_oracle(cuda, c3):
    P, A = c3
    r = ppa.solve(A, ppa.config_solve_config(3))
    assert r["converged"]
    assert np.all(r["residuals"] <= r["rtol"])
    lam = _analytic_c3()
    got = np.sort(r["eigenvalues"].real)
    # multiset check: eigenvalue clusters of multiplicity 3 and 6
    for z in got:
        assert np.min(np.abs(lam - z) / lam) < 1e-8
    assert abs(got[0] - 29.607874) < 1e-5
    g = _golden("c3_solve.json")
    assert g["converged"]
    ref = np.sort(_c(g["eigenvalues"]).real)
    for z in got:
        assert np.min(np.abs(ref - z) / ref) < 1e-8
    assert abs(r["cost"]["mvps"] - g["cost"]["mvps"]) <= 0.05 * g["cost"]["mvps"]


@pytest.mark.parametrize("k", [1, 2, 4, 5])
def test_config_solve_vs_fixture(cuda, k):
    g = _golden(f"c{k}_solve.json")
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
    cfg = ppa.config_solve_config(k)
    r = ppa.solve_double(A, cfg) if k == 5 else ppa.solve(A, cfg)
    assert r["converged"] == g["converged"]
    assert abs(r["rtol"] - g["rtol"]) <= 1e-10 * g["rtol"]  # same norm estimate
    # the polynomial is built before any Arnoldi cycle: it must agree for
    # every config (CGS2 vs MGS2 roundoff only)
    inner = _canon_pairs(_c(g["inner_poly"] if k == 5 else g["poly"]))
    got_inner = _canon_pairs(r["inner_poly"] if k == 5 else r["poly"])
    assert got_inner.size == inner.size
    assert np.max(np.abs(got_inner - inner) / np.abs(inner)) < 1e-6
    if not r["converged"]:
        # config 4 does not converge in 100 cycles on either side (DESIGN.md
        # "Config 4"); both run the full budget and end at a comparable
        # residual level
        assert r["cycles"] == g["cycles"] == cfg.max_cycles
        hist, ghist = r["cycle_max_residual"], np.array(g["cycle_max_residual"])
        # the trajectories agree closely early on (1e-12 observed over the
        # first 6 cycles), and stay at the same residual level throughout
        assert np.allclose(hist[:10], ghist[:10], rtol=1e-8, atol=0)
        assert 0.1 < np.min(hist) / np.min(ghist) < 10.0
        return
    assert np.all(r["residuals"] <= r["rtol"])
    if k != 5:
        # config 5's matvec count moves with the summation order even between
        # oracle variants (2 or 3 cycles); checked in test_nonnormal_vs_oracle_floor
        assert abs(r["cost"]["mvps"] - g["cost"]["mvps"]) <= 0.05 * g["cost"]["mvps"]
    if k in (1, 2):
        # simple spectra: the GPU and oracle trajectories agree to roundoff
        # through the early cycles (~1e-13 observed in cycles 1-2)
        hist, ghist = r["cycle_max_residual"], np.array(g["cycle_max_residual"])
        assert np.allclose(hist[:3], ghist[:3], rtol=1e-8, atol=0)
    if k in (2, 5):
        # Constant-Peclet convection-diffusion: eigenvalues are compared against
        # the oracle's own roundoff floor in test_nonnormal_vs_oracle_floor
        return
    got = np.sort_complex(r["eigenvalues"])
    ref = np.sort_complex(_c(g["eigenvalues"]))
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-8


@pytest.mark.parametrize("k", [2, 5])
def test_two_factor_pass_full_size_bit_exact(cuda, k):
    # BASELINE configs 2 and 5 at full size run the two-factor pass with two
    # CTAs per SM (spmv_dia2.cu): a mixed real/pair chain, its complement and
    # the nested phi(tau(A)) of solve_double, bit-identical to the oracle
    P = ppa.CsrMatrix.config(k)
    A = ppa.make_csr_operator(P)
    assert A.layout()["two_factor_pass"]
    Q = O.csr_operator(O.Csr.config(k))
    O.set_threads(os.cpu_count() or 1)
    lam_max = 8.0 * (P.n ** 0.5 + 1) ** 2
    r1 = O.leja_order([0.9 * lam_max, 0.5 * lam_max + 0.05j * lam_max,
                       0.5 * lam_max - 0.05j * lam_max, 0.2 * lam_max, 0.05 * lam_max])
    r2 = O.leja_order([0.9, 0.4 + 0.1j, 0.4 - 0.1j])
    v = ppa.normal_vector(P.n, 3, ppa.STREAM_ARNOLDI)
    x = cuda.tensor(v, device="cuda")
    y = cuda.empty(P.n, dtype=cuda.float64, device="cuda")
    for op, ref in (
        (ppa.make_poly_operator(A, r1), O.poly_operator(Q, r1)),
        (ppa.make_poly_complement_operator(A, r1), O.poly_operator(Q, r1, True)),
        (ppa.make_poly_operator(ppa.make_poly_complement_operator(A, r1), r2),
         O.poly_operator(O.poly_operator(Q, r1, True), r2)),
    ):
        op.apply(x, y)
        want = ref.apply(v)
        got = y.cpu().numpy()
        assert np.array_equal(got, want), np.linalg.norm(got - want) / np.linalg.norm(want)


# ---- non-normal configs 2 and 5: parity against the oracle's roundoff floor
def _convdiff_spectrum(N, pe=0.5, k=400):
    """Closed form of the constant-Peclet operator."""
    h = 1.0 / (N + 1)
    j = np.arange(1, 60)
    ax = (2 / h ** 2) * (1 - np.sqrt(1 - pe ** 2) * np.cos(j * np.pi * h))
    ay = (2 / h ** 2) * (1 - np.cos(j * np.pi * h))
    return np.sort((ax[:, None] + ay[None, :]).ravel())[:k]


def _oracle_variants(k):
    """Oracle solves of config k under three summation orders: the reference
    (MGS2, sequential dots; c{k}_solve.json) and the two roundoff-floor probes
    of roundoff_floor.json (classical CGS2 / MGS2 with blocked dots)."""
    out = [_golden(f"c{k}_solve.json")]
    fl = _golden("roundoff_floor.json")[f"config{k}"]
    out += [fl["1"], fl["2"]]
    return out


def _nearest_rel(a, b):
    b = np.asarray(b)
    return np.array([np.min(np.abs(z - b)) / abs(z) for z in a])


@pytest.mark.parametrize("k", [2, 5])
def test_nonnormal_vs_oracle_floor(cuda, k):
    """The certified Ritz values of configs 2 and 5 sit in the pseudospectrum
    (cond of the symmetrising scaling ~3^((N-1)/2)), where the
    summation order alone moves them.  The bar: the GPU's values lie within
    the spread the oracle itself shows under equally valid summation orders
    (its roundoff floor, measured and committed), every returned pair is
    residual-certified by an independent host check, and the cycle count and
    matvecs fall inside the oracle variants' range."""
    vs = _oracle_variants(k)
    evs = [_c(v["eigenvalues"]) for v in vs]
    # the oracle's floor: worst nearest-value distance between any two variants
    floor = max(np.max(_nearest_rel(evs[i], evs[j])) for i in range(3) for j in range(3)
                if i != j)
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
    cfg = ppa.config_solve_config(k, want_eigenvectors=True)
    r = ppa.solve_double(A, cfg) if k == 5 else ppa.solve(A, cfg)
    assert r["converged"] and all(v["converged"] for v in vs)
    cyc = [v["cycles"] for v in vs]
    mv = [v["cost"]["mvps"] for v in vs]
    assert min(cyc) <= r["cycles"] <= max(cyc), (r["cycles"], cyc)
    assert 0.95 * min(mv) <= r["cost"]["mvps"] <= 1.05 * max(mv), (r["cost"]["mvps"], mv)
    got = r["eigenvalues"]
    union = np.concatenate(evs)
    d = _nearest_rel(got, union)
    print(f"config {k}: oracle floor {floor:.3e}, GPU-to-oracle max {d.max():.3e}")
    assert d.max() <= floor, (d.max(), floor)
    if k == 2:
        # the floor is ~1e-5 here; the GPU sits inside it against every variant
        for e in evs:
            assert np.max(_nearest_rel(got, e)) <= floor
    # independent residual certificate: ||A y - mu y|| on the host (oracle SpMV)
    O.set_threads(os.cpu_count() or 1)
    Q = O.csr_operator(O.Csr.config(k))
    Y = r["eigenvectors"]
    for j, mu in enumerate(got):
        y = Y[:, j]
        ay = Q.apply(y.real) + 1j * Q.apply(y.imag)
        res = np.linalg.norm(ay - mu * y) / np.linalg.norm(y)
        assert res <= r["rtol"] * (1 + 1e-6), (j, mu, res, r["rtol"])
    # these are pseudo-eigenvalues: every certified value (GPU and oracle alike)
    # lies far from the true spectrum, whose smallest member is ~10x larger
    N = 1000 if k == 2 else 2048
    lam = _convdiff_spectrum(N)
    dg = _nearest_rel(got, lam)
    do = _nearest_rel(evs[0], lam)
    print(f"config {k}: distance to the closed-form spectrum GPU min {dg.min():.3f} "
          f"oracle min {do.min():.3f} (lambda_min {lam[0]:.3f})")
    assert dg.min() > 1.0 and do.min() > 1.0
