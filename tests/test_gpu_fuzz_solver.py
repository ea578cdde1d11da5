"""Seeded end-to-end solver fuzz on small symmetric problems with known
spectra: random m, k, nev, polynomial degree, stability copies, restart
variant, orthogonalisation.  Every converged eigenvalue must match the dense
spectrum (numpy) to 1e-8 and every true residual must be below rtol."""
import numpy as np
import pytest

import paper_1806_08020_b200 as ppa

pytestmark = pytest.mark.gpu


def _problem(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(300, 1500))
    bw = int(rng.integers(1, 6))
    rows, cols, vals = [], [], []
    B = {}
    for i in range(n):
        B[(i, i)] = float(rng.uniform(1.0, 50.0)) + 2.0 * bw
        for o in range(1, bw + 1):
            if i + o < n and rng.random() < 0.7:
                v = float(rng.standard_normal())
                B[(i, i + o)] = v
                B[(i + o, i)] = v
    for (i, j), v in sorted(B.items()):
        rows.append(i); cols.append(j); vals.append(v)
    D = np.zeros((n, n))
    D[rows, cols] = vals
    lam = np.sort(np.linalg.eigvalsh(D))
    m = int(rng.integers(20, 50))
    k = int(rng.integers(max(3, m // 4), m // 2))
    nev = int(rng.integers(2, min(k, 10) + 1))
    cfg = ppa.SolveConfig(m=m, k=k, nev=nev, degree=int(rng.choice([0, 5, 12, 25])),
                          seed=int(seed) + 1, max_cycles=400,
                          stability=str(rng.choice(["off", "pof_auto"])),
                          variant=str(rng.choice(["ritz", "harmonic"])),
                          orthogonalization=str(rng.choice(["cgs2", "dcgs2"])))
    return n, rows, cols, vals, lam, cfg


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_solver(cuda, seed):
    n, rows, cols, vals, lam, cfg = _problem(seed)
    A = ppa.make_csr_operator(ppa.CsrMatrix.from_triplets(n, rows, cols, vals))
    r = ppa.solve(A, cfg)
    assert r["converged"], (cfg, r["cycles"], r["cycle_max_residual"][-3:])
    assert np.all(r["residuals"] <= r["rtol"])
    # smallest-magnitude targets (no polynomial) or |1 - nu| ordering (with one):
    # every returned value is an eigenvalue of A
    for z in r["eigenvalues"]:
        assert abs(z.imag) < 1e-8 * abs(z)
        assert np.min(np.abs(lam - z.real)) <= 1e-8 * abs(z.real), (z, cfg)
    if cfg.degree == 0:
        got = np.sort(r["eigenvalues"].real)
        assert np.allclose(got, lam[:cfg.nev], rtol=1e-8), (got, lam[:cfg.nev], cfg)
