"""Seeded fuzz over the SpMV layouts: random stencil-like, banded and
irregular matrices (sizes 1..6000, empty rows, few or many distinct values,
explicit zeros), every layout cap, real/pair/complement epilogues - each
result bit-identical to the oracle's CSR loop (src/operators.cpp:39-48,
src/gmres_poly.cpp:117-147, 302-311)."""
import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = seed % 4
    n = int(rng.choice([1, 7, 33, 500, 2049, 6000]))
    rows, cols, vals = [], [], []
    if kind == 0:  # stencil: few diagonals, few values, some rows perturbed
        offs = sorted(set(rng.integers(-min(n, 300), min(n, 300) + 1, int(rng.integers(1, 10))).tolist()))
        table = rng.standard_normal(int(rng.integers(1, 6)))
        for i in range(n):
            for o in offs:
                j = i + o
                if 0 <= j < n and rng.random() > 0.02:
                    v = table[abs(o) % len(table)]
                    if rng.random() < 0.01:
                        v = float(rng.standard_normal())
                    rows.append(i); cols.append(j); vals.append(v)
    elif kind == 1:  # banded, many values, ragged
        bw = int(rng.integers(1, 2000))
        for i in range(n):
            if rng.random() < 0.1:
                continue
            for j in sorted(set(rng.integers(max(0, i - bw), min(n, i + bw + 1), int(rng.integers(1, 12))).tolist())):
                rows.append(i); cols.append(j); vals.append(float(rng.standard_normal()))
    elif kind == 2:  # irregular row lengths, random columns
        for i in range(n):
            L = int(rng.poisson(6))
            for j in sorted(set(rng.integers(0, n, L).tolist())):
                rows.append(i); cols.append(j); vals.append(float(rng.choice([0.0, -0.0, 1.5, -2.0, rng.standard_normal()])))
    else:  # diagonal-dominant tridiagonal with explicit zeros and -0.0
        for i in range(n):
            for o, v in ((-1, -1.0), (0, 2.0), (1, -0.0 if i % 5 == 0 else -1.0)):
                j = i + o
                if 0 <= j < n:
                    rows.append(i); cols.append(j); vals.append(v)
    return n, rows, cols, vals


def _roots(rng):
    r = list(rng.uniform(0.5, 50.0, int(rng.integers(1, 5))))
    z = rng.uniform(1, 40) + 1j * rng.uniform(0.5, 10)
    return O.leja_order(r + [z, np.conj(z)])


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_layouts(cuda, seed):
    n, rows, cols, vals = _case(seed)
    P = ppa.CsrMatrix.from_triplets(n, rows, cols, vals)
    Q = O.Csr.from_triplets(n, rows, cols, vals)
    assert P.fingerprint() == Q.info()[2]
    rng = np.random.default_rng(seed)
    x = O.normal_vector(n, seed + 1, 2)
    roots = _roots(rng)
    ref_y = O.csr_operator(Q).apply(x)
    ref_p = O.apply_poly(roots, O.csr_operator(Q), x)
    tau_o = O.poly_operator(O.csr_operator(Q), roots, True)
    ref_t = tau_o.apply(x, np.zeros(3))
    xd = cuda.tensor(x, device="cuda")
    for cap in ("auto", "csr", "sell32", "sell32_packed", "dia_coded"):
        A = ppa.make_csr_operator(P, cap)
        y = cuda.empty(n, dtype=cuda.float64, device="cuda")
        A.apply(xd, y)
        assert np.array_equal(y.cpu().numpy(), ref_y), (cap, A.layout())
        ppa.apply_poly(roots, A, xd, y)
        assert np.array_equal(y.cpu().numpy(), ref_p), (cap, A.layout())
        tau = ppa.make_poly_complement_operator(A, roots)
        tau.apply(xd, y)
        assert np.array_equal(y.cpu().numpy(), ref_t), (cap, A.layout())
