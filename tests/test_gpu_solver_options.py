"""Solver options beyond the default cycle loop, device vs oracle.

SolveConfig (inc/solver.hpp:45-52) carries check_mid_cycle/mid_cycle_stride
and stagnation_stop/_window/_rtol; EigResult (inc/solver.hpp:71-89) returns
eigenvectors.  SPEC.md:421 (mid-cycle checks behind a flag) and SPEC.md:621
(stagnation = <1% improvement of the max residual over 5 cycles) give the
semantics; the oracle restates both (oracle/ppa_oracle.cpp solve()).
"""
import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

pytestmark = pytest.mark.gpu

DIAG = np.arange(1.0, 2001.0)


def _pair(**kw):
    cfg = ppa.SolveConfig(m=30, k=15, nev=10, degree=0, seed=1, max_cycles=200, **kw)
    r = ppa.solve(ppa.make_diagonal(DIAG), cfg)
    okw = {}
    if kw.get("check_mid_cycle"):
        okw["mid_cycle_stride"] = kw.get("mid_cycle_stride", 5)
    if kw.get("stagnation_stop"):
        okw["stagnation_window"] = kw.get("stagnation_window", 5)
        okw["stagnation_rtol"] = kw.get("stagnation_rtol", 0.01)
    o = O.solve(O.diagonal_operator(DIAG), 30, 15, 10, degree=0, seed=1, max_cycles=200, **okw)
    return r, o


def test_mid_cycle_matches_oracle(cuda):
    r, o = _pair(check_mid_cycle=True, mid_cycle_stride=5)
    base, _ = _pair()
    assert r["converged"] and o["converged"]
    assert r["cycles"] == o["cycles"]
    # the early exit saves Arnoldi steps of the last cycle; checks cost mvps
    assert r["cycles"] <= base["cycles"]
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]
    assert np.all(r["residuals"] <= r["rtol"])
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1.0, 11.0), rtol=1e-8)


def test_mid_cycle_stops_inside_cycle(cuda):
    # With a degree-60 polynomial the second cycle converges well before m:
    # the mid-cycle check stops the extension early, the plain run does not.
    A = ppa.make_diagonal(np.arange(1.0, 1001.0))
    cfg = dict(m=50, k=20, nev=15, degree=60, seed=1)
    full = ppa.solve(A, ppa.SolveConfig(**cfg))
    mid = ppa.solve(A, ppa.SolveConfig(check_mid_cycle=True, mid_cycle_stride=5, **cfg))
    o = O.solve(O.diagonal_operator(np.arange(1.0, 1001.0)), 50, 20, 15, degree=60, seed=1,
                mid_cycle_stride=5)
    assert mid["converged"] and full["converged"] and o["converged"]
    assert mid["cycles"] == o["cycles"] == full["cycles"] == 2
    assert mid["cost"]["mvps"] < 0.8 * full["cost"]["mvps"]
    # A degree-60 polynomial on diag(1..1000) converges to a set with gaps
    # (1, 5..8, 14..18, 29..33) -- on the device and in the oracle alike, with
    # or without the early exit: the case check_ideal_order and the damping
    # heuristic exist for (section 6.3).
    assert np.allclose(np.sort(mid["eigenvalues"].real), np.sort(o["eigenvalues"].real),
                       rtol=1e-8)
    assert not ppa.check_ideal_order(mid["eigenvalues"], 15)
    assert abs(mid["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]


def test_stagnation_stop_matches_oracle(cuda):
    r, o = _pair(stagnation_stop=True, stagnation_window=3)
    assert r["cycles"] == o["cycles"] < 200
    h = r["cycle_max_residual"]
    best = np.minimum.accumulate(h)
    assert best[-1] > 0.99 * best[-1 - 3]
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]


def test_eigenvectors_output(cuda):
    P = ppa.CsrMatrix.convection_diffusion_const(40, 0.5)
    A = ppa.make_csr_operator(P)
    cfg = ppa.SolveConfig(m=40, k=20, nev=8, degree=8, seed=2, max_cycles=60,
                          want_eigenvectors=True)
    r = ppa.solve(A, cfg)
    assert r["converged"]
    Y = r["eigenvectors"]
    mu = r["eigenvalues"]
    assert Y.shape == (P.n, mu.size)
    rp, ci, va = P.arrays()
    import scipy.sparse as sp
    M = sp.csr_matrix((va, ci, rp), shape=(P.n, P.n))
    for j in range(mu.size):
        y = Y[:, j]
        assert abs(np.linalg.norm(y) - 1.0) < 1e-12
        res = np.linalg.norm(M @ y - mu[j] * y)
        # the reported residual is ||A y - mu y|| for the same unit y
        assert res <= max(2.0 * r["residuals"][j], 1e-12) + 1e-13
        assert res <= r["rtol"] * 1.0001
    # eigenvectors are off unless requested
    r2 = ppa.solve(A, ppa.SolveConfig(m=40, k=20, nev=8, degree=8, seed=2, max_cycles=60))
    assert "eigenvectors" not in r2


def test_harmonic_variant_matches_oracle(cuda):
    # SolveConfig::variant = harmonic: restart selection from the harmonic
    # Ritz pairs (src/arnoldi.cpp:208-246) on the device path and the oracle
    d = np.arange(1.0, 1001.0)
    cfg = ppa.SolveConfig(m=40, k=20, nev=10, degree=0, seed=3, max_cycles=300,
                          variant="harmonic")
    r = ppa.solve(ppa.make_diagonal(d), cfg)
    o = O.solve(O.diagonal_operator(d), 40, 20, 10, degree=0, seed=3, max_cycles=300,
                variant="harmonic")
    assert r["converged"] and o["converged"]
    assert np.allclose(np.sort(r["eigenvalues"].real), np.arange(1.0, 11.0), rtol=1e-8)
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]
    # and with a polynomial on a nonsymmetric matrix
    P = ppa.CsrMatrix.convection_diffusion(40)
    cfg = ppa.SolveConfig(m=40, k=20, nev=8, degree=12, seed=5, max_cycles=60,
                          variant="harmonic")
    r = ppa.solve(ppa.make_csr_operator(P), cfg)
    o = O.solve(O.csr_operator(O.Csr.convection_diffusion(40)), 40, 20, 8, degree=12, seed=5,
                max_cycles=60, variant="harmonic")
    assert r["converged"] and o["converged"]
    got, ref = np.sort_complex(r["eigenvalues"]), np.sort_complex(o["eigenvalues"])
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-8
    assert abs(r["cost"]["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]


def test_concurrent_solves_two_threads(cuda):
    # one context (stream, workspaces, pinned staging) per host thread: two
    # threads solving at once on their own streams get exactly the results of
    # the sequential solves (SPEC.md: concurrent solves need independent
    # CostRecords; operators are reentrant)
    import threading

    P = ppa.CsrMatrix.convection_diffusion(36)
    A = ppa.make_csr_operator(P)
    cfgs = [ppa.SolveConfig(m=30, k=15, nev=6, degree=8, seed=s, max_cycles=80) for s in (1, 2)]
    seq = [ppa.solve(A, c) for c in cfgs]
    out = [None, None]

    def run(i):
        s = cuda.cuda.Stream()
        ppa.set_stream(s)
        out[i] = ppa.solve(A, cfgs[i])
        s.synchronize()

    th = [threading.Thread(target=run, args=(i,)) for i in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(out, seq):
        assert np.array_equal(a["eigenvalues"], b["eigenvalues"])
        assert a["cost"]["mvps"] == b["cost"]["mvps"] and a["cycles"] == b["cycles"]


@pytest.mark.parametrize("degree", [0, 3])
def test_breakdown_inside_solve_matches_oracle(cuda, degree):
    # five distinct eigenvalues: every Krylov space breaks down at dimension 5,
    # inside the first cycle (the pipelined CGS2 extend has already enqueued
    # the next step); the solve checks that cycle's pairs and stops
    d = np.repeat([1.0, 2.0, 4.0, 7.0, 11.0], 100)
    cfg = ppa.SolveConfig(m=30, k=15, nev=3, degree=degree, seed=4, max_cycles=10)
    r = ppa.solve(ppa.make_diagonal(d), cfg)
    o = O.solve(O.diagonal_operator(d), 30, 15, 3, degree=degree, seed=4, max_cycles=10)
    assert r["converged"] == o["converged"] and r["cycles"] == o["cycles"] == 1
    assert (r["cost"]["mvps"], r["cost"]["dots"], r["cost"]["vops"]) == \
        (o["cost"]["mvps"], o["cost"]["dots"], o["cost"]["vops"])
    assert np.allclose(np.sort(r["eigenvalues"].real), np.sort(o["eigenvalues"].real),
                       rtol=1e-10)


_GRAPH_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
import paper_1806_08020_b200 as ppa
A = ppa.make_csr_operator(ppa.CsrMatrix.convection_diffusion_const(70, 0.5))
out = {}
r = ppa.solve(A, ppa.SolveConfig(m=30, k=15, nev=6, degree=12, seed=4, max_cycles=40))
out["single"] = [r["eigenvalues"].real.tolist(), r["eigenvalues"].imag.tolist(),
                 r["residuals"].tolist(), r["cost"], r["cycles"]]
r = ppa.solve_double(A, ppa.SolveConfig(m=30, k=15, nev=6, double_d1=4, double_d2=5, seed=4,
                                        max_cycles=40))
out["double"] = [r["eigenvalues"].real.tolist(), r["eigenvalues"].imag.tolist(),
                 r["residuals"].tolist(), r["cost"], r["cycles"]]
print(json.dumps(out))
"""


def test_chain_graphs_bit_identical(cuda):
    # PPA_CHAIN_GRAPHS=1 (recorded chains, one graph updated in place per
    # operator and stream): same eigenpairs, residuals and counters, bit for
    # bit, as direct launches - single and nested polynomial operators
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        env = dict(os.environ, PPA_CHAIN_GRAPHS=flag)
        p = subprocess.run([sys.executable, "-c", _GRAPH_CHILD % root], env=env,
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        res[flag] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["0"] == res["1"]
