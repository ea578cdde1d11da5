"""CPU-side checks of the product library (no GPU needed): the C-ABI library
loads and exports every symbol include/ppa_b200.h declares; host-side logic
(generators, RNG streams, Leja order, pof, stability copies, validation and
error mapping) is bit-exact with the oracle on identical inputs."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1806_08020_b200 as ppa
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ppa_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ppa_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 40
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1806_08020_b200", "libppa_b200.so"))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    # the shipped fatbin holds sm_100a SASS (no PTX-JIT fallback for other archs)
    import subprocess

    so = os.path.join(ROOT, "paper_1806_08020_b200", "libppa_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert ppa.lib().ppa_abi_version() == 3


def test_solve_config_default_matches_cpp():
    # ppa_solve_config_default fills SolveConfig's defaults (inc/solver.hpp:21-58),
    # including the delayed-CGS2 orthogonalisation the C++/Python layers use
    from paper_1806_08020_b200 import _capi
    c = _capi._SolveConfigC()
    assert ppa.lib().ppa_solve_config_default(ctypes.byref(c)) == 0
    assert (c.m, c.k, c.nev, c.degree, c.max_cycles) == (50, 20, 15, 0, 100)
    assert c.rtol_multiplier == 1e-8 and c.rtol_absolute == 0.0
    assert c.orthogonalization == 1 and ppa.SolveConfig().orthogonalization == "dcgs2"


@pytest.mark.parametrize("name,gen", [
    ("bidiag", lambda M: M.bidiagonal(777)),
    ("convdiff_ref", lambda M: M.convection_diffusion(50)),
    ("convdiff_const", lambda M: M.convection_diffusion_const(45, 0.5)),
    ("laplace3d", lambda M: M.laplacian_3d(17)),
    ("random_poisson", lambda M: M.random_poisson(20000, 16.0, 7)),
])
def test_generators_bit_exact(name, gen):
    P, Q = gen(ppa.CsrMatrix), gen(O.Csr)
    assert P.info() == Q.info()
    for a, b in zip(P.arrays(), Q.arrays()):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_config_fingerprints(k):
    fp = json.load(open(os.path.join(ROOT, "tests", "golden", "fingerprints.json")))
    n, nnz, f = ppa.CsrMatrix.config(k).info()
    assert (n, nnz, str(f)) == (fp[f"config{k}"]["n"], fp[f"config{k}"]["nnz"],
                                 fp[f"config{k}"]["fingerprint"])


def test_rng_streams_bit_exact():
    for seed, stream in [(1, 1), (2, 2), (3, 3), (12345, 4)]:
        assert np.array_equal(ppa.normal_vector(1001, seed, stream),
                              O.normal_vector(1001, seed, stream))
    v = ppa.normal_vector(200000, 7, 3)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1) < 0.01
    # threaded path (chunks split across host threads), odd length
    assert np.array_equal(ppa.normal_vector(200001, 7, 3), O.normal_vector(200001, 7, 3))


def _roots(rng, k_real=20, k_cplx=8):
    r = rng.uniform(0.5, 500.0, k_real)
    z = rng.uniform(1, 300, k_cplx) + 1j * rng.uniform(0.5, 40, k_cplx)
    allr = np.concatenate([r, z, np.conj(z)])
    rng.shuffle(allr)
    return allr


def test_leja_bit_exact():
    rng = np.random.default_rng(5)
    for _ in range(20):
        roots = _roots(rng)
        assert np.array_equal(ppa.leja_order(roots), O.leja_order(roots))
    assert np.array_equal(ppa.leja_order([1, 10, 5]), [10, 1, 5])


def test_pof_and_stability_bit_exact():
    rng = np.random.default_rng(6)
    for _ in range(10):
        roots = O.leja_order(_roots(rng))
        a, b = ppa.compute_pof(roots), O.compute_pof(roots)
        assert np.array_equal(a["log10_pof"], b["log10_pof"])
        assert np.array_equal(a["copies_needed"], b["copies_needed"])
    for lg in (5, 10, 18.5, 20, 40):
        roots = [1.0 - 10.0 ** lg, 1.0, 3.0]
        assert np.array_equal(ppa.add_stability_roots(roots), O.add_stability_roots(roots))
    big = 1e12 + 1e11j
    roots = [big, np.conj(big), 1.0, 2.0]
    assert np.array_equal(ppa.add_stability_roots(roots), O.add_stability_roots(roots))


def test_eval_poly_matches():
    roots = [3.0, 5 + 1j, 5 - 1j]
    for z in (0, 1.5, 2 + 3j):
        assert ppa.eval_poly(roots, z) == O.eval_poly(roots, z)


def test_validation_messages():
    with pytest.raises(ValueError, match="strictly increasing"):
        ppa.CsrMatrix.from_arrays(2, [0, 2, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="row_ptr endpoints"):
        ppa.CsrMatrix.from_arrays(2, [0, 1, 3], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="empty root list"):
        ppa.leja_order([])
    with pytest.raises(ValueError, match="at least two roots"):
        ppa.compute_pof([2.0])
    with pytest.raises(ValueError, match="config must be"):
        ppa.CsrMatrix.config(9)


def test_from_triplets_matches_oracle():
    rng = np.random.default_rng(2)
    r = rng.integers(0, 50, 400)
    c = rng.integers(0, 50, 400)
    v = rng.standard_normal(400)
    P = ppa.CsrMatrix.from_triplets(50, r, c, v)
    Q = O.Csr.from_triplets(50, r, c, v)
    for a, b in zip(P.arrays(), Q.arrays()):
        assert np.array_equal(a, b)


def test_no_gpu_fails_loudly():
    """Without a GPU the CUDA path must raise, never fall back to the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception, match="CUDA|cuda"):
        ppa.make_csr_operator(ppa.CsrMatrix.bidiagonal(10))


def test_config_table():
    for k in range(1, 6):
        cfg = ppa.config_solve_config(k)
        assert cfg.m > cfg.k > 0
    assert ppa.CONFIGS[3]["n"] == 160 ** 3


def test_bench_launch_count_model():
    # bench.py's launches-per-step mirrors gmres_poly.cpp apply_poly_csr: a
    # real root is one launch and a pair two; with the two-factor pass two
    # consecutive real roots, or one pair, share a launch
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    roots = [5.0, 4.0, 3 + 1j, 3 - 1j, 2.0, 1 + 2j, 1 - 2j, 0.5, 0.25, 0.125]
    assert bench.count_launches(roots) == 10
    # passes: (5,4) (3+-1j) (2) (1+-2j) (0.5,0.25) (0.125)
    assert bench.count_launches(roots, True) == 6
    assert bench.count_launches([], True) == 0
    assert bench.count_launches([1.0] * 51, True) == 26


def test_grid2_slab_argument_checks():
    """The sharded box-grid entry points reject bad arguments with the
    reference's invalid_argument convention before any device work."""
    from paper_1806_08020_b200 import _capi as C

    vals7 = [-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0]
    fake = 1 << 20  # never dereferenced: every case fails validation first
    cases = [
        dict(nd=7, ny=8, zo0=0, zo1=8, kind=3),            # kind out of range
        dict(nd=7, ny=8, zo0=3, zo1=4, kind=0),            # a slab of one plane
        dict(nd=7, ny=8, zo0=2, zo1=8, kind=0),            # left neighbour missing
        dict(nd=5, ny=8, zo0=0, zo1=8, kind=0),            # 2-D stencil needs ny = 1
    ]
    for c in cases:
        vals = vals7 if c["nd"] == 7 else vals7[:5]
        with pytest.raises(ValueError):
            C.grid2_slab_pass(c["nd"], 8, c["ny"], 8, vals, c["zo0"], c["zo1"], c["kind"], 1.0,
                              0.0, 1.0, fake, fake + 4096)
    with pytest.raises(ValueError):
        C.grid2_slab_pass(7, 8, 8, 8, vals7, 0, 8, 0, 1.0, 0.0, 1.0, fake, fake)  # x == y
    with pytest.raises(ValueError):
        C.grid2_slab_chain(7, 8, 8, 8, vals7, 0, 8, [(5, 1.0, 0.0, 0.0)], fake, fake + 4096)
    with pytest.raises(ValueError):  # a right neighbour without its role-1 buffer
        C.grid2_slab_chain(7, 8, 8, 8, vals7, 0, 4, [(0, 1.0, 0.0, 1.0)], fake, fake + 4096,
                           xr=(fake + 8192, 0), fr=fake + 16384)
