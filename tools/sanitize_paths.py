"""Every kernel family of the hot path once, at small sizes, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_paths.py [part ...]

Parts (default: all): spmv, grid, poly, arnoldi, solve.  Each part checks its
results against the SELL-32 path or known answers, so a sanitizer run is also
a functional run.  PYTORCH_NO_CUDA_MEMORY_CACHING=1 (set by the wrapper
tools/gpu/run_sanitizer.sh) makes every torch tensor its own cudaMalloc, so
memcheck sees accesses past a vector's end.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1806_08020_b200 as ppa  # noqa: E402

torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
dev = "cuda"


def vec(n, seed=1):
    return torch.tensor(ppa.normal_vector(n, seed, ppa.STREAM_ARNOLDI), device=dev)


def mats():
    return {
        "bidiag": ppa.CsrMatrix.bidiagonal(3000),
        "convdiff2d": ppa.CsrMatrix.convection_diffusion_const(70),
        "laplace3d": ppa.CsrMatrix.laplacian_3d(22),
        "poisson": ppa.CsrMatrix.random_poisson(6000, 16.0, 4),
    }


ROOTS = ppa.leja_order(np.array([9000.0, 4000 + 900j, 4000 - 900j, 1500.0, 300.0, 40.0, 7.0]))


def part_spmv():
    """SpMV and the fused factor chain in every layout, bit-identical to SELL-32."""
    for name, m in mats().items():
        n = m.n
        x = vec(n)
        ref = None
        for lay in ("sell32", "csr", "sell32_packed", "dia_coded", "auto"):
            A = ppa.make_csr_operator(m, lay)
            y = torch.empty(n, dtype=torch.float64, device=dev)
            ppa.spmv(A, x, y)
            out = torch.empty(n, dtype=torch.float64, device=dev)
            ppa.apply_poly(ROOTS, A, x, out)
            torch.cuda.synchronize()
            got = (y.cpu().numpy(), out.cpu().numpy())
            if ref is None:
                ref = got
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), (name, lay)
        print("spmv ok", name, A.layout()["layout"])


def part_grid():
    """The two-factor passes (presence form and box-grid form), complement included."""
    for name in ("convdiff2d", "laplace3d"):
        m = mats()[name]
        n = m.n
        x = vec(n, 2)
        S = ppa.make_csr_operator(m, "sell32")
        A = ppa.make_csr_operator(m)
        assert A.layout()["two_factor_pass"], A.layout()
        for mk in (ppa.make_poly_operator, ppa.make_poly_complement_operator):
            ya = torch.empty(n, dtype=torch.float64, device=dev)
            ys = torch.empty(n, dtype=torch.float64, device=dev)
            mk(A, ROOTS).apply(x, ya)
            mk(S, ROOTS).apply(x, ys)
            torch.cuda.synchronize()
            assert torch.equal(ya, ys), (name, mk.__name__)
        print("grid ok", name, A.layout()["grid"], A.layout()["grid_pass"])


def part_poly():
    """build_gmres_poly (device Arnoldi under delayed CGS2) and the nested operator."""
    m = mats()["convdiff2d"]
    A = ppa.make_csr_operator(m)
    b = vec(m.n, 3)
    roots, _ = ppa.build_gmres_poly(A, b, 8)
    tau = ppa.make_poly_complement_operator(A, roots)
    phi = ppa.make_poly_operator(tau, ROOTS[:3])
    y = torch.empty(m.n, dtype=torch.float64, device=dev)
    phi.apply(b, y)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    print("poly ok", len(roots), phi.mvps_per_apply())


def part_arnoldi():
    """arnoldi_init / extend under both orthogonalisations, restart, Ritz vectors, spmm."""
    m = mats()["laplace3d"]
    n = m.n
    A = ppa.make_csr_operator(m)
    for ortho in ("cgs2", "dcgs2"):
        st = ppa.arnoldi_init(vec(n, 5), n, 12)
        st.set_orthogonalization(ortho)
        st.extend(A, 12)
        kk = st.thick_restart(5)
        st.extend(A, 12)
        yr = torch.empty(n, dtype=torch.float64, device=dev)
        yi = torch.empty(n, dtype=torch.float64, device=dev)
        st.ritz_vector(0, yr, yi)
        torch.cuda.synchronize()
        H = st.H
        assert np.isfinite(H).all() and st.cur_dim == 12, (ortho, st.cur_dim)
        print("arnoldi ok", ortho, "restart kept", kk, "ld", st.ld)
    Y = torch.stack([vec(n, s) for s in (1, 2, 3)]).contiguous()  # 3 columns, ld = n
    AY = torch.empty_like(Y)
    ppa.spmm(A, Y, n, 3, AY, n)
    y1 = torch.empty(n, dtype=torch.float64, device=dev)
    for j in range(3):
        ppa.spmv(A, Y[j], y1)
        torch.cuda.synchronize()
        assert torch.equal(AY[j], y1), j
    print("spmm ok")


def part_solve():
    """One polynomial-preconditioned solve and one double-polynomial solve."""
    r = ppa.solve(ppa.make_csr_operator(ppa.CsrMatrix.bidiagonal(2000)),
                  ppa.SolveConfig(m=20, k=10, nev=5, degree=6, seed=1, want_eigenvectors=True))
    lam = np.sort(r["eigenvalues"].real)
    assert r["converged"] and np.allclose(lam, np.arange(1.0, 6.0), rtol=1e-8), lam
    print("solve ok", r["cycles"], r["cost"]["mvps"])
    m = ppa.CsrMatrix.laplacian_3d(14)
    r = ppa.solve_double(ppa.make_csr_operator(m),
                         ppa.SolveConfig(m=16, k=8, nev=4, double_d1=3, double_d2=4, seed=3,
                                         max_cycles=30))
    print("solve_double ok", r["converged"], r["cycles"], r["cost"]["mvps"])


PARTS = {"spmv": part_spmv, "grid": part_grid, "poly": part_poly, "arnoldi": part_arnoldi,
         "solve": part_solve}

if __name__ == "__main__":
    for p in (sys.argv[1:] or list(PARTS)):
        PARTS[p]()
    torch.cuda.synchronize()
    print("sanitize_paths: all parts done")
