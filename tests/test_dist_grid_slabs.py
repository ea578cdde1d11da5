"""Sharded box-grid pass with the halo exchange fused into the kernel
(dist.py ShardedGridPoly, kernels/spmv_grid2.cu slab mode).

CPU: the plane partition and the two-factor pass list.  GPU: z-slabs of 2-D
and 3-D boxes run as "virtual ranks" in one process - each slab's pass reads
its neighbours' buffers and waits on their epoch flags inside the kernel,
the slabs' passes are launched one after another on one stream (so no
kernel waits on a kernel that has not run; two ranks may not share a GPU
with kernels that wait on each other) - and the concatenated result must
equal the unsharded pi(A)v of the oracle bit for bit; the collective class
at world size 1."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_1806_08020_b200.dist import grid_passes, partition_planes


def test_partition_planes():
    assert partition_planes(160, 8)[0] == (0, 20) and partition_planes(160, 8)[-1] == (140, 160)
    assert partition_planes(7, 3) == [(0, 3), (3, 5), (5, 7)]
    with pytest.raises(ValueError):
        partition_planes(5, 3)  # a slab of one plane: its halo spans two ranks


def test_grid_passes():
    # the single-GPU chain's grouping: pairs alone, real roots two at a time,
    # a real root followed by a pair or by nothing alone
    plan = [(False, 1.0, 0.0), (False, 2.0, 0.0), (True, 3.0, 4.0), (False, 5.0, 0.0),
            (True, 6.0, 7.0), (False, 8.0, 0.0)]
    assert grid_passes(plan) == [(0, 1.0, 0.0, 2.0), (1, 3.0, 4.0, 0.0), (2, 5.0, 0.0, 0.0),
                                 (1, 6.0, 7.0, 0.0), (2, 8.0, 0.0, 0.0)]


def _box(nx, ny, nz, vals):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_dia2 import _box as box
    return box(nx, ny, nz, vals)


ROOTS = [4.5e4, 2e4 + 3e3j, 2e4 - 3e3j, 9e3, 150.0, 3e4, 1.2e3 + 4e2j, 1.2e3 - 4e2j, 6e3, 700.0]


def _virtual_slabs(cuda, nx, ny, nz, vals, world, roots, v):
    """Every slab's pass of every factor pair, in rank order per pass, on
    the current stream; returns the owned planes concatenated."""
    from paper_1806_08020_b200 import _capi as C

    nd = 7 if ny > 1 else 5
    D = nx * ny
    ranges = partition_planes(nz, world)
    passes = grid_passes(C.factor_plan(roots))
    bufs = [[cuda.zeros((z1 - z0) * D, dtype=cuda.float64, device="cuda") for _ in range(2)]
            for z0, z1 in ranges]
    flags = cuda.zeros((world, 8), dtype=cuda.int64, device="cuda")
    err = cuda.zeros(4, dtype=cuda.int32, device="cuda")
    fl = [flags[q].data_ptr() for q in range(world)]
    for q, (z0, z1) in enumerate(ranges):
        bufs[q][0].copy_(v[z0 * D:z1 * D])
        C.halo_publish(fl[q], 1)
    for k, (kind, a0, a1, b0) in enumerate(passes):
        for q, (z0, z1) in enumerate(ranges):
            left, right = q - 1 if q > 0 else None, q + 1 if q + 1 < world else None
            C.grid2_slab_pass(nd, nx, ny, nz, vals, z0, z1, kind, a0, a1, b0,
                              bufs[q][k % 2], bufs[q][(k + 1) % 2],
                              xl=bufs[left][k % 2].data_ptr() if left is not None else 0,
                              zl0=ranges[left][0] if left is not None else 0,
                              fl=fl[left] if left is not None else 0,
                              xr=bufs[right][k % 2].data_ptr() if right is not None else 0,
                              fr=fl[right] if right is not None else 0,
                              epoch=1 + k, err=err.data_ptr(), own=fl[q])
    assert int(err[0].item()) == 0
    # every pass published its epoch from inside (flag word 0; word 1 counts
    # the publishing CTAs); a lone slab has no neighbours to publish to
    assert flags[:, 0].tolist() == [1 + len(passes) if world > 1 else 1] * world
    return torch.cat([bufs[q][len(passes) % 2] for q in range(world)]).cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("box,world", [((40, 30, 24), 2), ((40, 30, 24), 3), ((40, 30, 24), 5),
                                       ((160, 160, 8), 2), ((64, 1, 50), 2), ((64, 1, 50), 4),
                                       ((2048, 1, 12), 3)])
@pytest.mark.parametrize("sym", [False, True])
def test_slab_passes_bit_exact(cuda, box, world, sym):
    # slabs of 2-D and 3-D boxes; Leja order interleaves conjugate pairs,
    # real-root pairs and lone real roots (one-level passes): the sharded
    # passes reproduce the unsharded pi(A)v bit for bit
    from oracle import oracle as O

    nx, ny, nz = box
    nd = 7 if ny > 1 else 5
    if sym:
        vals = [-2.5] * (nd // 2) + [9.0] + [-2.5] * (nd // 2)
    else:
        vals = [float(t) for t in np.random.default_rng(nx + nz).choice(
            [-1.0, 2.5, -0.75, 4.0, 0.5, -3.0, 6.0], size=nd)]
    n, rp, ci, vv = _box(nx, ny, nz, vals)
    v = O.normal_vector(n, 5, 5)
    roots = O.leja_order(ROOTS)
    got = _virtual_slabs(cuda, nx, ny, nz, vals, world, roots, cuda.tensor(v, device="cuda"))
    ref = O.apply_poly(roots, O.csr_operator(O.Csr.from_arrays(n, rp, ci, vv)), v)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_slab_pass_matches_single_gpu_pass(cuda):
    # one slab = the whole box: the slab entry point equals the operator's
    # own box-grid chain on config-3-shaped planes
    import paper_1806_08020_b200 as ppa
    from oracle import oracle as O

    nx = ny = 160
    nz = 10
    h2 = 161.0 ** 2
    vals = [-h2, -h2, -h2, 6 * h2, -h2, -h2, -h2]
    n, rp, ci, vv = _box(nx, ny, nz, vals)
    v = O.normal_vector(n, 2, 3)
    roots = O.leja_order(np.linspace(30.0, 311000.0, 8))
    got = _virtual_slabs(cuda, nx, ny, nz, vals, 1, roots, cuda.tensor(v, device="cuda"))
    A = ppa.make_csr_operator(ppa.CsrMatrix.from_arrays(n, rp, ci, vv))
    y = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.apply_poly(roots, A, cuda.tensor(v, device="cuda"), y)
    assert np.array_equal(got, y.cpu().numpy())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_sharded_grid_poly_ws1(cuda):
    # the collective class at world size 1 (IPC export, flags, fence,
    # publish; no neighbours), twice in a row: equals the oracle
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1806_08020_b200.dist import ShardedGridPoly

    if not dist.is_initialized():
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
                          WORLD_SIZE="1")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        nx, ny, nz = 48, 20, 16
        vals = [-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0]
        n, rp, ci, vv = _box(nx, ny, nz, vals)
        sg = ShardedGridPoly(nx, ny, nz, vals, dist)
        roots = O.leja_order(ROOTS)
        ref_op = O.csr_operator(O.Csr.from_arrays(n, rp, ci, vv))
        for seed in (3, 4):
            v = O.normal_vector(n, seed, seed)
            out = sg.apply(roots, cuda.tensor(v, device="cuda")).clone()
            sg.check()
            assert np.array_equal(out.cpu().numpy(), O.apply_poly(roots, ref_op, v))
        sg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_solve_on_grid_slabs_ws1(cuda):
    # the sharded solve with its polynomial operator on the fused-halo slab
    # pass reproduces the same solve on the plan's exchange exactly (both
    # pi(A)v paths are bit-identical to the unsharded product)
    import torch.distributed as dist

    import paper_1806_08020_b200 as ppa
    from paper_1806_08020_b200.dist import (CudaBackend, HaloPlan, ShardedGridPoly,
                                            ShardedSolver, box_row_ranges)

    if not dist.is_initialized():
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
                          WORLD_SIZE="1")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        N = 24
        P = ppa.CsrMatrix.laplacian_3d(N)
        n = P.n
        rp, ci, va = P.arrays()
        mid = ((N // 2) * N + N // 2) * N + N // 2  # an interior row: its 7 values in order
        vals = [float(t) for t in va[rp[mid]:rp[mid + 1]]]
        plan = HaloPlan.build(rp, ci, va, n, dist, ranges=box_row_ranges(N, N, N, 1))
        vec = lambda s: torch.tensor(ppa.normal_vector(n, 2, s), device="cuda")
        out = []
        for grid in (None, ShardedGridPoly(N, N, N, vals, dist)):
            sol = ShardedSolver(plan, CudaBackend(plan), dist, grid=grid)
            out.append(sol.solve(vec(2), vec(3), vec(1), 40, 20, 15, degree=20, max_cycles=60))
            if grid is not None:
                grid.check()
                grid.close()
        a, b = out
        assert a["converged"] and b["converged"]
        assert a["cycles"] == b["cycles"] and a["mvps"] == b["mvps"]
        assert np.array_equal(np.asarray(a["eigenvalues"]), np.asarray(b["eigenvalues"]))
    finally:
        dist.destroy_process_group()
