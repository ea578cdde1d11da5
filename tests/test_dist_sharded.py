"""Row-block sharded pi(A)v (paper_1806_08020_b200/dist.py): the halo plan and
exchange logic on CPU over gloo with world sizes 2 and 3, the local arithmetic
supplied by an oracle-backed test backend; and the product CUDA backend at
world size 1 on the GPU.  Every owned row is summed in the CSR's column order,
so the sharded result must equal the unsharded oracle pi(A)v bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    "laplace3d": lambda O: O.Csr.laplacian_3d(11),
    "convdiff": lambda O: O.Csr.convection_diffusion(25),
    "random": lambda O: O.Csr.random_poisson(1500, 6.0, 9),
    "bidiag": lambda O: O.Csr.bidiagonal(701),
}


def _roots(O):
    return O.leja_order([3.0, 900.0, 450.0 + 120.0j, 450.0 - 120.0j, 75.0])


class OracleBackend:
    """Test-only CPU backend: torch CPU vectors, the oracle's CSR loop for the
    products and numpy for the (FMA-free) factor epilogues."""

    def __init__(self, plan, O):
        m = O.Csr.from_arrays(plan.n_ext, plan.row_ptr, plan.col_idx, plan.values)
        self.op = O.csr_operator(m)

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64)

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def gather(self, t, idx):
        return t[torch.as_tensor(idx)].contiguous()

    def copy_(self, dst, src):
        dst.copy_(src)

    # tall-skinny primitives of the sharded solve (torch CPU stand-ins for
    # the CUDA backend's kernels; same contracts)
    def basis(self, cols, n):
        ld = (n + 31) // 32 * 32
        return torch.zeros((cols, ld), dtype=torch.float64), ld

    def cgs_dot(self, V, ld, n, c, w):
        return V[:c, :n] @ w

    def cgs_update_dot(self, V, ld, n, c, w, h):
        w -= V[:c, :n].T @ h
        return torch.cat([V[:c, :n] @ w, (w @ w).reshape(1)])

    def cgs_store(self, V, ld, n, c, w, h2, hsub):
        V[c, :n] = (w - V[:c, :n].T @ h2) / hsub

    def combine(self, V, ld, n, d, G, p, Out, ldo):
        Y = (torch.as_tensor(np.asarray(G, dtype=np.float64)).T @ V[:d, :n]).clone()
        Out[:p, :n] = Y

    def dot(self, x, y):
        return (x @ y).reshape(1)

    def factor(self, x, y, mode, c0=0.0, c1=0.0, o=None):
        xs = x.numpy()
        s = self.op.apply(xs)
        if mode == 0:
            z = s
        elif mode == 1:
            z = xs + c0 * s
        else:
            z = (o.numpy() + c1 * xs) + c0 * s
        y.copy_(torch.from_numpy(z))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1806_08020_b200.dist import HaloPlan, ShardedPoly

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        O.set_threads(1)
        P = CASES[case](O)
        n = P.info()[0]
        rp, ci, va = P.arrays()
        plan = HaloPlan.build(rp, ci, va, n, dist)
        sp = ShardedPoly(plan, OracleBackend(plan, O), dist)
        v = O.normal_vector(n, 3, 3)
        r0, r1 = plan.ranges[rank]
        out = sp.apply(_roots(O), torch.tensor(v[r0:r1]))
        q.put((rank, r0, r1, out.numpy().copy(), sorted(plan.send), sorted(plan.recv)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_pi_gloo(ws, case):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, case, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = CASES[case](O)
    n = P.info()[0]
    ref = O.apply_poly(_roots(O), O.csr_operator(P), O.normal_vector(n, 3, 3))
    got = np.zeros(n)
    for rank, r0, r1, out, send, recv in res:
        got[r0:r1] = out
    assert np.array_equal(got, ref)
    if case in ("laplace3d", "convdiff", "bidiag"):  # banded: neighbours only
        for rank, r0, r1, out, send, recv in res:
            assert set(send) <= {rank - 1, rank + 1} and set(recv) <= {rank - 1, rank + 1}


def _pull_worker(rank, ws, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1806_08020_b200.dist import HaloPlan, ShardedPoly, peer_pull_lists

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        P = CASES[case](O)
        n = P.info()[0]
        plan = HaloPlan.build(*P.arrays(), n, dist)
        sp = ShardedPoly(plan, OracleBackend(plan, O), dist)
        # a vector whose owned entries are the global row numbers
        x = torch.zeros(plan.n_ext, dtype=torch.float64)
        r0, r1 = plan.ranges[rank]
        x[plan.owned] = torch.arange(r0, r1, dtype=torch.float64)
        sends = [None] * ws
        dist.all_gather_object(sends, plan.send)
        xs = [None] * ws
        dist.all_gather_object(xs, x.numpy().copy())
        # the peer pull from every owner's buffer, simulated on the host
        pulled = x.clone().numpy()
        for owner, idx, off in peer_pull_lists(plan, sends, rank):
            pulled[off:off + idx.size] = xs[owner][idx]
        sp.exchange(x)  # NCCL-style exchange (gloo here)
        q.put((rank, bool(np.array_equal(pulled, x.numpy()))))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("case", ["laplace3d", "random"])
def test_peer_pull_lists_match_exchange(ws, case):
    # the peer-memory halo (dist.PeerHalo) pulls exactly what the
    # point-to-point exchange delivers, for banded and random matrices
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_pull_worker, args=(r, ws, port, case, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values()), res


def _solve_worker(rank, ws, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1806_08020_b200.dist import HaloPlan, ShardedSolver

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        O.set_threads(1)
        P, kw = SOLVES[case](O)
        n = P.info()[0]
        plan = HaloPlan.build(*P.arrays(), n, dist)
        r0, r1 = plan.ranges[rank]
        vec = lambda s: torch.tensor(O.normal_vector(n, kw["seed"], s)[r0:r1])
        sol = ShardedSolver(plan, OracleBackend(plan, O), dist)
        r = sol.solve(vec(2), vec(3), vec(1), kw["m"], kw["k"], kw["nev"], degree=kw["degree"],
                      max_cycles=kw["max_cycles"])
        q.put((rank, r))
        dist.barrier()
    finally:
        dist.destroy_process_group()


SOLVES = {
    "config1": lambda O: (O.Csr.config(1), dict(m=30, k=15, nev=10, degree=10, seed=1,
                                               max_cycles=100)),
    "laplace3d": lambda O: (O.Csr.laplacian_3d(12), dict(m=30, k=15, nev=6, degree=0, seed=2,
                                                         max_cycles=200)),
}


@pytest.mark.parametrize("case", sorted(SOLVES))
def test_sharded_solve_gloo_ws2(case):
    # the row-sharded solve (all reductions all-reduced) agrees with the
    # single-process oracle solve: same eigenvalues, matvec count within 5 %
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_solve_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    P, kw = SOLVES[case](O)
    o = O.solve(O.csr_operator(P), kw["m"], kw["k"], kw["nev"], degree=kw["degree"],
                seed=kw["seed"], max_cycles=kw["max_cycles"])
    a, b = res[0], res[1]
    assert np.array_equal(a["eigenvalues"], b["eigenvalues"])  # replicated decisions
    assert a["converged"] and o["converged"]
    assert np.all(a["residuals"] <= a["rtol"])
    got, ref = np.sort_complex(a["eigenvalues"]), np.sort_complex(o["eigenvalues"])
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-8
    assert abs(a["mvps"] - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]


def test_partition_and_local_part():
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_1806_08020_b200.dist import HaloPlan, partition_rows

    assert partition_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition_rows(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    P = O.Csr.laplacian_3d(6)
    rp, ci, va = P.arrays()
    ranges = partition_rows(216, 3)
    nl, nloc, nr, lrp, lci, vals, recv, wants = HaloPlan.local_part(rp, ci, va, ranges, 1)
    assert nloc == 72 and nl == 36 and nr == 36  # one 6x6 plane each side
    # monotone renumbering: local columns increase along every owned row
    for i in range(nl, nl + nloc):
        row = lci[lrp[i]:lrp[i + 1]]
        assert np.all(np.diff(row) > 0)
    assert recv == {0: (0, 36), 2: (nl + nloc, nl + nloc + 36)}
    assert wants[0] == list(range(36, 72)) and wants[2] == list(range(144, 180))


@pytest.mark.gpu
def test_sharded_cuda_backend_ws1(cuda):
    # the product backend at world size 1 (no halo): the sharded driver and
    # ppa_spmv_factor reproduce apply_poly bit for bit
    import torch.distributed as dist

    import paper_1806_08020_b200 as ppa
    from oracle import oracle as O
    from paper_1806_08020_b200.dist import CudaBackend, HaloPlan, ShardedPoly

    if not dist.is_initialized():
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
                          WORLD_SIZE="1")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        P = ppa.CsrMatrix.laplacian_3d(14)
        n = P.n
        rp, ci, va = P.arrays()
        plan = HaloPlan.build(rp, ci, va, n, dist)
        sp = ShardedPoly(plan, CudaBackend(plan), dist)
        v = O.normal_vector(n, 3, 3)
        out = sp.apply(_roots(O), torch.tensor(v, device="cuda"))
        ref = O.apply_poly(_roots(O), O.csr_operator(O.Csr.laplacian_3d(14)), v)
        assert np.array_equal(out.cpu().numpy(), ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_solve_cuda_ws1(cuda):
    # the product backend drives the sharded solve at world size 1 and agrees
    # with the device solve (eigenvalues 1e-8, matvec count within 5 %)
    import torch.distributed as dist

    import paper_1806_08020_b200 as ppa
    from oracle import oracle as O
    from paper_1806_08020_b200.dist import CudaBackend, HaloPlan, ShardedSolver

    if not dist.is_initialized():
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
                          WORLD_SIZE="1")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        P = ppa.CsrMatrix.config(1)
        n = P.n
        plan = HaloPlan.build(*P.arrays(), n, dist)
        vec = lambda s: torch.tensor(ppa.normal_vector(n, 1, s), device="cuda")
        sol = ShardedSolver(plan, CudaBackend(plan), dist)
        r = sol.solve(vec(2), vec(3), vec(1), 30, 15, 10, degree=10, max_cycles=100)
        g = ppa.solve(ppa.make_csr_operator(P), ppa.config_solve_config(1))
        assert r["converged"] and g["converged"]
        got, ref = np.sort_complex(r["eigenvalues"]), np.sort_complex(g["eigenvalues"])
        assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-8
        assert abs(r["mvps"] - g["cost"]["mvps"]) <= 0.05 * g["cost"]["mvps"]
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_local_cgs_sweeps_equal_cgs2_step(cuda):
    # the rank-local sweeps of the sharded solve at world size 1 (no
    # all-reduce) reproduce the single-GPU CGS2 step bit for bit: same
    # kernels, same summation order
    import paper_1806_08020_b200 as ppa
    from oracle import oracle as O

    P = ppa.CsrMatrix.laplacian_3d(30)
    A = ppa.make_csr_operator(P)
    n, c = P.n, 24
    st = ppa.arnoldi_init(cuda.tensor(O.normal_vector(n, 5, 3), device="cuda"), n, c)
    st.extend(A, c)
    ld = st.ld
    w0 = cuda.empty(n, dtype=cuda.float64, device="cuda")
    ppa.spmv(A, st.V_ptr + 8 * ld * (c - 1), w0)
    # reference: the fused single-GPU step into a copy of the basis
    V = cuda.empty((c + 1) * ld, dtype=cuda.float64, device="cuda")
    V.copy_(cuda.as_tensor(np.zeros((c + 1) * ld), device="cuda"))
    ppa.ts_combine(st.V_ptr, ld, n, c, cuda.tensor(np.eye(c).T.ravel(), device="cuda"), c, V, ld)
    V2 = V.clone()
    w = w0.clone()
    Hc = cuda.empty(c + 2, dtype=cuda.float64, device="cuda")
    flag = cuda.zeros(2, dtype=cuda.int32, device="cuda")
    ppa.cgs2_step(V, ld, n, c, w, Hc, flag)
    # the three local sweeps
    w2 = w0.clone()
    h1 = cuda.empty(c, dtype=cuda.float64, device="cuda")
    s2 = cuda.empty(c + 1, dtype=cuda.float64, device="cuda")
    ppa._capi.cgs_dot_local(V2, ld, n, c, w2, h1)
    ppa._capi.cgs_update_dot_local(V2, ld, n, c, w2, h1, s2)
    h2 = s2[:c].cpu().numpy()
    d2 = float(s2[c].item()) - float(sum(x * x for x in h2))
    hs = cuda.full((1,), np.sqrt(d2), dtype=cuda.float64, device="cuda")
    ppa._capi.cgs_store_local(V2, ld, n, c, w2, s2[:c], hs)
    assert np.array_equal((h1 + s2[:c]).cpu().numpy(), Hc[:c].cpu().numpy())
    assert float(hs.item()) == float(Hc[c].item())
    assert cuda.equal(V2[c * ld:c * ld + n], V[c * ld:c * ld + n])
    # and the local dot of the reductions
    out = cuda.empty(1, dtype=cuda.float64, device="cuda")
    ppa._capi.dot_local(w0, w0, n, out)
    assert abs(float(out.item()) - float((w0 @ w0).item())) <= 1e-12 * float((w0 @ w0).item())


@pytest.mark.gpu
def test_peer_halo_pull_kernel(cuda):
    # the pull kernel on one GPU with a local "owner" buffer: the gather, the
    # fence (wait only) and the acquire wait on a flag published later from
    # another stream (no second rank: the wait primitive itself)
    import time

    from paper_1806_08020_b200 import _capi as C
    from paper_1806_08020_b200.dist import _DESC, _device_view

    n_src, n_ext = 5000, 300
    src = C.dev_alloc(8 * n_src)
    flag = C.dev_alloc(64)
    err = C.dev_alloc(16)
    try:
        sv = _device_view(cuda, src, n_src)
        sv.copy_(cuda.arange(n_src, dtype=cuda.float64, device="cuda") * 0.5)
        x = cuda.zeros(n_ext, dtype=cuda.float64, device="cuda")
        idx = cuda.tensor([7, 4999, 0, 123, 2500, 11], dtype=cuda.int64, device="cuda")
        desc = np.array([(src, idx.data_ptr(), 6, 100, flag)], dtype=_DESC)
        dd = cuda.as_tensor(desc.view(np.uint8), device="cuda")
        C.halo_publish(flag, 1)
        C.halo_pull(dd.data_ptr(), 1, 6, x, 1, err)
        cuda.cuda.synchronize()
        got = x.cpu().numpy()
        assert np.array_equal(got[100:106], 0.5 * np.array([7, 4999, 0, 123, 2500, 11]))
        assert not got[:100].any() and not got[106:].any()
        # wait: a fence for epoch 2 on a non-blocking stream spins until
        # another stream stores the flag
        import paper_1806_08020_b200 as ppa

        import threading

        from cuda.bindings import runtime as cudart

        def nb_stream():  # non-blocking: no implicit sync with the legacy stream
            err_, h = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
            assert int(err_) == 0
            return h

        ready, go = threading.Event(), threading.Event()

        def publisher():
            # another thread: its own library context and stream, set up
            # before the wait starts (creating a context synchronises the
            # device, which would wait for the spinning kernel itself)
            sb = nb_stream()
            ppa.set_stream(int(sb))
            C.halo_publish(flag, 1)
            cudart.cudaStreamSynchronize(sb)
            ready.set()
            go.wait()
            C.halo_publish(flag, 2)
            cudart.cudaStreamSynchronize(sb)

        th = threading.Thread(target=publisher)
        th.start()
        ready.wait()
        sa = nb_stream()
        ppa.set_stream(int(sa))
        try:
            C.halo_pull(dd.data_ptr(), 1, 0, None, 2, err)
            time.sleep(0.05)
            assert int(cudart.cudaStreamQuery(sa)[0]) != 0  # still waiting
            go.set()
            th.join()
            cudart.cudaStreamSynchronize(sa)
        finally:
            ppa.set_stream(cuda.cuda.current_stream())
        cuda.cuda.synchronize()
        e = _device_view(cuda, err, 2, cuda.int32).cpu().numpy()
        assert e[0] == 0, e
        h = C.ipc_get_handle(src)
        assert len(h) == 64 and any(h)
    finally:
        for p in (src, flag, err):
            C.dev_free(p)


@pytest.mark.gpu
def test_sharded_peer_ws1(cuda):
    # PeerHalo at world size 1 (no peers: the fence and publish still run)
    # leaves the sharded pi(A)v bit-identical to apply_poly
    import torch.distributed as dist

    import paper_1806_08020_b200 as ppa
    from oracle import oracle as O
    from paper_1806_08020_b200.dist import CudaBackend, HaloPlan, ShardedPoly

    if not dist.is_initialized():
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
                          WORLD_SIZE="1")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        P = ppa.CsrMatrix.laplacian_3d(14)
        plan = HaloPlan.build(*P.arrays(), P.n, dist)
        sp = ShardedPoly(plan, CudaBackend(plan), dist, peer=True)
        v = O.normal_vector(P.n, 3, 3)
        out = sp.apply(_roots(O), torch.tensor(v, device="cuda")).clone()
        sp.peer.check()
        ref = O.apply_poly(_roots(O), O.csr_operator(O.Csr.laplacian_3d(14)), v)
        assert np.array_equal(out.cpu().numpy(), ref)
    finally:
        dist.destroy_process_group()
