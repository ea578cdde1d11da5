"""World-size-2 CPU (gloo) coverage of the N>1 bench path: replicas run the
same seeded pi(A)v independently (no data-path collective; DESIGN.md
"Multi-GPU: replicas only"), timing is the max over ranks, and the whole-job
value is the weak-scaling aggregate."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    import sys
    import time

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws))
    import torch.distributed as dist

    import bench
    from oracle import oracle as O

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    O.set_threads(1)
    A = O.csr_operator(O.Csr.laplacian_3d(16))
    roots = O.leja_order(np.linspace(30.0, 3000.0, 6))
    v = O.normal_vector(16 ** 3, 2, 3)
    t0 = time.perf_counter()
    y = O.apply_poly(roots, A, v)
    ms = (time.perf_counter() - t0) * 1e3 * (1 + rank)  # rank-dependent timing
    mx = bench.reduce_max(ms, ws)
    digest = float(np.sum(y * np.arange(len(y))))
    out = [0.0, 0.0]
    import torch

    t = torch.tensor([digest], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = (ms, mx, digest, float(t.item()), bench.whole_job_gbs(1e9, mx, ws))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_gloo_ws2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (ms0, mx0, d0, dmax0, v0), (ms1, mx1, d1, dmax1, v1) = res[0], res[1]
    assert mx0 == mx1 == max(ms0, ms1)           # max over ranks
    assert d0 == d1 == dmax0                     # replicas are bit-identical
    assert v0 == pytest.approx(2 * 1e9 / (mx0 * 1e-3) / 1e9)  # weak-scaling aggregate
