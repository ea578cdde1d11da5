"""Row-block sharded pi(A)v over torch.distributed.

Rank q owns the rows [r0_q, r1_q) of A and the same block of every vector.
Its local matrix keeps the owned rows with the columns renumbered into an
extended vector

    x_ext = [ left halo (n_left) | owned block (n_local) | right halo ]

where the halos are the off-rank columns the owned rows touch, lower-ranked
owners on the left and higher-ranked on the right, each sorted.  The
renumbering is monotone, so every row keeps its entries in global column
order, and the owned rows sit at local rows n_left.. (near the diagonal, so
the stencil layouts still apply).  A product A x then needs exactly one
exchange: each rank sends every peer the owned entries that peer's rows touch
(planned once, by swapping the receive lists) and receives its halos;
afterwards the local fused factor kernel runs on x_ext unchanged.  Banded
matrices only talk to neighbouring ranks (config 3 split in z-slabs: 160^2
rows per neighbour and SpMV, against ~53 MB of local matrix stream).

The point-to-point exchange is the path's only data collective, so pi(A)v
needs one halo exchange per SpMV (two per conjugate pair) and no reduction.
Each owned row is summed in the CSR's own column order by the same kernels
as the single-GPU path, so the sharded pi(A)v is bit-identical to the
unsharded one for any number of ranks.

The local arithmetic is supplied by a backend:
  * CudaBackend (the product): torch CUDA tensors and the C-ABI factor kernel
    (ppa_spmv_factor), exchange over NCCL;
  * the tests plug an oracle-backed CPU backend in to run the exchange logic
    on gloo with world size 2 and 3.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


def partition_rows(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous row blocks, sizes differing by at most one."""
    if world < 1:
        raise ValueError("partition_rows: world must be >= 1")
    base, extra = divmod(n, world)
    out, r0 = [], 0
    for q in range(world):
        r1 = r0 + base + (1 if q < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def owner_of(col: np.ndarray, ranges: Sequence[Tuple[int, int]]) -> np.ndarray:
    starts = np.array([r0 for r0, _ in ranges], dtype=np.int64)
    return np.searchsorted(starts, col, side="right") - 1


@dataclass
class HaloPlan:
    """Local matrix and exchange lists of one rank."""

    rank: int
    ranges: List[Tuple[int, int]]
    n_left: int
    n_local: int
    n_right: int
    # local square CSR over n_ext rows/columns; rows outside the owned block
    # [n_left, n_left + n_local) are empty
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    recv: Dict[int, Tuple[int, int]] = field(default_factory=dict)  # peer -> x_ext slice
    send: Dict[int, np.ndarray] = field(default_factory=dict)       # peer -> x_ext indices

    @property
    def n_ext(self) -> int:
        return self.n_left + self.n_local + self.n_right

    @property
    def owned(self) -> slice:
        return slice(self.n_left, self.n_left + self.n_local)

    @staticmethod
    def local_part(row_ptr, col_idx, values, ranges, rank):
        """Owned rows, renumbered columns and the receive lists (no communication)."""
        r0, r1 = ranges[rank]
        rp = np.asarray(row_ptr, dtype=np.int64)
        ci = np.asarray(col_idx, dtype=np.int64)
        va = np.asarray(values, dtype=np.float64)
        p0, p1 = int(rp[r0]), int(rp[r1])
        cols = ci[p0:p1]
        vals = va[p0:p1].copy()
        left = np.unique(cols[cols < r0])
        right = np.unique(cols[cols >= r1])
        n_left, n_local, n_right = int(left.size), r1 - r0, int(right.size)
        local_cols = np.empty_like(cols)
        lo, hi = cols < r0, cols >= r1
        mid = ~(lo | hi)
        local_cols[lo] = np.searchsorted(left, cols[lo])
        local_cols[mid] = n_left + (cols[mid] - r0)
        local_cols[hi] = n_left + n_local + np.searchsorted(right, cols[hi])
        n_ext = n_left + n_local + n_right
        lrp = np.zeros(n_ext + 1, dtype=np.int64)
        lrp[n_left + 1:n_left + n_local + 1] = rp[r0 + 1:r1 + 1] - p0
        lrp[n_left + n_local + 1:] = lrp[n_left + n_local]
        recv, wants = {}, {}
        for base, halo in ((0, left), (n_left + n_local, right)):
            if not halo.size:
                continue
            owners = owner_of(halo, ranges)
            for q in np.unique(owners):
                idx = np.nonzero(owners == q)[0]
                recv[int(q)] = (base + int(idx[0]), base + int(idx[-1]) + 1)
                wants[int(q)] = halo[idx].tolist()
        return (n_left, n_local, n_right, lrp.astype(np.int32), local_cols.astype(np.int32),
                vals, recv, wants)

    @classmethod
    def build(cls, row_ptr, col_idx, values, n: int, dist, group=None,
              ranges=None) -> "HaloPlan":
        """Collective: every rank calls it with the matrix rows it owns
        (the arrays may hold the whole matrix; only the owned rows are read).
        `ranges` overrides the row partition (e.g. box_row_ranges, so that the
        rows match a ShardedGridPoly's z-slabs)."""
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        ranges = list(ranges) if ranges is not None else partition_rows(n, world)
        if len(ranges) != world or ranges[0][0] != 0 or ranges[-1][1] != n:
            raise ValueError("HaloPlan.build: ranges must partition [0, n) over the ranks")
        (n_left, n_local, n_right, lrp, lci, vals, recv, wants) = cls.local_part(
            row_ptr, col_idx, values, ranges, rank)
        # tell each owner which of its columns this rank needs
        everyone: List[Optional[dict]] = [None] * world
        dist.all_gather_object(everyone, wants, group=group)
        send = {}
        r0 = ranges[rank][0]
        for q in range(world):
            if q == rank or everyone[q] is None:
                continue
            need = everyone[q].get(rank)
            if need:
                send[q] = n_left + (np.asarray(need, dtype=np.int64) - r0)
        return cls(rank=rank, ranges=ranges, n_left=n_left, n_local=n_local, n_right=n_right,
                   row_ptr=lrp, col_idx=lci, values=vals, recv=recv, send=send)


class CudaBackend:
    """Product backend: the local matrix as a device operator, vectors as
    torch CUDA tensors, factors through ppa_spmv_factor."""

    def __init__(self, plan: HaloPlan, layout: str = "auto"):
        import torch

        from . import _capi as C

        self.torch = torch
        self.C = C
        m = C.CsrMatrix.from_arrays(plan.n_ext, plan.row_ptr, plan.col_idx, plan.values)
        self.op = C.make_csr_operator(m, layout)

    def empty(self, n):
        return self.torch.empty(n, dtype=self.torch.float64, device="cuda")

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device="cuda")

    def from_host(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a), dtype=self.torch.float64,
                                    device="cuda")

    def to_host(self, t):
        return t.detach().cpu().numpy()

    def factor(self, x_ext, y_ext, mode, c0=0.0, c1=0.0, o=None):
        self.C.spmv_factor(self.op, x_ext, y_ext, mode, c0, c1, o)

    def gather(self, t, idx):
        return t[self.torch.as_tensor(idx, device=t.device)]

    def copy_(self, dst, src):
        dst.copy_(src)

    # -- tall-skinny basis kernels with rank-local sums (cgs.cu, tallskinny.cu)
    def basis(self, cols, n):
        """Column-major basis: row j of the returned (cols, ld) tensor is
        column j; ld a multiple of 32 doubles (TMA tiles, aligned columns)."""
        ld = (n + 31) // 32 * 32
        return self.torch.zeros((cols, ld), dtype=self.torch.float64, device="cuda"), ld

    def cgs_dot(self, V, ld, n, c, w):
        out = self.empty(c)
        self.C.cgs_dot_local(V, ld, n, c, w, out)
        return out

    def cgs_update_dot(self, V, ld, n, c, w, h):
        out = self.empty(c + 1)
        self.C.cgs_update_dot_local(V, ld, n, c, w, h, out)
        return out

    def cgs_store(self, V, ld, n, c, w, h2, hsub):
        self.C.cgs_store_local(V, ld, n, c, w, h2, hsub)

    def combine(self, V, ld, n, d, G, p, Out, ldo):
        g = self.torch.as_tensor(np.asfortranarray(G).ravel(order="F"), dtype=self.torch.float64,
                                 device="cuda")
        self.C.ts_combine(V, ld, n, d, g, p, Out, ldo)

    def dot(self, x, y):
        out = self.empty(1)
        self.C.dot_local(x, y, x.numel(), out)
        return out


def peer_pull_lists(plan: HaloPlan, sends: Sequence[Optional[dict]], rank: int):
    """What this rank pulls from each owner: [(owner, indices into the owner's
    x_ext, destination offset in this rank's x_ext)], from every rank's send
    lists (sends[q] = plan.send of rank q).  Pulling these reproduces
    ShardedPoly.exchange over NCCL entry for entry."""
    out = []
    for q, (a, z) in sorted(plan.recv.items()):
        idx = np.asarray(sends[q][rank], dtype=np.int64)
        if idx.size != z - a:
            raise RuntimeError(f"peer_pull_lists: rank {q} sends {idx.size} entries, "
                               f"{z - a} expected")
        out.append((q, idx, a))
    return out


_DESC = np.dtype([("src", "<u8"), ("src_index", "<u8"), ("count", "<i8"),
                  ("dst_offset", "<i8"), ("flag", "<u8")])  # ppa_peer_halo


class PeerHalo:
    """Halo exchange over peer memory (NVLink / NVSwitch) without NCCL
    (kernels/peer_halo.cu).  Collective constructor.

    Every rank allocates its ShardedPoly vectors (roles 0, 1: the ping-pong
    pair; 2: the pair temporary t1) and an epoch flag with ppa_dev_alloc,
    exports them as CUDA IPC handles, and maps the buffers and flags of the
    ranks it receives halos from.  An exchange of role r is then: publish my
    epoch e (after the kernel that wrote my role-r vector), and one pull
    kernel that waits for every owner's flag >= e and gathers
    x_ext[recv slice] = owner_vector[owner's send list] straight from the
    owners' HBM.  No collective call and no staging copy per SpMV."""

    ROLES = 3

    def __init__(self, plan: HaloPlan, dist, group=None):
        import torch

        from . import _capi as C

        self.C, self.torch, self.plan = C, torch, plan
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        n_ext = plan.n_ext
        self.bufs = [C.dev_alloc(8 * max(n_ext, 1)) for _ in range(self.ROLES)]
        self.flag = C.dev_alloc(64)
        self.err = C.dev_alloc(16)
        self.views = [_device_view(torch, b, n_ext) for b in self.bufs]
        mine = {"bufs": [C.ipc_get_handle(b) for b in self.bufs],
                "flag": C.ipc_get_handle(self.flag),
                "send": {int(q): np.asarray(idx, dtype=np.int64) for q, idx in plan.send.items()}}
        everyone: List[Optional[dict]] = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        self.opened = []
        descs = [[] for _ in range(self.ROLES)]
        self.idx_dev = []
        self.max_count = 0
        lists = peer_pull_lists(plan, [e["send"] if e else {} for e in everyone], rank)
        for q, idx, a in lists:
            info = everyone[q]
            peer_bufs = [C.ipc_open(h) for h in info["bufs"]]
            peer_flag = C.ipc_open(info["flag"])
            self.opened += peer_bufs + [peer_flag]
            it = torch.as_tensor(idx, device="cuda")
            self.idx_dev.append(it)
            for r in range(self.ROLES):
                descs[r].append((peer_bufs[r], it.data_ptr(), idx.size, a, peer_flag))
            self.max_count = max(self.max_count, int(idx.size))
        self.npeers = len(descs[0])
        self.desc_dev = []
        for r in range(self.ROLES):
            arr = np.array(descs[r], dtype=_DESC) if descs[r] else np.zeros(1, dtype=_DESC)
            self.desc_dev.append(torch.as_tensor(arr.view(np.uint8), device="cuda"))
        self.epoch = 0

    def exchange(self, role: int) -> None:
        self.epoch += 1
        self.C.halo_publish(self.flag, self.epoch)
        if self.npeers:
            self.C.halo_pull(self.desc_dev[role].data_ptr(), self.npeers, self.max_count,
                             self.views[role], self.epoch, self.err)

    def fence(self) -> None:
        """Wait until every peer finished its pulls of the previous exchanges
        (collective): called before a product rewrites its role buffers."""
        self.epoch += 1
        self.C.halo_publish(self.flag, self.epoch)
        if self.npeers:
            self.C.halo_pull(self.desc_dev[0].data_ptr(), self.npeers, 0, None, self.epoch,
                             self.err)

    def check(self) -> None:
        """Raises if a pull timed out (flags never arrived)."""
        e = self.torch.empty(1, dtype=self.torch.int32, device="cuda")
        e.copy_(_device_view(self.torch, self.err, 1, self.torch.int32))
        if int(e.item()):
            raise RuntimeError("PeerHalo: an owner's epoch flag never arrived")

    def close(self) -> None:
        for p in self.opened:
            self.C.ipc_close(p)
        self.opened = []


def _device_view(torch, ptr: int, n: int, dtype=None):
    """A torch CUDA tensor over raw device memory (no copy, not owned)."""
    dtype = dtype or torch.float64
    typestr = {torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8"}[dtype]

    class _V:
        __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3, "strides": None, "stream": None}

    return torch.as_tensor(_V(), device="cuda")


class ShardedPoly:
    """pi(A) v on the owned row block of every rank (collective call).

    Halos travel over NCCL point-to-point (batch_isend_irecv) or, with
    peer=True on GPUs, over peer memory (PeerHalo: no collective per SpMV)."""

    def __init__(self, plan: HaloPlan, backend, dist, group=None, peer: bool = False):
        self.plan = plan
        self.b = backend
        self.dist = dist
        self.group = group
        self._send_idx = {q: idx for q, idx in plan.send.items()}
        self.peer = PeerHalo(plan, dist, group) if peer else None

    def exchange(self, x_ext) -> None:
        """Fill the halo part of x_ext from the owning ranks."""
        if self.peer is not None:
            role = next(r for r, v in enumerate(self.peer.views) if v.data_ptr() == x_ext.data_ptr())
            self.peer.exchange(role)
            return
        p, d = self.plan, self.dist
        ops, keep = [], []
        for q, idx in sorted(self._send_idx.items()):
            buf = self.b.gather(x_ext, idx)
            keep.append(buf)
            ops.append(d.P2POp(d.isend, buf, q, group=self.group))
        recvs = []
        for q, (a, z) in sorted(p.recv.items()):
            buf = self.b.empty(z - a)
            recvs.append((a, z, buf))
            ops.append(d.P2POp(d.irecv, buf, q, group=self.group))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        for a, z, buf in recvs:
            self.b.copy_(x_ext[a:z], buf)

    def apply(self, roots, v_local):
        """pi(A) v for the owned block v_local (backend vector of n_local)."""
        from . import _capi as C

        p = self.plan
        plan = C.factor_plan(roots)
        if self.peer is not None:
            self.peer.fence()
            cur, nxt, t1 = self.peer.views
        else:
            cur, nxt, t1 = self.b.zeros(p.n_ext), self.b.zeros(p.n_ext), self.b.zeros(p.n_ext)
        self.b.copy_(cur[p.owned], v_local)
        for pair, c0, c1 in plan:
            self.exchange(cur)
            if not pair:
                self.b.factor(cur, nxt, 1, c0)
            else:
                self.b.factor(cur, t1, 0)
                self.exchange(t1)
                self.b.factor(t1, nxt, 2, c0, c1, cur)
            cur, nxt = nxt, cur
        return cur[p.owned]


# ------------------------------------------- sharded box-grid pass (fused) --
# Box-grid stencils (configs 2, 3, 5) split into z-slabs, two polynomial
# factors per pass (one where the plan leaves a real root alone), the halo
# exchange inside the pass kernel: the producer
# warp of rank q's box-grid pass (kernels/spmv_grid2.cu, slab mode) copies the
# two planes below its slab straight from rank q-1's buffer and the two above
# from rank q+1's, over NVLink through CUDA IPC mappings, after an acquire
# wait on that neighbour's epoch flag.  No collective, no pull kernel and no
# x_ext staging per pass; each rank moves 16 n_local bytes per two factors
# plus 4 halo planes.
#
# Epochs: every rank publishes epoch e once its vector x_e is ready (after the
# copy of v with ppa_halo_publish, then from inside each pass: its last CTA,
# found by a ticket counter, fences system-wide and releases the flag), in the
# same order on every rank, so "neighbour flag >= e" means "x_e is complete and
# every pass before it, including its reads of my buffers, has finished".
# Pass k reads the neighbours' x_k (the pass waits for it); it overwrites my
# x_{k-1} buffer, which the neighbours read during their pass k-1, only in
# the planes they read after its own wait on their x_k, which they publish
# after finishing pass k-1.  A new product first waits for the neighbours'
# last publish of the previous one before it overwrites x_0.


def partition_planes(nz: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous plane blocks (sizes differing by at most one), each with
    >= 2 planes: a neighbour's two halo planes then belong to one rank."""
    if world < 1:
        raise ValueError("partition_planes: world must be >= 1")
    if nz < 2 * world:
        raise ValueError("partition_planes: every slab needs >= 2 planes")
    return partition_rows(nz, world)


GRID_TWO_REAL, GRID_PAIR, GRID_ONE_REAL = 0, 1, 2


def box_row_ranges(nx: int, ny: int, nz: int, world: int) -> List[Tuple[int, int]]:
    """The row blocks of ShardedGridPoly's z-slabs (for HaloPlan.build)."""
    D = nx * ny
    return [(z0 * D, z1 * D) for z0, z1 in partition_planes(nz, world)]


def grid_passes(plan) -> List[Tuple[int, float, float, float]]:
    """Passes (kind, a0, a1, b0) of a factor plan in apply_poly's order
    (src/gmres_poly.cpp:129-143): a conjugate pair is one pass (kind 1), two
    consecutive real roots one pass (kind 0), a real root followed by a pair
    or by nothing a one-level pass (kind 2) - the grouping of the single-GPU
    chain (gmres_poly.cpp apply_poly_csr)."""
    out, k = [], 0
    while k < len(plan):
        pair, c0, c1 = plan[k]
        if pair:
            out.append((GRID_PAIR, c0, c1, 0.0))
            k += 1
        elif k + 1 < len(plan) and not plan[k + 1][0]:
            out.append((GRID_TWO_REAL, c0, 0.0, plan[k + 1][1]))
            k += 2
        else:
            out.append((GRID_ONE_REAL, c0, 0.0, 0.0))
            k += 1
    return out


class ShardedGridPoly:
    """pi(A) v for an nx x ny x nz box stencil (ny = 1: 5-point 2-D) split
    into z-slabs, one per rank, with the halo exchange fused into the pass
    kernel (collective constructor; CUDA, one GPU per rank).

    `vals` are the nd diagonal values in increasing offset (nd = 7 in 3-D,
    5 in 2-D).  apply(roots, v_local) takes and returns the owned planes."""

    def __init__(self, nx: int, ny: int, nz: int, vals, dist, group=None):
        import torch

        from . import _capi as C

        self.C, self.torch, self.dist, self.group = C, torch, dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.nx, self.ny, self.nz = nx, ny, nz
        self.nd = 7 if ny > 1 else 5
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        if self.vals.size != self.nd:
            raise ValueError(f"ShardedGridPoly: {self.nd} diagonal values expected")
        self.ranges = partition_planes(nz, self.world)
        self.z0, self.z1 = self.ranges[self.rank]
        self.D = nx * ny
        self.n_local = (self.z1 - self.z0) * self.D
        self.bufs = [C.dev_alloc(8 * self.n_local) for _ in range(2)]
        self.flag = C.dev_alloc(64)
        self.err = C.dev_alloc(16)
        self.views = [_device_view(torch, b, self.n_local) for b in self.bufs]
        mine = {"bufs": [C.ipc_get_handle(b) for b in self.bufs],
                "flag": C.ipc_get_handle(self.flag)}
        everyone: List[Optional[dict]] = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.opened = []
        self.nb = {}
        for side, q in (("left", self.rank - 1), ("right", self.rank + 1)):
            if 0 <= q < self.world:
                bufs = [C.ipc_open(h) for h in everyone[q]["bufs"]]
                flag = C.ipc_open(everyone[q]["flag"])
                self.opened += bufs + [flag]
                self.nb[side] = (bufs, flag, self.ranges[q][0])
        # the neighbours' flags as wait-only halo descriptors (the fence of a
        # new product)
        descs = [(0, 0, 0, 0, nb[1]) for nb in self.nb.values()]
        arr = np.array(descs, dtype=_DESC) if descs else np.zeros(1, dtype=_DESC)
        self.fence_desc = torch.as_tensor(arr.view(np.uint8), device="cuda")
        self.epoch = 0

    def _publish(self) -> None:
        self.epoch += 1
        self.C.halo_publish(self.flag, self.epoch)

    def apply(self, roots, v_local):
        C = self.C
        passes = grid_passes(C.factor_plan(roots))
        if self.nb:
            # the neighbours finished every pass of the previous product
            C.halo_pull(self.fence_desc.data_ptr(), len(self.nb), 0, None, self.epoch, self.err)
        self.views[0].copy_(v_local)
        self._publish()
        left, right = self.nb.get("left"), self.nb.get("right")
        # every pass in one C call (ppa_grid2_slab_chain): pass k reads role
        # k % 2, waits for epoch + k and its last CTA publishes epoch + k + 1
        role = C.grid2_slab_chain(self.nd, self.nx, self.ny, self.nz, self.vals, self.z0, self.z1,
                                  passes, self.bufs[0], self.bufs[1],
                                  xl=tuple(left[0]) if left else (0, 0),
                                  zl0=left[2] if left else 0, fl=left[1] if left else 0,
                                  xr=tuple(right[0]) if right else (0, 0),
                                  fr=right[1] if right else 0, epoch0=self.epoch, err=self.err,
                                  own=self.flag)
        self.epoch += len(passes)
        return self.views[role]

    def check(self) -> None:
        """Raises if a neighbour's flag never arrived during a pass."""
        e = self.torch.empty(1, dtype=self.torch.int32, device="cuda")
        e.copy_(_device_view(self.torch, self.err, 1, self.torch.int32))
        if int(e.item()):
            raise RuntimeError("ShardedGridPoly: a neighbour's epoch flag never arrived")

    def close(self) -> None:
        """Unmap the neighbours' buffers and free this rank's (collective: the
        neighbours must be done with them)."""
        for p in self.opened:
            self.C.ipc_close(p)
        self.opened = []
        self.torch.cuda.synchronize()
        for p in self.bufs + [self.flag, self.err]:
            self.C.dev_free(p)
        self.bufs, self.views = [], []


# ------------------------------------------------------------ sharded solve --
# Thick-restarted Arnoldi with the Krylov basis sharded by rows.  Every
# reduction (CGS2 coefficients, norms, Rayleigh quotients, residuals) is a
# rank-local sum followed by an all-reduce, so every rank holds the same
# Hessenberg matrix and the replicated host work (Ritz pairs, restart QR,
# Leja order) makes identical decisions on every rank.  The tall-skinny work
# (CGS2 sweeps, V*Q, Ritz vectors, dots) runs in the backend: the repo's
# kernels on CUDA, torch CPU ops in the gloo tests; the operator is the
# sharded pi(A)v above.  Same algorithm as the single-GPU solve
# (csrc/solver.cpp) with classical CGS2; the summation order
# of the cross-rank reductions differs, so results agree to roundoff.

_PAIR_TOL = 1e-10  # src/arnoldi.cpp:16


def _is_complex(z: complex) -> bool:
    return abs(z.imag) > _PAIR_TOL * max(1.0, abs(z))


def _arrange(values, vectors, ordering: str):
    """sort_pairs (src/arnoldi.cpp:40-95): stable by key, conjugate mates
    adjacent, +imag first."""
    key = (lambda z: abs(1.0 - z)) if ordering == "target_one" else abs
    idx = sorted(range(len(values)), key=lambda i: key(values[i]))
    used, out = set(), []
    for i in idx:
        if i in used:
            continue
        used.add(i)
        if not _is_complex(values[i]):
            out.append(i)
            continue
        mate = next((j for j in idx if j not in used and
                     abs(values[i] - np.conj(values[j])) <= _PAIR_TOL * max(1.0, abs(values[i]))),
                    None)
        if mate is None:
            out.append(i)
            continue
        used.add(mate)
        out += [i, mate] if values[i].imag >= 0.0 else [mate, i]
    return np.asarray(values)[out], np.asarray(vectors)[:, out]


class ShardedSolver:
    """solve() over row-sharded vectors (collective: every rank calls it).

    The Krylov basis is column-major on every rank (the backend's basis()),
    and each CGS2 step runs the single-GPU kernels' three sweeps with
    rank-local sums (CudaBackend: ppa_cgs_dot_local, ppa_cgs_update_dot_local,
    ppa_cgs_store_local, TMA-pipelined like the single-GPU step) and one
    all-reduce after each of the first two: c doubles, then c + 1 (the
    second-pass coefficients and ||w||^2; the subdiagonal follows by
    Pythagoras as in cgs2_step).  Ritz vectors and the thick-restart V*Q are
    ts_combine on the local rows; norms and Rayleigh quotients are local dots
    plus an all-reduce."""

    def __init__(self, plan: HaloPlan, backend, dist, group=None, peer: bool = False,
                 grid: Optional["ShardedGridPoly"] = None):
        """grid: a ShardedGridPoly over the same rows (plan built with
        box_row_ranges): the polynomial operator then runs as fused-halo
        box-grid passes; single SpMVs (polynomial build, residual checks)
        stay on the plan's exchange."""
        import torch

        self.torch = torch
        self.plan = plan
        self.b = backend
        self.dist = dist
        self.group = group
        self.sp = ShardedPoly(plan, backend, dist, group, peer=peer)
        self.grid = grid
        if grid is not None and (grid.z0 * grid.D, grid.z1 * grid.D) != tuple(
                plan.ranges[plan.rank]):
            raise ValueError("ShardedSolver: the grid's slab and the plan's rows differ "
                             "(build the plan with box_row_ranges)")
        self.mvps = 0

    # -- reductions ----------------------------------------------------------
    def _allreduce(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def _dot(self, x, y) -> float:
        return float(self._allreduce(self.b.dot(x, y)).item())

    def _norm(self, w) -> float:
        return float(np.sqrt(self._dot(w, w)))

    # -- operators -----------------------------------------------------------
    def _spmv(self, x):
        p = self.plan
        if self.sp.peer is not None:
            self.sp.peer.fence()
            xe = self.sp.peer.views[0]
        else:
            xe = self.b.zeros(p.n_ext)
        ye = self.b.zeros(p.n_ext)
        self.b.copy_(xe[p.owned], x)
        self.sp.exchange(xe)
        self.b.factor(xe, ye, 0)
        self.mvps += 1
        return ye[p.owned].clone()

    def _op(self, x):
        if self.roots is None:
            return self._spmv(x)
        self.mvps += len(self.roots)
        if self.grid is not None:
            return self.grid.apply(self.roots, x).clone()
        return self.sp.apply(self.roots, x).clone()

    # -- Arnoldi -------------------------------------------------------------
    def _init(self, v0, m):
        n = self.plan.n_local
        V, ld = self.b.basis(m + 1, n)
        V[0, :n] = v0 / self._norm(v0)
        return (V, ld), np.zeros((m + 1, m))

    def _extend(self, B, H, j0, m, op):
        """CGS2 steps j0..m-1; returns (cur_dim, breakdown)."""
        V, ld = B
        n = self.plan.n_local
        for j in range(j0, m):
            w = op(V[j, :n]).contiguous()
            c = j + 1
            h1 = self._allreduce(self.b.cgs_dot(V, ld, n, c, w))
            s2 = self._allreduce(self.b.cgs_update_dot(V, ld, n, c, w, h1))
            h1h, s2h = h1.cpu().numpy(), s2.cpu().numpy()
            h2h, nw = s2h[:c], s2h[c]
            d2 = nw - float(h2h @ h2h)
            hsub = float(np.sqrt(d2)) if d2 > 0.0 else 0.0
            col = h1h + h2h
            H[:c, j] = col
            if not np.isfinite(hsub) or hsub <= 1e-14 * np.sqrt(col @ col + hsub * hsub):
                H[j + 1, j] = 0.0
                return j + 1, True
            H[j + 1, j] = hsub
            hs = self.torch.full((1,), hsub, dtype=self.torch.float64, device=w.device)
            self.b.cgs_store(V, ld, n, c, w, s2[:c], hs)
        return m, False

    def _ritz(self, H, d, ordering):
        vals, vecs = np.linalg.eig(H[:d, :d])
        vecs = vecs / np.linalg.norm(vecs, axis=0)
        return _arrange(vals, vecs, ordering)

    def _check(self, B, d, vals, vecs, nev):
        """Rayleigh quotients and true residuals of the first nev pairs."""
        V, ld = B
        n = self.plan.n_local
        Y, ldy = self.b.basis(2, n)
        mus, res = [], []
        i = 0
        while i < min(nev, len(vals)):
            g = vecs[:, i]
            if not _is_complex(vals[i]):
                self.b.combine(V, ld, n, d, g.real.reshape(d, 1), 1, Y, ldy)
                yr = Y[0, :n] / self._norm(Y[0, :n])
                ay = self._spmv(yr)
                mu = self._dot(yr, ay)
                res.append(self._norm(ay - mu * yr))
                mus.append(complex(mu, 0.0))
                i += 1
                continue
            self.b.combine(V, ld, n, d, np.stack([g.real, g.imag], axis=1), 2, Y, ldy)
            nrm = np.sqrt(self._dot(Y[0, :n], Y[0, :n]) + self._dot(Y[1, :n], Y[1, :n]))
            yr, yi = Y[0, :n] / nrm, Y[1, :n] / nrm
            ar, ai = self._spmv(yr), self._spmv(yi)
            # mu = y^H A y for unit y = yr + i yi
            re = self._dot(yr, ar) + self._dot(yi, ai)
            im = self._dot(yr, ai) - self._dot(yi, ar)
            r = np.sqrt(self._norm(ar - re * yr + im * yi) ** 2 +
                        self._norm(ai - re * yi - im * yr) ** 2)
            mus += [complex(re, im), complex(re, -im)]
            res += [r, r]
            i += 2
        return mus[:nev], res[:nev]

    def _restart(self, B, H, m, vals, vecs, k):
        """thick_restart (src/arnoldi.cpp:267-334) on the sharded basis."""
        V, ld = B
        n = self.plan.n_local
        cols, j = [], 0
        while len(cols) < k and j < len(vals):
            if not _is_complex(vals[j]):
                cols.append(vecs[:, j].real)
                j += 1
            else:
                if len(cols) + 2 > k:
                    break
                cols += [vecs[:, j].real, vecs[:, j].imag]
                j += 2
        kk = len(cols)
        Q, _ = np.linalg.qr(np.stack(cols, axis=1))
        Hk = Q.T @ H[:m, :m] @ Q
        hrow = H[m, m - 1] * Q[m - 1]
        self.b.combine(V, ld, n, m, Q, kk, V, ld)  # V[:, :kk] = V[:, :m] Q, in place
        V[kk, :n] = V[m, :n]
        w = V[kk, :n]
        c = self._allreduce(self.b.cgs_dot(V, ld, n, kk, w))
        s = self._allreduce(self.b.cgs_update_dot(V, ld, n, kk, w, c))
        rn = float(np.sqrt(s[kk].item()))
        V[kk, :n] = w / rn
        Hk = Hk + np.outer(c.cpu().numpy(), hrow)
        H[:] = 0.0
        H[:kk, :kk] = Hk
        H[kk, :kk] = rn * hrow
        return kk

    # -- driver ----------------------------------------------------------------
    def solve(self, v0_poly, v0_arnoldi, v0_norm, m, k, nev, degree=0, rtol_multiplier=1e-8,
              max_cycles=100, stability=False):
        from . import _capi as C

        self.roots = None
        # norm estimate: five power steps
        x = v0_norm / self._norm(v0_norm)
        est = 0.0
        for it in range(5):
            y = self._spmv(x)
            est = self._norm(y)
            if est == 0.0:
                break
            x = y / est
        rtol = rtol_multiplier * est
        ordering = "smallest_magnitude"
        if degree > 0:
            Bb, Hb = self._init(v0_poly, degree)
            d, _ = self._extend(Bb, Hb, 0, degree, self._spmv)
            Hd = Hb[:d, :d].copy()
            hs = Hb[d, d - 1]
            if hs != 0.0:
                f = np.linalg.solve(Hd.T, np.eye(d)[:, d - 1])
                Hd[:, d - 1] += hs * hs * f
            self.roots = C.leja_order(np.linalg.eigvals(Hd))
            if stability and len(self.roots) >= 2:
                self.roots = C.add_stability_roots(self.roots, len(self.roots))
            ordering = "target_one"
        B, H = self._init(v0_arnoldi, m)
        cur, cycles, mus, res = 0, 0, [], []
        for cycles in range(1, max_cycles + 1):
            d, bd = self._extend(B, H, cur, m, self._op)
            vals, vecs = self._ritz(H, d, ordering)
            mus, res = self._check(B, d, vals, vecs, nev)
            if all(r <= rtol for r in res) or bd or cycles == max_cycles:
                break
            cur = self._restart(B, H, m, vals, vecs, k)
        return {"eigenvalues": np.asarray(mus), "residuals": np.asarray(res), "rtol": rtol,
                "converged": bool(len(res) == nev and all(r <= rtol for r in res)),
                "cycles": cycles, "mvps": self.mvps, "poly": self.roots}
