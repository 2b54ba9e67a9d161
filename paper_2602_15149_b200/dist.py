"""Multi-GPU slab decomposition with fixed halo lists.

TLSPH neighbours never change (total Lagrangian, kernel_geom.py:1-6), so the
partition and halo lists are computed once.  Each rank owns a slab of
particles along the longest axis, equal counts, ties broken by global index.
It keeps
  * its owned particles (positions [0, n_own) on the device, Morton order);
  * a halo block [n_own, n_all): every off-rank particle its owned rows
    reference, grouped by owner rank, within an owner by global index.
Owned rows keep the reference's summation order (ascending global partner
index), so every rank computes exactly what one GPU computes for the same
particles: results are bit-identical for any rank count.

Per force evaluation the step needs two exchanges (SURVEY.md 8(e) option 1):
the (u, s) records before pass A and the (P L, v) records before pass B.
``HaloExchange`` packs the send rows into one contiguous buffer and receives
straight into the halo rows (no unpack), as grouped point-to-point sends over
torch.distributed -- NCCL over NVLink on the B200 box, gloo in the CPU tests.
The dt maxima are combined with an all-reduce MAX on their (non-negative)
IEEE bit patterns, which is exact.

Everything here is host/plumbing logic usable with CPU tensors, so the
partition, the exchange plan and the exchange itself are tested with a gloo
world of 2 processes on CPU (tests/test_dist.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def longest_axis(X):
    ext = X.max(axis=0) - X.min(axis=0)
    return int(np.argmax(ext))


def slab_owner(X, nranks, axis=None):
    """owner[i] in [0, nranks): equal-count slabs along ``axis`` (default:
    the longest), ordered by (coordinate, global index)."""
    n = X.shape[0]
    axis = longest_axis(X) if axis is None else axis
    order = np.lexsort((np.arange(n), X[:, axis]))
    owner = np.empty(n, dtype=np.int32)
    bounds = [(n * r) // nranks for r in range(nranks + 1)]
    for r in range(nranks):
        owner[order[bounds[r]:bounds[r + 1]]] = r
    return owner, axis


def subset_for_rank(X, owner, rank, axis, reach):
    """Global ids (ascending) of the particles a rank must see: its slab
    extended by the interaction reach along the slab axis."""
    mine = np.flatnonzero(owner == rank)
    lo = X[mine, axis].min() - reach * (1.0 + 1e-6)
    hi = X[mine, axis].max() + reach * (1.0 + 1e-6)
    return np.flatnonzero((X[:, axis] >= lo) & (X[:, axis] <= hi))


@dataclass
class HaloPlan:
    """Exchange plan of one rank.

    halo_gid: global ids of the halo block, grouped by owner, ascending
    recv_off/recv_cnt: per peer rank, its slice of the halo block
    send_rows/send_cnt: per peer rank, the local OWNED positions to send, in
    the order the peer stores them."""
    rank: int
    nranks: int
    n_own: int
    halo_gid: np.ndarray
    recv_off: np.ndarray
    recv_cnt: np.ndarray
    send_rows: list
    send_cnt: np.ndarray

    @property
    def n_halo(self):
        return int(self.halo_gid.shape[0])


def _comm_device(group=None):
    """Tensors for collectives live on the GPU for NCCL, on the CPU for gloo."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def halo_order(needed_gid, owner):
    """Exchange order of a rank's halo block: by owner rank, then global id."""
    needed_gid = np.unique(np.asarray(needed_gid, dtype=np.int64))
    own_of = owner[needed_gid]
    return needed_gid[np.lexsort((needed_gid, own_of))]


def build_halo_plan(owned_gid, own_pos, needed_gid, owner, group=None):
    """Collective over the process group.

    owned_gid: global ids this rank owns; own_pos: their local positions
    (device order); needed_gid: global ids of off-rank particles referenced
    by owned rows.  Requests travel with all_to_all (variable sizes)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    nranks = dist.get_world_size(group)
    cdev = _comm_device(group)
    halo_gid = halo_order(needed_gid, owner)
    halo_owner = owner[halo_gid]
    recv_cnt = np.bincount(halo_owner, minlength=nranks).astype(np.int64)
    recv_off = np.concatenate([[0], np.cumsum(recv_cnt)[:-1]])
    # exchange request sizes, then the requested ids
    cnt_t = torch.tensor(recv_cnt, dtype=torch.int64, device=cdev)
    got_cnt = torch.empty_like(cnt_t)
    dist.all_to_all_single(got_cnt, cnt_t, group=group)
    send_cnt = got_cnt.cpu().numpy().astype(np.int64)
    req = torch.from_numpy(halo_gid.astype(np.int64)).to(cdev)
    got = torch.empty(int(send_cnt.sum()), dtype=torch.int64, device=cdev)
    dist.all_to_all_single(got, req, output_split_sizes=send_cnt.tolist(),
                           input_split_sizes=recv_cnt.tolist(), group=group)
    got = got.cpu().numpy()
    pos_of = dict(zip(np.asarray(owned_gid).tolist(), np.asarray(own_pos).tolist()))
    send_rows = []
    o = 0
    for q in range(nranks):
        ids = got[o:o + send_cnt[q]]
        send_rows.append(np.array([pos_of[int(g)] for g in ids], dtype=np.int64))
        o += send_cnt[q]
    return HaloPlan(rank=rank, nranks=nranks, n_own=len(owned_gid), halo_gid=halo_gid,
                    recv_off=recv_off, recv_cnt=recv_cnt, send_rows=send_rows,
                    send_cnt=send_cnt)


class HaloExchange:
    """Fills the halo rows [n_own, n_all) of a (n_all, width) tensor from the
    owners, with grouped isend/irecv.  Works for CPU (gloo) and CUDA (NCCL)
    tensors alike."""

    def __init__(self, plan: HaloPlan, device, group=None):
        import torch
        import torch.distributed as dist
        self.plan = plan
        self.group = group
        self.idx = [torch.from_numpy(r).to(device) if len(r) else None for r in plan.send_rows]
        # gloo moves CPU tensors only: a CUDA buffer is staged through the host
        # (used to run the multi-rank device path on one GPU in tests)
        self.stage = (dist.get_backend(group) == "gloo"
                      and torch.device(device).type == "cuda")

    def exchange(self, buf):
        """buf: tensor whose first dimension is n_all (owned then halo)."""
        if self.stage:
            host = buf.cpu()
            self._exchange(host, cpu_idx=True)
            buf[self.plan.n_own:].copy_(host[self.plan.n_own:])
            return buf
        return self._exchange(buf)

    def _exchange(self, buf, cpu_idx=False):
        import torch.distributed as dist
        p = self.plan
        ops = []
        sends = []
        for q in range(p.nranks):
            if q == p.rank:
                continue
            if p.send_cnt[q]:
                idx = self.idx[q].cpu() if cpu_idx else self.idx[q]
                pk = buf.index_select(0, idx)
                sends.append(pk)
                ops.append(dist.P2POp(dist.isend, pk, q, group=self.group))
            if p.recv_cnt[q]:
                a = p.n_own + int(p.recv_off[q])
                view = buf[a:a + int(p.recv_cnt[q])]
                ops.append(dist.P2POp(dist.irecv, view, q, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        del sends
        return buf


def allreduce(t, op="max", group=None):
    """In-place all-reduce of a (device) tensor; staged through the host for
    gloo.  MAX on the int64 bit patterns of non-negative doubles is the exact
    global max of the dt maxima."""
    import torch.distributed as dist
    rop = {"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op]
    if dist.get_backend(group) == "gloo" and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=rop, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=rop, group=group)
    return t


class PlaneOwner:
    """owner[g] for the global ids g of an x-major box lattice cut into slabs
    of whole planes: plane = g // plane_size, owner = the slab holding it."""

    def __init__(self, bounds, plane_size):
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.plane_size = int(plane_size)

    def __getitem__(self, g):
        plane = np.asarray(g, dtype=np.int64) // self.plane_size
        return (np.searchsorted(self.bounds, plane, side="right") - 1).astype(np.int32)


@dataclass
class LatticeSlab:
    """A rank's part of a box-lattice body built without the rest of it
    (cases.make_case(slab=...)): the planes [lo, hi) it holds on the host --
    its own slab [bounds[rank], bounds[rank + 1]) plus the interaction reach --
    and their global ids (x-major: g = plane * plane_size + in-plane index)."""
    rank: int
    nranks: int
    bounds: np.ndarray
    plane_size: int
    lo: int
    hi: int
    n_global: int

    @property
    def gid(self):
        return np.arange(self.lo * self.plane_size, self.hi * self.plane_size, dtype=np.int64)

    @staticmethod
    def plane_bounds(nplanes, nranks):
        return np.array([(nplanes * r) // nranks for r in range(nranks + 1)], dtype=np.int64)


class BodyPartition:
    """One rank's share of one body: its slab, the halo region it reads,
    and (after ``complete``) the halo block in exchange order.

    ``sub``: global ids of the region (ascending); ``host_rows``: their rows
    in the host state arrays (the global ids when the host holds the whole
    body, 0..len(sub) for a slab-local build)."""

    def __init__(self, X, owner, rank, axis, reach):
        self._init(subset_for_rank(X, owner, rank, axis, reach), owner, rank, None)

    @classmethod
    def from_slab(cls, slab):
        """Partition of a slab-local body: owners by whole planes, the host
        arrays hold exactly the slab plus its reach."""
        self = cls.__new__(cls)
        owner = PlaneOwner(slab.bounds, slab.plane_size)
        sub = slab.gid
        self._init(sub, owner, slab.rank, np.arange(sub.shape[0], dtype=np.int64))
        return self

    def _init(self, sub, owner, rank, host_rows):
        self.rank = rank
        self.owner = owner
        self.sub = sub                                                # global ids
        self.host_rows = sub if host_rows is None else host_rows
        self.owned_mask = owner[self.sub] == rank
        self.owned_rows = np.flatnonzero(self.owned_mask)             # subset rows
        self.owned_gid = self.sub[self.owned_rows]
        self.halo_rows = None
        self.needed_gid = None

    def complete(self, dadj):
        """Halo = off-rank partners of the owned rows (from the device CSR
        built on the subset), ordered as HaloPlan expects."""
        import torch
        dev = dadj.indptr.device
        counts = dadj.indptr[1:] - dadj.indptr[:-1]
        row_of = torch.repeat_interleave(torch.arange(dadj.n, device=dev), counts)
        owned = torch.from_numpy(self.owned_mask).to(dev)
        cols = torch.unique(dadj.indices[owned[row_of]].long()).cpu().numpy()
        gid = self.sub[cols]
        off = self.owner[gid] != self.rank
        self.needed_gid = halo_order(gid[off], self.owner)
        self.halo_rows = np.searchsorted(self.sub, self.needed_gid).astype(np.int64)   # sub ascending


class PeerHalo:
    """Halo exchange through peer memory instead of messages.

    Each rank maps its slab neighbours' `us` and `rb` record arrays (CUDA IPC
    handles shared through the process group; over NVLink on an 8-GPU box)
    and the step kernels store every boundary particle's records straight
    into the neighbours' halo rows as they produce them: pass A the pass-B
    record, pass B the new (u, s).  The transfer rides on the compute -- no
    pack kernel, no send/recv.  Ordering comes from the per-step collectives
    the step already has or adds: a barrier all-reduce after pass A (the
    neighbours' records have landed before pass B reads them, and they are
    done reading their (u, s) halo before pass B overwrites it) and the dt
    all-reduce after pass B (the new (u, s) have landed before the next pass
    A; the neighbours are done with their pass-B records before the next
    pass A overwrites them).

    ``peer_slot`` (2, n_all) int32: for each owned particle, its row in the
    side-k neighbour's arrays (-1: not sent there).  Up to two neighbours per
    rank (slabs); None from ``build`` when the plan needs more."""

    def __init__(self, slot, peers, keep):
        self.slot = slot
        self.peers = peers          # [(us, rb)] per side: the neighbours' tensors (mapped)
        self._keep = keep

    @classmethod
    def build(cls, plan, us, rb, group=None):
        """Collective.  plan: this rank's HaloPlan; us, rb: its record arrays."""
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        me = plan.rank
        mine = {"n_own": plan.n_own, "recv_off": plan.recv_off.tolist(),
                "us": reduce_tensor(us), "rb": reduce_tensor(rb),
                "sides": [q for q in range(plan.nranks) if plan.send_cnt[q] > 0]}
        allinfo = [None] * plan.nranks
        dist.all_gather_object(allinfo, mine, group=group)
        send_to = mine["sides"]
        ok = len(send_to) <= 2 and all(len(a["sides"]) <= 2 for a in allinfo)
        if not ok:
            return None
        n_all = int(us.shape[0])
        slot = torch.full((2, n_all), -1, dtype=torch.int32)
        peers, keep = [], []
        for side, q in enumerate(send_to):
            info = allinfo[q]
            base = int(info["n_own"]) + int(info["recv_off"][me])
            rows = torch.from_numpy(np.asarray(plan.send_rows[q], dtype=np.int64))
            slot[side, rows] = torch.arange(base, base + rows.shape[0], dtype=torch.int32)
            fn, args = info["us"]
            pu = fn(*args)
            fn, args = info["rb"]
            pr = fn(*args)
            peers.append((pu, pr))
            keep.extend([pu, pr])
        return cls(slot.to(us.device).contiguous(), peers, keep)

    def fill(self, d):
        """Set the peer-store fields of a tl_body descriptor."""
        import ctypes as C
        d.peer_slot = C.c_void_p(self.slot.data_ptr())
        for k in range(2):
            if k < len(self.peers):
                d.peer_us[k] = C.c_void_p(self.peers[k][0].data_ptr())
                d.peer_rb[k] = C.c_void_p(self.peers[k][1].data_ptr())
            else:
                d.peer_us[k] = None
                d.peer_rb[k] = None
