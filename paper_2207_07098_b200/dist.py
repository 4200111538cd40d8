"""Element partition across GPUs: halo plans for dssum and deterministic reductions.

One process per GPU (torch.distributed, NCCL over NVLink on the GPU box; gloo on
CPU for tests).  The mesh is split into contiguous element ranges -- z-slabs on
the box meshes, whose elements are numbered x fastest (mesh.py:199-219).

dssum across ranks.  Every rank owns the global gather-scatter
numbering (bit-exact, built once on its own GPU) and derives, for each shared
gid with a local copy, the full list of copies in global ascending local-index
order.  A copy owned by another rank is read from a receive buffer filled with
the *raw* local values that rank sends (no partial sums), so each rank sums
exactly the reference sequence 0.0 + v_0 + v_1 + ... and the result is bitwise
independent of the number of GPUs.  Send/receive lists are sorted by global copy
index on both sides, so no index exchange is needed.

Reductions (C2, C3).  glsc3 partials are all-gathered and summed in rank order
by one tiny kernel (deterministic for a given GPU count); CFL uses MAX.
"""

import os
import sys
import time

import numpy as np
import torch

from . import _lib

#: seconds a failing rank keeps its process (and so its IPC-mapped mailboxes and
#: halo inboxes) alive after an uncaught exception -- well past the 5 s poll
#: timeout of the peer kernels (csrc/peer.cuh), so a peer that is, or soon starts,
#: spinning on this rank's flags times out and returns (every later peer call
#: then returns at once) instead of polling unmapped memory after this exit
ABORT_GRACE_S = float(os.environ.get("SEMFLOW_B200_ABORT_GRACE_S", "12"))


def _abort_grace_hook(prev, grace=None):
    def hook(tp, val, tb):
        prev(tp, val, tb)
        try:
            sys.stderr.flush()
            time.sleep(ABORT_GRACE_S if grace is None else grace)
        except BaseException:
            pass
    hook.semflow_grace = True
    return hook


def install_abort_grace():
    """On an uncaught exception, report it, then keep the process alive for
    ABORT_GRACE_S before it exits (installed once peer memory is mapped)."""
    if not getattr(sys.excepthook, "semflow_grace", False):
        sys.excepthook = _abort_grace_hook(sys.excepthook)


class Comm:
    """Process-group wrapper; world == 1 makes every collective a no-op."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.collectives = 0
        self.peer = None
        if (self.world > 1 and torch.cuda.is_available() and dist.get_backend(group) == "nccl"
                and os.environ.get("SEMFLOW_B200_PEER", "1") != "0"):
            self.peer = _PeerReducer(self)
            install_abort_grace()

    def close(self):
        if self.peer is not None:
            self.peer.close()
            self.peer = None

    @property
    def active(self):
        return self.world > 1

    def check(self):
        """Raise if a peer-memory collective (allreduce or halo) timed out."""
        if self.peer is not None:
            self.peer.check()

    def sum_(self, t):
        """In place: t <- sum over ranks of t (rank order; t is a small device vector)."""
        if self.world == 1:
            return t
        k = t.numel()
        self.collectives += 1
        if t.is_cuda and self.peer is not None and k <= _PeerReducer.KMAX and t.is_contiguous():
            self.peer.allreduce_(t)
            return t
        if t.is_cuda:
            buf = torch.empty(self.world * k, dtype=t.dtype, device=t.device)
            _lib.nvtx_push("C2 allreduce:all_gather")
            self.dist.all_gather_into_tensor(buf, t.contiguous().view(-1), group=self.group)
            _lib.nvtx_pop()
            _lib.call("sf_rank_sum_f64", _lib.ptr(buf), self.world, k, _lib.ptr(t), _lib.stream_ptr(t.device))
        else:   # gloo (CPU tests): same rank-order summation
            parts = [torch.empty(k, dtype=t.dtype) for _ in range(self.world)]
            self.dist.all_gather(parts, t.contiguous().view(-1), group=self.group)
            acc = torch.zeros(k, dtype=t.dtype)
            for r in range(self.world):
                acc = acc + parts[r]
            t.view(-1).copy_(acc)
        return t

    def max_(self, t):
        if self.world == 1:
            return t
        _lib.nvtx_push("C3 max:all_reduce")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        _lib.nvtx_pop()
        self.collectives += 1
        return t

    def any(self, flag):
        """Host bool OR over ranks."""
        if self.world == 1:
            return bool(flag)
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        t = torch.tensor([1.0 if flag else 0.0], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item() > 0.0)

    def gather_elements(self, t, starts):
        """Concatenate every rank's element slice (leading axes kept, element axis
        = -4) into the global array on all ranks (checkpoints; not on the hot path)."""
        if self.world == 1:
            return t
        counts = [starts[r + 1] - starts[r] for r in range(self.world)]
        emax = max(counts)
        lead = t.shape[:-4]
        pad = torch.zeros(lead + (emax,) + t.shape[-3:], dtype=t.dtype, device=t.device)
        pad[..., :t.shape[-4], :, :, :] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad.contiguous(), group=self.group)
        return torch.cat([p[..., :c, :, :, :] for p, c in zip(parts, counts)], dim=-4)

    def gather_to_root(self, t, starts):
        """Rank 0: the global array (element axis -4) as host numpy; other ranks: None.
        Only rank 0 receives, and the result goes to the host at once, so a
        checkpoint holds one global field at a time on rank 0 alone."""
        if self.world == 1:
            return t.detach().cpu().numpy()
        counts = [starts[r + 1] - starts[r] for r in range(self.world)]
        emax = max(counts)
        lead = t.shape[:-4]
        pad = torch.zeros(lead + (emax,) + t.shape[-3:], dtype=t.dtype, device=t.device)
        pad[..., :t.shape[-4], :, :, :] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(pad, parts, dst=self.dist.get_global_rank(self.group, 0) if self.group else 0,
                         group=self.group)
        if self.rank != 0:
            return None
        host = [p[..., :c, :, :, :].cpu().numpy() for p, c in zip(parts, counts)]
        del parts
        return np.concatenate(host, axis=-4)

    def exchange(self, sends, recvs):
        """Post all sends/receives (dict peer -> tensor) and wait (stream-ordered on CUDA)."""
        if self.world == 1 or (not sends and not recvs):
            return
        P2POp = self.dist.P2POp
        ops = []
        for q in sorted(set(sends) | set(recvs)):
            if q in recvs and recvs[q].numel():
                ops.append(P2POp(self.dist.irecv, recvs[q], q, self.group))
            if q in sends and sends[q].numel():
                ops.append(P2POp(self.dist.isend, sends[q], q, self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        self.collectives += 1


class _PeerReducer:
    """NVLink mailboxes for the glsc3 allreduce (csrc/peer.cu).

    Each rank cudaMallocs a mailbox, exports it with CUDA IPC, and maps every
    peer's; a reduction is then one 32-thread kernel (P2P stores + acquire polls)
    instead of an NCCL all-gather plus a combine kernel.  Same rank-order sum.
    """

    KMAX = 4

    def __init__(self, comm):
        import ctypes

        lib = _lib.load()
        self.comm = comm
        self.dev = torch.device("cuda", torch.cuda.current_device())
        nbytes = 8 * lib.sf_peer_mailbox_doubles(comm.world)
        own = ctypes.c_void_p()
        _lib.call("sf_dev_alloc_zero", nbytes, ctypes.byref(own))
        self.own = own.value
        hb = lib.sf_ipc_handle_bytes()
        h = ctypes.create_string_buffer(hb)
        _lib.call("sf_ipc_get_handle", self.own, h)
        handles = [None] * comm.world
        comm.dist.all_gather_object(handles, h.raw, group=comm.group)
        self.opened = []
        ptrs = []
        for r, hr in enumerate(handles):
            if r == comm.rank:
                ptrs.append(self.own)
                continue
            p = ctypes.c_void_p()
            _lib.call("sf_ipc_open_handle", ctypes.create_string_buffer(hr, hb), ctypes.byref(p))
            self.opened.append(p.value)
            ptrs.append(p.value)
        self.boxes = (ctypes.c_void_p * comm.world)(*ptrs)
        self.error = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # reductions executed so far, advanced on the device by each call that
        # really exchanges (a gated pass that skips leaves it alone): the call
        # number and the mailbox bank are never kernel arguments, so every call
        # has the same arguments and graph-captured reductions stay in step
        self.seq = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.calls = 0          # host count of enqueued reductions (statistics only)
        torch.cuda.synchronize()
        comm.dist.barrier(group=comm.group)

    def fused_args(self):
        """(boxes, world, rank, seq, error) for one fused kernel+collective call."""
        self.calls += 1
        return (self.boxes, self.comm.world, self.comm.rank, _lib.ptr(self.seq), _lib.ptr(self.error))

    def allreduce_(self, t):
        self.calls += 1
        _lib.call("sf_peer_allreduce_f64", self.boxes, self.comm.world, self.comm.rank, _lib.ptr(self.seq),
                  _lib.ptr(self.error), _lib.ptr(t), t.numel(), _lib.ptr(t), _lib.stream_ptr(t.device))

    def failed(self):
        return bool(int(self.error.item()))

    def check(self):
        if self.failed():
            raise RuntimeError("peer allreduce / halo exchange timed out (a rank did not arrive within 5 s)")

    def close(self):
        for p in self.opened:
            _lib.call("sf_ipc_close_handle", p)
        self.opened = []
        if self.own:
            torch.cuda.synchronize()
            _lib.call("sf_dev_free", self.own)
            self.own = None


class _RawPtr:
    """Duck-typed device pointer (``data_ptr()``) for buffers not owned by torch."""

    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


class BankedRecv(_RawPtr):
    """The receive buffer of an NVLink halo exchange: bank 0 of the inbox, plus the
    device call counter and bank stride from which the dssum picks the bank of
    the current exchange (sf_dssum_blk_f64 recv_seq / recv_bank)."""

    def __init__(self, p, seq_ptr, bank):
        super().__init__(p)
        self.seq_ptr = seq_ptr
        self.bank = bank


class HaloIPC:
    """IPC inboxes for the NVLink halo exchange of one HaloPlan (csrc/halo.cu).

    Collective at construction (every rank of ``comm`` builds its own for the same
    space).  ``exchange(v)`` enqueues the put and the wait kernels on the current
    stream and returns this rank's receive buffer for the call (an inbox bank)."""

    HEADER = 32

    def __init__(self, comm, plan):
        import ctypes

        lib = _lib.load()
        self.comm = comm
        self.plan = plan
        me = comm.rank
        self.n_recv = max(int(plan.n_recv_total), 1)
        nbytes = 8 * lib.sf_halo_inbox_doubles(self.n_recv)
        own = ctypes.c_void_p()
        _lib.call("sf_dev_alloc_zero", nbytes, ctypes.byref(own))
        self.own = own.value
        hb = lib.sf_ipc_handle_bytes()
        h = ctypes.create_string_buffer(hb)
        _lib.call("sf_ipc_get_handle", self.own, h)
        info = (h.raw, {int(q): int(o) for q, o in plan.recv_off.items()}, self.n_recv, list(plan.peers))
        allinfo = [None] * comm.world
        comm.dist.all_gather_object(allinfo, info, group=comm.group)
        peers = list(plan.peers)
        for q in peers:
            if me not in allinfo[q][3]:
                raise RuntimeError(f"halo plan is not symmetric: rank {me} -> {q}")
        self.opened = []
        dst, stride, flag = [], [], []
        for q in peers:
            p = ctypes.c_void_p()
            _lib.call("sf_ipc_open_handle", ctypes.create_string_buffer(allinfo[q][0], hb), ctypes.byref(p))
            self.opened.append(p.value)
            dst.append(p.value + 8 * (self.HEADER + allinfo[q][1][me]))
            stride.append(allinfo[q][2])
            flag.append(p.value + 8 * me)
        n = len(peers)
        self.n_peers = n
        self.peer_rank = (ctypes.c_int * max(n, 1))(*peers)
        seg = [plan.send_off[q] for q in peers] + [int(plan.send_all.numel())]
        self.seg = (ctypes.c_longlong * (n + 1))(*seg)
        self.dst = (ctypes.c_void_p * max(n, 1))(*dst)
        self.stride = (ctypes.c_longlong * max(n, 1))(*stride)
        self.flag = (ctypes.c_void_p * max(n, 1))(*flag)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        self.error = comm.peer.error if comm.peer is not None else torch.zeros(1, dtype=torch.int32, device=dev)
        # the exchange counter is header word SEQ of the own inbox (zeroed at
        # allocation, advanced by halo_put on the device); the receive buffer
        # handed to the dssum names both banks and that counter
        self.recv = BankedRecv(self.own + 8 * self.HEADER, self.own + 8 * self.SEQ, self.n_recv)
        self.calls = 0
        torch.cuda.synchronize()
        comm.dist.barrier(group=comm.group)

    SEQ = 16

    def put(self, v):
        """Enqueue the NVLink stores of this rank's interface copies (the call
        number advances on the device)."""
        if self.n_peers == 0:
            return
        self.calls += 1
        _lib.call("sf_halo_put_f64", _lib.ptr(v), _lib.ptr(self.plan.send_all), self.n_peers, self.peer_rank,
                  self.seg, self.dst, self.stride, self.flag, self.own, _lib.ptr(self.counter),
                  _lib.ptr(self.error), _lib.stream_ptr(v.device))

    def wait(self, device):
        """Enqueue the wait for the peers' copies of the last put; returns the
        receive buffer (both inbox banks + the device call counter)."""
        if self.n_peers == 0:
            return None
        _lib.call("sf_halo_wait", self.own, self.n_peers, self.peer_rank, _lib.ptr(self.error),
                  _lib.stream_ptr(device))
        self.comm.collectives += 1
        return self.recv

    def exchange(self, v):
        self.put(v)
        return self.wait(v.device)

    def check(self):
        if int(self.error.item()):
            raise RuntimeError("halo exchange timed out (a peer did not publish within 5 s)")

    def close(self):
        for p in self.opened:
            _lib.call("sf_ipc_close_handle", p)
        self.opened = []
        if self.own:
            torch.cuda.synchronize()
            _lib.call("sf_dev_free", self.own)
            self.own = None


_SINGLE = None


def single():
    global _SINGLE
    if _SINGLE is None:
        _SINGLE = Comm.__new__(Comm)
        _SINGLE.dist = None
        _SINGLE.group = None
        _SINGLE.rank, _SINGLE.world, _SINGLE.collectives = 0, 1, 0
        _SINGLE.peer = None
    return _SINGLE


def element_ranges(E, world):
    """Contiguous balanced element ranges: starts[r] .. starts[r+1]."""
    return [E * r // world for r in range(world + 1)]


class HaloPlan:
    """Shared-gid maps of one rank with remote copies routed through a receive buffer.

    sh_off / sh_perm: int32, over the shared gids with >= 1 local copy, ordered
    by their lowest local copy.  sh_perm entries < P_loc are local indices; entries
    >= P_loc index the concatenated receive buffer.  send_idx[q] / n_recv[q]: the
    local indices sent to peer q and the number of values received from it, both
    in global copy-index order.
    """

    def __init__(self, sh_off, sh_perm, n_shared, P_loc, send_idx, n_recv):
        self.sh_off = sh_off
        self.sh_perm = sh_perm
        self.n_shared = n_shared
        self.P_loc = P_loc
        self.send_idx = send_idx        # dict q -> int32 tensor
        self.n_recv = n_recv            # dict q -> int
        self.peers = sorted(set(send_idx) | set(n_recv))
        off = 0
        self.recv_off = {}
        for q in self.peers:
            self.recv_off[q] = off
            off += n_recv.get(q, 0)
        self.n_recv_total = off
        self.send_all = (torch.cat([send_idx[q] for q in self.peers if q in send_idx])
                         if send_idx else torch.zeros(0, dtype=torch.int32, device=sh_perm.device))
        so = 0
        self.send_off = {}
        for q in self.peers:
            self.send_off[q] = so
            so += int(send_idx[q].numel()) if q in send_idx else 0


def build_halo_plan(gid, perm, offsets, starts, rank, nnn):
    """Plan for `rank` from the global numbering (pure torch; CPU or CUDA tensors)."""
    dev = gid.device
    e0, e1 = starts[rank], starts[rank + 1]
    g0 = e0 * nnn
    P_loc = (e1 - e0) * nnn
    counts = offsets[1:] - offsets[:-1]
    gid_loc = gid[g0:g0 + P_loc]
    rel = torch.unique(gid_loc[counts[gid_loc] > 1])          # shared gids with a local copy
    n_shared = int(rel.numel())
    cnt = counts[rel]
    start = torch.repeat_interleave(offsets[rel], cnt)
    seg = torch.zeros(n_shared + 1, dtype=torch.int64, device=dev)
    if n_shared:
        seg[1:] = torch.cumsum(cnt, 0)
    within = torch.arange(int(seg[-1]), device=dev) - torch.repeat_interleave(seg[:-1], cnt)
    copies = perm[start + within]                             # global copy indices, gid-grouped, ascending
    owner_elem = copies // nnn
    st = torch.tensor(starts, dtype=torch.int64, device=dev)
    owner = torch.searchsorted(st, owner_elem, right=True) - 1
    entry = torch.empty_like(copies)
    local = owner == rank
    entry[local] = copies[local] - g0
    send_idx, n_recv = {}, {}
    gid_of_copy = torch.repeat_interleave(rel, cnt)
    remote_peers = torch.unique(owner[~local]).tolist()
    recv_base = P_loc
    for q in sorted(remote_peers):
        # values received from q: q's copies of gids we share with q, by global copy index
        from_q = torch.nonzero(owner == q).view(-1)           # already in (gid, copy) order
        order = torch.argsort(copies[from_q])
        pos = torch.empty_like(order)
        pos[order] = torch.arange(order.numel(), device=dev)
        entry[from_q] = recv_base + pos
        n_recv[q] = int(from_q.numel())
        recv_base += n_recv[q]
        # values sent to q: my copies of the gids that have a copy on q
        gids_q = torch.unique(gid_of_copy[from_q])
        mine = local & torch.isin(gid_of_copy, gids_q)
        mc = copies[mine]
        send_idx[q] = (torch.sort(mc).values - g0).to(torch.int32)
    # order shared gids by lowest local copy (locality of the dssum kernel)
    big = torch.iinfo(torch.int64).max
    key = torch.where(local, copies, torch.full_like(copies, big))
    seg_id = torch.repeat_interleave(torch.arange(n_shared, device=dev), cnt)
    first = torch.full((n_shared,), big, dtype=torch.int64, device=dev)
    if n_shared:
        first.scatter_reduce_(0, seg_id, key, reduce="amin")
    gorder = torch.argsort(first)
    cnt_o = cnt[gorder]
    sh_off = torch.zeros(n_shared + 1, dtype=torch.int64, device=dev)
    if n_shared:
        sh_off[1:] = torch.cumsum(cnt_o, 0)
    src = torch.repeat_interleave(seg[:-1][gorder], cnt_o) + (
        torch.arange(int(sh_off[-1]), device=dev) - torch.repeat_interleave(sh_off[:-1], cnt_o))
    sh_perm = entry[src]
    if P_loc + recv_base >= 2 ** 31:
        raise ValueError("local + halo points exceed int32 indexing")
    return HaloPlan(sh_off.to(torch.int32), sh_perm.to(torch.int32), n_shared, P_loc, send_idx, n_recv)


def dssum_reference_cpu(values_by_rank, plans, mode=0):
    """Emulate the dssum kernel + exchange on the CPU for every rank (test helper).

    values_by_rank[r]: 1-D float64 numpy array of rank r's local values.  Returns
    the per-rank outputs.  Follows sf_dssum_f64 exactly: raw copies exchanged,
    sequential sum over the gid's copies in global order, write-back of local copies.
    """
    outs = []
    for r, plan in enumerate(plans):
        v = values_by_rank[r].copy()
        recv = np.zeros(plan.n_recv_total)
        for q in plan.peers:
            # what q sends to r
            pq = plans[q]
            vals = values_by_rank[q][pq.send_idx[r].cpu().numpy()] if r in pq.send_idx else np.zeros(0)
            o = plan.recv_off[q]
            recv[o:o + plan.n_recv.get(q, 0)] = vals
        off = plan.sh_off.cpu().numpy()
        perm = plan.sh_perm.cpu().numpy()
        src = np.concatenate([values_by_rank[r], recv])
        for g in range(plan.n_shared):
            acc = 0.0
            for o in range(off[g], off[g + 1]):
                acc = acc + src[perm[o]]
            if mode == 1:
                acc = acc * (1.0 / (off[g + 1] - off[g]))
            for o in range(off[g], off[g + 1]):
                if perm[o] < plan.P_loc:
                    v[perm[o]] = acc
        outs.append(v)
    return outs


def init_from_env():
    """torch.distributed init for a torchrun launch (NCCL on CUDA), else single."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return single()
    import torch.distributed as dist

    if not dist.is_initialized():
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return Comm()
