"""Partitioned construction of the gather-scatter numbering (one rank's share).

The reference numbers the global nodes of the whole mesh at once
(space.py:265-314): coincident GLL points form one node, and nodes are ranked
by the coordinates of their representative (lowest local copy), x primary.
With one process per GPU the global build needs the coordinates and the
int64 maps of ALL points on every rank (a 2M-element lx=8 mesh: 25 GB of
coordinates and 17 GB of maps per GPU).  Here every rank works on its own
contiguous element range only:

1. topological keys of its boundary points (space.topo_keys) -- equal keys are
   coincident points on a conforming mesh;
2. a point can be shared with rank q only if every vertex defining its key is
   used by an element of q (vertex -> rank bitmasks from the connectivity,
   which every rank holds): those points' (key, global index) are sent to q,
   and every rank merges its own keys with what it received;
3. the halo plan of the multi-GPU dssum (dist.HaloPlan) follows from the merged
   groups exactly as dist.build_halo_plan derives it from the global maps;
4. the reference's global ids: each node is owned by the rank of its lowest
   copy; owners rank their nodes by (x, y, z, representative) with a
   distributed sample sort (splitters from all_gathered samples, one
   all-to-all of keys, a local sort, prefix offsets, ranks sent back), and the
   ids reach the other copies through one plan exchange.

Everything is torch (CUDA on the GPU box, CPU + gloo in the tests), O(P / N)
memory per rank plus the interface, and bitwise equal to the global build.
"""

import torch

from . import dist as _dist
from .errors import ConfigError

_M30 = (1 << 30) - 1


def vertex_rank_masks(elements, starts, nv):
    """(nv,) int64 bitmask of the ranks whose elements use each vertex."""
    m = torch.zeros(nv, dtype=torch.int64, device=elements.device)
    for q in range(len(starts) - 1):
        v = torch.unique(elements[starts[q]:starts[q + 1]].reshape(-1))
        m[v] |= 1 << q
    return m


def point_peer_masks(k1, k2, vmask):
    """Ranks that may hold a copy of each keyed point: AND of the masks of the
    vertices in its key (vertex: 1 id, edge: 2 ids, face: 3 of its 4 ids)."""
    kind = k1 >> 60
    a = (k1 >> 30) & _M30
    b = k1 & _M30
    c = (k2 >> 16).clamp(max=vmask.numel() - 1)
    m = vmask[a]
    m = torch.where(kind >= 1, m & vmask[b], m)
    return torch.where(kind == 2, m & vmask[c], m)


def all_gather_cat(comm, t):
    """Concatenation of every rank's equal-shaped tensor t (rank order)."""
    if comm.dist.get_backend(comm.group) == "nccl":
        out = torch.empty((comm.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        comm.dist.all_gather_into_tensor(out, t.contiguous(), group=comm.group)
        return out
    parts = [torch.empty_like(t) for _ in range(comm.world)]
    comm.dist.all_gather(parts, t.contiguous(), group=comm.group)
    return torch.cat(parts)


def alltoallv(comm, sends, width, dtype, dev):
    """Exchange variable-length (rows, width) tensors: sends[q] -> received[q].
    Sizes travel first (all_gather), then one batched send/recv round."""
    W, r = comm.world, comm.rank
    sz = torch.zeros(W, dtype=torch.int64, device=dev)
    for q, t in sends.items():
        sz[q] = t.shape[0]
    allsz = all_gather_cat(comm, sz).view(W, W).cpu()
    recvs = {q: torch.empty((int(allsz[q, r]), width), dtype=dtype, device=dev)
             for q in range(W) if q != r and int(allsz[q, r]) > 0}
    comm.exchange({q: t.contiguous() for q, t in sends.items() if t.shape[0]}, recvs)
    return recvs


def _lexsort(cols):
    """Permutation sorting rows by cols[0], then cols[1], ... (stable sorts)."""
    o = torch.sort(cols[-1], stable=True).indices
    for c in reversed(cols[:-1]):
        o = o[torch.sort(c[o], stable=True).indices]
    return o


def _ordered(x):
    """float64 -> int64 with the same order (+0.0 and -0.0 folded)."""
    b = (x + 0.0).contiguous().view(torch.int64)
    return torch.where(b < 0, torch.bitwise_not(b) | torch.iinfo(torch.int64).min, b)


def _tuple_ge(keys, s):
    """Rows of keys (n, 4) lexicographically >= the tuple s (4,)."""
    ge = keys[:, 3] >= s[3]
    for c in (2, 1, 0):
        ge = (keys[:, c] > s[c]) | ((keys[:, c] == s[c]) & ge)
    return ge


def global_ranks(comm, keys, oversample=64):
    """Global position of each local row of keys (n, 4) int64 in the
    lexicographic order of all ranks' rows (rows are distinct)."""
    W, r = comm.world, comm.rank
    dev = keys.device
    n = keys.shape[0]
    o = _lexsort([keys[:, c] for c in range(4)])
    sk = keys[o]
    # splitters from evenly spaced samples of every rank
    k = oversample * W
    pick = (torch.arange(k, device=dev, dtype=torch.int64) * max(n - 1, 0)) // max(k - 1, 1)
    smp = torch.full((k, 4), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    if n:
        smp[:] = sk[pick]
    cnt = torch.tensor([n], dtype=torch.int64, device=dev)
    alls = all_gather_cat(comm, smp)
    allc = all_gather_cat(comm, cnt)
    valid = torch.cat([torch.arange(k, device=dev) < min(int(c), 1) * k for c in allc.cpu()])
    alls = alls[valid]
    so = _lexsort([alls[:, c] for c in range(4)])
    alls = alls[so]
    m = alls.shape[0]
    split = [alls[(m * j) // W] for j in range(1, W)] if m else []
    bucket = torch.zeros(n, dtype=torch.int64, device=dev)
    for s in split:
        bucket += _tuple_ge(sk, s).to(torch.int64)
    # keys + (origin position) to their bucket's rank
    payload = torch.cat([sk, o.view(-1, 1)], dim=1)
    sends = {q: payload[bucket == q] for q in range(W) if q != r}
    recvs = alltoallv(comm, sends, 5, torch.int64, dev)
    mine = [payload[bucket == r]] + [recvs[q] for q in sorted(recvs)]
    srcs = [torch.full((mine[0].shape[0],), r, dtype=torch.int64, device=dev)] + \
           [torch.full((recvs[q].shape[0],), q, dtype=torch.int64, device=dev) for q in sorted(recvs)]
    mine = torch.cat(mine)
    src = torch.cat(srcs)
    lo = _lexsort([mine[:, c] for c in range(4)])
    # bucket sizes -> global offset of this rank's bucket
    bsz = torch.tensor([mine.shape[0]], dtype=torch.int64, device=dev)
    allb = all_gather_cat(comm, bsz)
    base = int(allb[:r].sum())
    rank_of = torch.empty(mine.shape[0], dtype=torch.int64, device=dev)
    rank_of[lo] = base + torch.arange(mine.shape[0], device=dev)
    # ranks back to the origin rows
    out = torch.empty(n, dtype=torch.int64, device=dev)
    me = src == r
    out[mine[me, 4]] = rank_of[me]
    back = {q: torch.stack([mine[src == q, 4], rank_of[src == q]], dim=1) for q in range(W) if q != r}
    got = alltoallv(comm, back, 2, torch.int64, dev)
    for t in got.values():
        out[t[:, 0]] = t[:, 1]
    return out


def plan_sum(comm, plan, vals):
    """Sum of the copies of every shared node (int64, any order: exact), written
    to the local copies -- the dssum over a plan in torch (setup only)."""
    dev = vals.device
    P = plan.P_loc
    sends = {q: vals[plan.send_idx[q].long()].view(-1, 1) for q in plan.send_idx}
    recvs = alltoallv(comm, sends, 1, vals.dtype, dev)
    rb = torch.zeros(max(plan.n_recv_total, 0), dtype=vals.dtype, device=dev)
    for q, t in recvs.items():
        rb[plan.recv_off[q]:plan.recv_off[q] + t.shape[0]] = t.view(-1)
    src = torch.cat([vals, rb])
    off = plan.sh_off.long()
    cnt = off[1:] - off[:-1]
    seg = torch.repeat_interleave(torch.arange(plan.n_shared, device=dev), cnt)
    tot = torch.zeros(plan.n_shared, dtype=vals.dtype, device=dev).index_add_(0, seg, src[plan.sh_perm.long()])
    out = vals.clone()
    loc = plan.sh_perm.long() < P
    out[plan.sh_perm.long()[loc]] = tot[seg[loc]]
    return out


def partitioned_numbering(elements, coords_loc, n, comm, starts, nv):
    """This rank's share of the gather-scatter numbering without any global
    per-point array.  elements: (E, 8) global connectivity (device);
    coords_loc: (3, El, n, n, n) of this rank's elements.  Returns
    (gid (P_loc,) int64 in the reference's global numbering, HaloPlan,
    mult8 (P_loc,) uint8, n_gid)."""
    dev = coords_loc.device
    r, W = comm.rank, comm.world
    e0, e1 = starts[r], starts[r + 1]
    El = e1 - e0
    nnn = n ** 3
    P = El * nnn
    g0 = e0 * nnn
    k1, k2, gpt = topo_keys_local(elements[e0:e1], n)
    vmask = vertex_rank_masks(elements, starts, nv)
    pm = point_peer_masks(k1, k2, vmask) & ~(1 << r)
    gidx = gpt + g0
    trip = torch.stack([k1, k2, gidx], dim=1)
    sends = {}
    for q in range(W):
        if q != r:
            sel = ((pm >> q) & 1) == 1
            sends[q] = trip[sel]
    recvs = alltoallv(comm, sends, 3, torch.int64, dev)
    del pm, vmask
    # merge own and received keys; groups = runs of equal (k1, k2), copies by global index
    parts = [trip] + [recvs[q] for q in sorted(recvs)]
    owner = torch.cat([torch.full((trip.shape[0],), r, dtype=torch.int64, device=dev)] +
                      [torch.full((recvs[q].shape[0],), q, dtype=torch.int64, device=dev) for q in sorted(recvs)])
    allk = torch.cat(parts)
    del parts, recvs, trip
    o = _lexsort([allk[:, 0], allk[:, 1], allk[:, 2]])
    sk, so = allk[o], owner[o]
    del allk, owner
    newg = torch.ones(sk.shape[0], dtype=torch.bool, device=dev)
    if sk.shape[0] > 1:
        newg[1:] = (sk[1:, 0] != sk[:-1, 0]) | (sk[1:, 1] != sk[:-1, 1])
    grp = torch.cumsum(newg.to(torch.int64), 0) - 1
    ng = int(grp[-1]) + 1 if grp.numel() else 0
    local = so == r
    has_local = torch.zeros(ng, dtype=torch.bool, device=dev)
    has_local[grp[local]] = True
    keep = has_local[grp]
    sk, so, grp, local = sk[keep], so[keep], grp[keep], local[keep]
    # renumber kept groups densely
    _, grp = torch.unique_consecutive(grp, return_inverse=True)
    ng = int(grp[-1]) + 1 if grp.numel() else 0
    cnt = torch.bincount(grp, minlength=ng)
    if cnt.numel() and int(cnt.max()) > 255:
        raise ConfigError("a global id has more than 255 local copies")
    gstart = torch.zeros(ng + 1, dtype=torch.int64, device=dev)
    gstart[1:] = torch.cumsum(cnt, 0)
    copies = sk[:, 2]

    # multiplicity of every local point (interior points: 1)
    mult = torch.ones(P, dtype=torch.int64, device=dev)
    mult[copies[local] - g0] = cnt[grp[local]]

    # ---- halo plan (as dist.build_halo_plan from the global maps)
    shared = cnt > 1
    sel = shared[grp]
    c_copies, c_owner, c_grp, c_local = copies[sel], so[sel], grp[sel], local[sel]
    sg = torch.nonzero(shared).view(-1)                   # kept shared groups, key order
    remap = torch.full((ng,), -1, dtype=torch.int64, device=dev)
    remap[sg] = torch.arange(sg.numel(), device=dev)
    c_grp = remap[c_grp]
    n_shared = int(sg.numel())
    scnt = cnt[sg]
    entry = torch.empty_like(c_copies)
    entry[c_local] = c_copies[c_local] - g0
    send_idx, n_recv = {}, {}
    recv_base = P
    for q in sorted(torch.unique(c_owner[~c_local]).tolist()):
        from_q = torch.nonzero(c_owner == q).view(-1)
        ordq = torch.argsort(c_copies[from_q])
        pos = torch.empty_like(ordq)
        pos[ordq] = torch.arange(ordq.numel(), device=dev)
        entry[from_q] = recv_base + pos
        n_recv[q] = int(from_q.numel())
        recv_base += n_recv[q]
        gq = torch.zeros(n_shared, dtype=torch.bool, device=dev)
        gq[c_grp[from_q]] = True
        mine = c_local & gq[c_grp]
        send_idx[q] = (torch.sort(c_copies[mine]).values - g0).to(torch.int32)
    big = torch.iinfo(torch.int64).max
    keyl = torch.where(c_local, c_copies, torch.full_like(c_copies, big))
    first = torch.full((n_shared,), big, dtype=torch.int64, device=dev)
    if n_shared:
        first.scatter_reduce_(0, c_grp, keyl, reduce="amin")
    gorder = torch.argsort(first)
    cnt_o = scnt[gorder]
    sh_off = torch.zeros(n_shared + 1, dtype=torch.int64, device=dev)
    if n_shared:
        sh_off[1:] = torch.cumsum(cnt_o, 0)
    seg0 = torch.zeros(n_shared + 1, dtype=torch.int64, device=dev)
    if n_shared:
        seg0[1:] = torch.cumsum(scnt, 0)
    src = torch.repeat_interleave(seg0[:-1][gorder], cnt_o) + (
        torch.arange(int(sh_off[-1]), device=dev) - torch.repeat_interleave(sh_off[:-1], cnt_o))
    sh_perm = entry[src]
    if P + recv_base >= 2 ** 31:
        raise ConfigError("local + halo points exceed int32 indexing")
    plan = _dist.HaloPlan(sh_off.to(torch.int32), sh_perm.to(torch.int32), n_shared, P, send_idx, n_recv)

    # ---- global ids: owners rank their nodes by (x, y, z, representative)
    own_grp = local & (copies == sk[gstart[grp], 2])      # this rank holds the group's lowest copy
    rep_loc = copies[own_grp] - g0                        # local index of owned boundary nodes
    interior = torch.ones(P, dtype=torch.bool, device=dev)
    interior[gpt] = False
    rep_loc = torch.cat([rep_loc, torch.nonzero(interior).view(-1)])
    flat = coords_loc.reshape(3, -1)
    keys = torch.stack([_ordered(flat[0][rep_loc]), _ordered(flat[1][rep_loc]), _ordered(flat[2][rep_loc]),
                        rep_loc + g0], dim=1)
    grank = global_ranks(comm, keys)
    # ids to every copy: the owner's lowest copy carries gid + 1, the plan sums
    val = torch.zeros(P, dtype=torch.int64, device=dev)
    val[rep_loc] = grank + 1
    gid = plan_sum(comm, plan, val) - 1
    ntot = int(all_gather_cat(comm, torch.tensor([keys.shape[0]], dtype=torch.int64, device=dev)).sum())
    return gid, plan, mult.to(torch.uint8), ntot


def topo_keys_local(elements_loc, n):
    from .space import topo_keys

    return topo_keys(elements_loc, n)
