"""Device-resident function space and gather-scatter (reference space.py).

``build_space(mesh, basis)`` builds everything on the GPU:

* GLL coordinates and geometric factors with the sm_100a setup kernels, bit-
  identical to the reference's numba-lane ``build_space`` (space.py:195-262);
* the gather-scatter numbering (space.py:265-314).  The reference groups
  coincident points with a KD-tree and union-find; here coincident points are
  grouped *topologically* -- a GLL point on an element vertex, edge or face is
  keyed by the mesh-vertex ids of that entity plus its canonical position on it
  -- which yields the same groups on every conforming mesh the reference
  accepts, in O(P log P) device sorts instead of 80 s of host work at 32^3.
  Group ids are then ordered exactly as the reference orders them (lexicographic
  by the *exact bits* of the representative's (x, y, z), representative = lowest
  local index), and ``perm``/``offsets`` follow (ascending local index within a
  gid).  gid/perm/offsets are bit-identical to the reference (tests/test_setup_parity.py).

Memory layout in HBM (per rank): fields (E, n, n, n) float64; geom (6, E, n^3);
rx (3, 3, E, n^3); bm; uint8 multiplicity (1 B/point, for glsc3 weights);
int32 shared-gid maps (S_g + 1 offsets, S_l perm) for dssum; per-element
bitmasks (ceil(n^3/32) uint32 words) for masks and the shared-point set.
"""

import math

import numpy as np
import torch

from . import _device, _lib, traffic
from . import topology as _topo
from .errors import ConfigError, GeometryError, TopologyError

_FACE_NORMAL_SIGN = (-1.0, 1.0, 1.0, -1.0, -1.0, 1.0)

#: dssum kernel: "blk" (element-range blocks, default) or "cls" (class by class)
import os as _os

_DSSUM_KERNEL = _os.environ.get("SEMFLOW_B200_DSSUM", "blk")
_DSSUM_ITEMS = int(_os.environ.get("SEMFLOW_B200_DSSUM_ITEMS", 1024))   # shared gids per block


# --------------------------------------------------------------------------- bits

def pack_bits(flags):
    """(E, nnn) bool -> (E, ceil(nnn/32)) int32 words, bit p of element e = flags[e, p]."""
    E, nnn = flags.shape
    wpe = (nnn + 31) // 32
    pad = wpe * 32 - nnn
    f = flags.to(torch.int64)
    if pad:
        f = torch.nn.functional.pad(f, (0, pad))
    f = f.view(E, wpe, 32)
    sh = torch.arange(32, device=flags.device, dtype=torch.int64)
    words = (f << sh).sum(dim=2)
    words = torch.where(words >= 2**31, words - 2**32, words)
    return words.to(torch.int32).contiguous()


# --------------------------------------------------------------------------- gather-scatter

def interior_run(iface, E):
    """Longest run [lo, hi) of elements 0..E-1 containing none of the sorted
    element ids ``iface``, with an even start and an even (or E) end -- the
    interior computed while a halo exchange travels; None if shorter than 2."""
    edges = np.concatenate([[-1], np.asarray(iface, dtype=np.int64), [E]])
    gaps = edges[1:] - edges[:-1] - 1
    k = int(np.argmax(gaps))
    lo, hi = int(edges[k]) + 1, int(edges[k + 1])
    lo += lo & 1
    hi = hi if hi == E else hi - (hi & 1)
    return (lo, hi) if hi - lo >= 2 else None


class GatherScatter:
    """Direct-stiffness summation QQ^T on device (reference space.py:20-76).

    Reference-format maps (int64 device tensors ``gid``, ``perm``, ``offsets``;
    float64 ``mult``/``invmult`` on demand) are kept for parity checks and the
    unique-value helpers.  The hot path uses only the *shared* maps:
    ``sh_off``/``sh_perm`` (int32) over the gids of multiplicity > 1, and the
    uint8 multiplicity ``mult8`` for glsc3 weights.
    """

    def __init__(self, gid, perm, offsets, shape, comm=None, starts=None, plan=None, mult8=None, n_gid=None):
        """gid/perm/offsets: the GLOBAL reference-format numbering.  With a
        multi-rank ``comm``, this rank owns elements starts[rank]..starts[rank+1]
        and its dssum reads the other ranks' copies through a halo exchange.
        Partitioned build (partition.py): ``gid`` is this rank's slice, perm /
        offsets are None and ``plan``, ``mult8``, ``n_gid`` come with it."""
        from . import dist as _dist

        self.shape = tuple(shape)
        self.device = gid.device
        self.comm = comm if comm is not None else _dist.single()
        E = self.shape[0]
        P = E * int(np.prod(self.shape[1:])) if len(self.shape) > 1 else int(gid.numel())
        self.P = P
        if P >= 2**31 - 1:
            raise ConfigError("more than 2^31 local points on one device; partition the mesh")
        self.plan = None
        if plan is not None:
            self.n_gid = int(n_gid)
            self._init_ranked(gid.contiguous(), plan, mult8.contiguous())
            return
        self.n_gid = int(offsets.numel() - 1)
        counts = offsets[1:] - offsets[:-1]
        if counts.numel() and int(counts.max()) > 255:
            raise TopologyError("a global id has more than 255 local copies")
        if self.comm.world > 1:
            nnn = P // E
            r = self.comm.rank
            g0 = starts[r] * nnn
            gl = gid[g0:g0 + P].clone()
            self._init_ranked(gl, _dist.build_halo_plan(gid, perm, offsets, starts, r, nnn),
                              counts[gl].to(torch.uint8).contiguous())
            return
        self.gid = gid
        self.perm = perm
        self.offsets = offsets
        self.mult8 = counts[gid].to(torch.uint8).contiguous()
        # shared gids (multiplicity > 1), processed in the order of their lowest
        # local copy: consecutive threads of the dssum kernel then touch
        # neighbouring memory (the per-gid summation order is unaffected)
        shared_g = torch.nonzero(counts > 1).view(-1)
        self.n_shared = int(shared_g.numel())
        first = perm[offsets[shared_g]]
        g_sorted = shared_g[torch.argsort(first)]
        cnt = counts[g_sorted]
        self.sh_off = torch.zeros(self.n_shared + 1, dtype=torch.int32, device=self.device)
        if self.n_shared:
            self.sh_off[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        total = int(cnt.sum()) if self.n_shared else 0
        start = torch.repeat_interleave(offsets[g_sorted], cnt)
        within = torch.arange(total, device=self.device) - torch.repeat_interleave(
            self.sh_off[:-1].to(torch.int64), cnt)
        self.sh_perm = perm[start + within].to(torch.int32).contiguous()
        E = self.shape[0]
        nnn = P // E if E else 0
        self.shared_bits = pack_bits((self.mult8 > 1).view(E, nnn)) if E else None
        self._masked_perm = {}
        self._mult = None
        if self.device.type == "cuda":
            self._build_classes()

    def _init_ranked(self, gid_loc, plan, mult8):
        """Multi-rank state: local gid slice, halo plan, multiplicities."""
        from . import dist as _dist

        E = self.shape[0]
        nnn = self.P // E
        self.gid = gid_loc
        self.perm = self.offsets = None      # global maps are not kept per rank
        self.mult8 = mult8
        self.plan = plan
        self.n_shared = plan.n_shared
        self.sh_off = plan.sh_off.contiguous()
        self.sh_perm = plan.sh_perm.contiguous()
        self.shared_bits = pack_bits((self.mult8 > 1).view(E, nnn))
        self._sendbuf = torch.empty(int(plan.send_all.numel()), dtype=torch.float64, device=self.device)
        self._recvbuf = torch.empty(max(plan.n_recv_total, 1), dtype=torch.float64, device=self.device)
        # NVLink halo (csrc/halo.cu) when the peer-memory path is up; NCCL otherwise
        self._ipc = None
        if self.comm.peer is not None and _os.environ.get("SEMFLOW_B200_HALO", "ipc") != "nccl":
            self._ipc = _dist.HaloIPC(self.comm, plan)
        self._masked_perm = {}
        self._mult = None
        # every host-synchronising derivation done now: an operator application
        # may first run inside a CUDA-graph capture (krylov._graph_buffers)
        if self.device.type == "cuda":
            self._build_classes()
            self.interior_range()

    # ------------------------------------------------------------ properties
    @property
    def mult(self):
        if self._mult is None:
            self._mult = self.mult8.to(torch.float64).view(self.shape)
        return self._mult

    @property
    def invmult(self):
        return 1.0 / self.mult

    @property
    def shared_local_points(self):
        return int(self.sh_perm.numel())

    # ------------------------------------------------------------ kernels
    def interior_range(self):
        """(lo, hi): the longest run of local elements with no interface copy (even
        bounds), computed once -- the operator computes [0, lo) and [hi, E) first,
        posts the halo exchange, then computes [lo, hi) while it travels.  None
        when there is no such run (single rank, NCCL path, tiny partitions)."""
        if getattr(self, "_interior", False) is not False:
            return self._interior
        self._interior = None
        if self.plan is None or not self.plan.peers or self._ipc is None:
            return None
        E = self.shape[0]
        nnn = self.P // E
        self._interior = interior_run(torch.unique(self.plan.send_all.long() // nnn).cpu().numpy(), E)
        return self._interior

    def halo_put(self, v):
        self._ipc.put(v)

    def halo_wait(self):
        return self._ipc.wait(self.device)

    def halo_exchange(self, v):
        """Send this rank's interface copies of field v, receive the peers' (raw values).
        Returns the receive buffer (None on a single rank)."""
        plan = self.plan
        if plan is None or not plan.peers:
            return None
        if self._ipc is not None:
            return self._ipc.exchange(v)
        st = _lib.stream_ptr(self.device)
        _lib.call("sf_gather_f64", _lib.ptr(self._sendbuf), _lib.ptr(v), _lib.ptr(plan.send_all),
                  int(plan.send_all.numel()), st)
        sends = {q: self._sendbuf[plan.send_off[q]:plan.send_off[q] + int(plan.send_idx[q].numel())]
                 for q in plan.send_idx}
        recvs = {q: self._recvbuf[plan.recv_off[q]:plan.recv_off[q] + plan.n_recv[q]] for q in plan.n_recv}
        self.comm.exchange(sends, recvs)
        return self._recvbuf

    def _build_classes(self):
        """Multiplicity-class layout of the shared maps (sf_dssum_cls_f64): pairs,
        quads, octets at fixed stride, the rest in CSR; order within a class kept."""
        dev = self.device
        off = self.sh_off.long()
        cnt = off[1:] - off[:-1]
        parts, n = [], {}
        for c in (2, 4, 8):
            sel = torch.nonzero(cnt == c).view(-1)
            n[c] = int(sel.numel())
            idx = (off[sel].view(-1, 1) + torch.arange(c, device=dev).view(1, c)).reshape(-1)
            parts.append(self.sh_perm[idx])
        other = torch.nonzero((cnt != 2) & (cnt != 4) & (cnt != 8)).view(-1)
        oc = cnt[other]
        gen_off = torch.zeros(other.numel() + 1, dtype=torch.int64, device=dev)
        if other.numel():
            gen_off[1:] = torch.cumsum(oc, 0)
        within = torch.arange(int(gen_off[-1]), device=dev) - torch.repeat_interleave(gen_off[:-1], oc)
        parts.append(self.sh_perm[torch.repeat_interleave(off[other], oc) + within])
        # pairs segment padded to a multiple of 4 ints: the quads/octets after it
        # are read as 16-byte int4 (csrc/gs.cu pairs_span)
        self.cls_pad2 = (-2 * n[2]) % 4
        pad = torch.zeros(self.cls_pad2, dtype=parts[0].dtype, device=dev)
        self.cls_perm = torch.cat([parts[0], pad] + parts[1:]).to(torch.int32).contiguous()
        self.cls_n = (n[2], n[4], n[8])
        self.cls_gen_off = gen_off.to(torch.int32).contiguous()
        self.cls_n_gen = int(other.numel())
        n_all = sum(int(t.numel()) for t in parts)
        n_loc = sum(int((t < self.P).sum()) for t in parts)
        self.dss_bytes = traffic.dssum_bytes(n_loc, n_all - n_loc, n[2] + n[4] + n[8] + self.cls_n_gen)
        # element-range blocks for sf_dssum_blk_f64: every class's items are ordered
        # by lowest local copy, so a block's items are one contiguous run per class
        E = self.shape[0]
        nnn = self.P // E if E else 1
        big = torch.iinfo(torch.int64).max
        keys = []
        for c, part in zip((2, 4, 8), parts[:3]):
            p = part.view(-1, c).long()
            keys.append(torch.where(p < self.P, p, torch.full_like(p, big)).min(dim=1).values // nnn
                        if p.numel() else p.new_zeros(0))
        gp = parts[3].long()
        if other.numel():
            item = torch.repeat_interleave(torch.arange(other.numel(), device=dev), oc)
            kl = torch.where(gp < self.P, gp, torch.full_like(gp, big))
            keys.append(torch.full((other.numel(),), big, dtype=torch.int64, device=dev)
                        .scatter_reduce(0, item, kl, "amin") // nnn)
        else:
            keys.append(gp.new_zeros(0))
        total = sum(int(k.numel()) for k in keys)
        eb = max(1, round(_DSSUM_ITEMS * E / total)) if total else 1
        nb = (E + eb - 1) // eb if total else 0
        edges = torch.arange(nb + 1, device=dev, dtype=torch.int64) * eb
        self.cls_nb, self.cls_eb = nb, eb
        self.cls_bstart = torch.cat([torch.searchsorted(k.contiguous(), edges) for k in keys]).to(torch.int32) \
            if nb else torch.zeros(4, dtype=torch.int32, device=dev)

    def dssum_into(self, v, mode, u=None, perm=None, pre=None, recv=False):
        """In-place dssum of one scalar row v (mode 0 add / 1 avg / 2 masked with u).
        ``perm``: a flagged copy of ``cls_perm`` (masked operators); ``pre``: the
        masked copies receive pre * u (operator applied with sf_ax_pre_f64);
        ``recv``: the receive buffer of an exchange the caller already posted."""
        if recv is False:
            recv = self.halo_exchange(v)
        if not hasattr(self, "cls_perm"):
            self._build_classes()
        n2, n4, n8 = self.cls_n
        pm = self.cls_perm if perm is None else perm
        self.account_dssum()
        seq_ptr = getattr(recv, "seq_ptr", None)        # banked NVLink inbox (dist.BankedRecv)
        if _DSSUM_KERNEL == "cls" and pre is None and seq_ptr is None:
            _lib.call("sf_dssum_cls_f64", _lib.ptr(v), _lib.ptr(pm), n2, n4, n8, _lib.ptr(self.cls_gen_off),
                      self.cls_n_gen, mode, _lib.ptr(u), _lib.ptr(recv), self.P, _lib.stream_ptr(self.device))
        else:
            _lib.call("sf_dssum_blk_f64", _lib.ptr(v), _lib.ptr(pm), n2, n4, n8, _lib.ptr(self.cls_gen_off),
                      _lib.ptr(self.cls_bstart), self.cls_nb, mode, _lib.ptr(u), _lib.ptr(pre), _lib.ptr(recv),
                      self.P, seq_ptr, getattr(recv, "bank", 0), _lib.stream_ptr(self.device))

    def account_dssum(self):
        """Credit one dssum's algorithmic bytes to the step accounting (traffic.py)."""
        if _lib.ACCOUNT:
            if not hasattr(self, "cls_perm"):
                self._build_classes()
            _lib.BYTES[0] += self.dss_bytes

    def _dssum_rows(self, flat, mode, u=None):
        for row in range(flat.shape[0]):
            self.dssum_into(flat[row], mode, u[row] if u is not None else None)

    def add_(self, u):
        """In-place QQ^T u (any leading axes, one row per leading index)."""
        _lib.require_cuda(u)
        flat = u.view(-1, self.P)
        self._dssum_rows(flat, 0)
        return u

    def avg_(self, u):
        _lib.require_cuda(u)
        flat = u.view(-1, self.P)
        self._dssum_rows(flat, 1)
        return u

    def add(self, u):
        """QQ^T u into a new tensor (space.py:38-49)."""
        return self.add_(u.contiguous().clone())

    def avg(self, u):
        """Multiplicity-weighted average, sum * (1.0/count) (space.py:51-60)."""
        return self.avg_(u.contiguous().clone())

    def masked_perm(self, keep_flat):
        """Class-layout shared perm (cls_perm) with bit 31 set on the local copies
        whose mask is 0 -- the map of a masked operator's dssum."""
        if not hasattr(self, "cls_perm"):
            self._build_classes()
        loc = self.cls_perm.long()
        is_local = loc < self.P
        dropped = torch.zeros_like(is_local)
        dropped[is_local] = ~keep_flat[loc[is_local]]
        return torch.where(dropped, self.cls_perm | torch.tensor(-2**31, dtype=torch.int32, device=self.device),
                           self.cls_perm).contiguous()

    def dot_async(self, u, v, out):
        """Write <u, v>_{1/mult} (summed over ranks) into the device scalar ``out``."""
        w = _device.workspace(self.device)
        peer = self.comm.peer
        if peer is not None:
            _lib.call("sf_glsc3_peer_f64", _lib.ptr(u), _lib.ptr(v), _lib.ptr(self.mult8), self.P, *w.args(),
                      _lib.ptr(out), *peer.fused_args(), _lib.stream_ptr(self.device))
            return out
        _lib.call("sf_glsc3_f64", 1, ctypes_ptrs([u]), ctypes_ptrs([v]), _lib.ptr(self.mult8), self.P,
                  *w.args(), _lib.ptr(out), _lib.stream_ptr(self.device))
        self.comm.sum_(out)
        return out

    def dot(self, u, v):
        """Multiplicity-weighted inner product of scalar fields (space.py:72-76), host float."""
        if u.numel() != self.P or v.numel() != self.P:
            raise ValueError("GatherScatter.dot takes scalar fields (the reference's invmult "
                             "weighting does not broadcast over vector fields)")
        w = _device.workspace(self.device)
        self.dot_async(u.contiguous(), v.contiguous(), w.slots[0:1])
        return w.read(0)[0]

    def gather_unique(self, u):
        """One value per global id, the value of its first copy in global local-
        index order (space.py:62-64): shape (n_gid,).  On a partitioned space a
        collective -- every rank contributes the gids whose first copy it holds
        (lowest local index of the gid on the lowest rank that has one) and every
        rank gets the whole vector, bit for bit."""
        if self.perm is not None:
            return u.reshape(-1)[self.perm[self.offsets[:-1]]]
        from .partition import all_gather_cat

        own = self._first_copies()
        g = self.gid.long()[own]
        v = u.reshape(-1)[own].to(torch.float64)
        comm = self.comm
        n = torch.tensor([own.numel()], dtype=torch.int64, device=self.device)
        counts = all_gather_cat(comm, n).cpu().tolist()
        m = max(counts)
        pad_g = torch.zeros(m, dtype=torch.int64, device=self.device)
        pad_v = torch.zeros(m, dtype=torch.float64, device=self.device)
        pad_g[:g.numel()] = g
        pad_v[:v.numel()] = v
        all_g = all_gather_cat(comm, pad_g).view(comm.world, m)
        all_v = all_gather_cat(comm, pad_v).view(comm.world, m)
        out = torch.empty(self.n_gid, dtype=torch.float64, device=self.device)
        for q, c in enumerate(counts):
            out[all_g[q, :c]] = all_v[q, :c]
        return out

    def _first_copies(self):
        """Local indices that are the first copy of their gid (partitioned space)."""
        own = getattr(self, "_own_first", None)
        if own is not None:
            return own
        g = self.gid.long()
        idx = torch.arange(g.numel(), device=self.device)
        first = torch.full((self.n_gid,), g.numel(), dtype=torch.int64, device=self.device)
        first.scatter_reduce_(0, g, idx, reduce="amin", include_self=True)
        keep = first[g] == idx
        # a gid shared with a lower rank has its first copy there (ranks hold
        # ascending element ranges); the halo plan sends every local copy of such gids
        r = self.comm.rank
        for q, sidx in self.plan.send_idx.items():
            if q < r:
                keep[sidx.long()] = False
        self._own_first = idx[keep]
        return self._own_first

    def scatter_unique(self, vals, shape):
        """Spread per-global-id values (n_gid,) to every local copy (space.py:66-70)."""
        vals = torch.as_tensor(vals, dtype=torch.float64, device=self.device)
        if self.perm is None:
            return vals[self.gid.long()].view(shape)
        counts = self.offsets[1:] - self.offsets[:-1]
        out = torch.empty(int(np.prod(shape)), dtype=torch.float64, device=self.device)
        out[self.perm] = torch.repeat_interleave(vals, counts)
        return out.view(shape)


def ctypes_ptrs(tensors):
    import ctypes

    arr = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    return arr


# --------------------------------------------------------------------------- topology

def _boundary_point_table(n):
    """Per local boundary point of an element: kind and the corners/positions that key it.

    Returns numpy arrays over the nb boundary points: lp (local index), kind
    (0 vertex, 1 edge, 2 face), corners (nb, 4) and positions (nb, 2).
    For edges corners[:, :2] are the edge ends at parameter 0 and m; for faces
    corners = (c00, c10, c01, c11) over the two in-face axes a1 < a2.
    """
    m = n - 1
    lp, kind, cor, pos = [], [], [], []
    for i in range(n):
        for j in range(n):
            for k in range(n):
                idx = (i, j, k)
                inner = [0 < v < m for v in idx]
                ni = sum(inner)
                if ni == 3:
                    continue
                hi = [1 if v == m else 0 for v in idx]
                if ni == 0:
                    c = hi[0] | (hi[1] << 1) | (hi[2] << 2)
                    lp.append((i * n + j) * n + k); kind.append(0)
                    cor.append((c, c, c, c)); pos.append((0, 0))
                elif ni == 1:
                    ax = inner.index(True)
                    base = [hi[0], hi[1], hi[2]]
                    base[ax] = 0
                    ca = base[0] | (base[1] << 1) | (base[2] << 2)
                    cb = ca | (1 << ax)
                    lp.append((i * n + j) * n + k); kind.append(1)
                    cor.append((ca, cb, ca, cb)); pos.append((idx[ax], 0))
                else:
                    a1, a2 = [a for a in range(3) if inner[a]]
                    fixed = [a for a in range(3) if not inner[a]][0]
                    base = [0, 0, 0]
                    base[fixed] = hi[fixed]

                    def corner(b1, b2):
                        c = list(base)
                        c[a1] = b1
                        c[a2] = b2
                        return c[0] | (c[1] << 1) | (c[2] << 2)

                    lp.append((i * n + j) * n + k); kind.append(2)
                    cor.append((corner(0, 0), corner(1, 0), corner(0, 1), corner(1, 1)))
                    pos.append((idx[a1], idx[a2]))
    return (np.array(lp, dtype=np.int64), np.array(kind, dtype=np.int64),
            np.array(cor, dtype=np.int64), np.array(pos, dtype=np.int64))


def topo_keys(elements, n):
    """Topological keys (k1, k2) of every boundary point of the given elements and
    the point's index within the block (element-major): two points coincide in a
    conforming mesh iff their keys are equal.  Vertices are keyed by their vertex
    id; edge points by the edge's two vertex ids and the position along the edge
    counted from the lower id; face points by the face's lowest vertex id, its two
    neighbours on the face and the in-face position in the frame anchored at the
    lowest id.  elements: (E, 8) int64 vertex ids (< 2^30)."""
    dev = elements.device
    E = elements.shape[0]
    nnn = n ** 3
    m = n - 1
    if E and int(elements.max()) >= 2**30:
        raise ConfigError("vertex ids must be < 2^30")
    lp, kind, cor, pos = (torch.from_numpy(a).to(dev) for a in _boundary_point_table(n))
    nb = lp.numel()
    V = elements[:, cor.view(-1)].view(E, nb, 4)            # (E, nb, 4) vertex ids
    kind_b = kind.view(1, nb).expand(E, nb)
    p1 = pos[:, 0].view(1, nb).expand(E, nb)
    p2 = pos[:, 1].view(1, nb).expand(E, nb)
    va, vb, vc, vd = V[..., 0], V[..., 1], V[..., 2], V[..., 3]
    # edges: orient from the lower vertex id
    e_lo = torch.minimum(va, vb)
    e_hi = torch.maximum(va, vb)
    e_pos = torch.where(va < vb, p1, m - p1)
    # faces: origin at the lowest vertex id, first axis toward its lower neighbour
    four = torch.stack([va, vb, vc, vd], dim=-1)            # (c00, c10, c01, c11)
    v0, arg = four.min(dim=-1)
    b1 = arg & 1
    b2 = arg >> 1
    nA = four.gather(-1, ((1 - b1) | (b2 << 1)).unsqueeze(-1)).squeeze(-1)   # neighbour along a1
    nB = four.gather(-1, (b1 | ((1 - b2) << 1)).unsqueeze(-1)).squeeze(-1)   # neighbour along a2
    q1 = torch.where(b1 == 0, p1, m - p1)
    q2 = torch.where(b2 == 0, p2, m - p2)
    f_P = torch.where(nA < nB, q1, q2)
    f_Q = torch.where(nA < nB, q2, q1)
    f_lo = torch.minimum(nA, nB)
    f_hi = torch.maximum(nA, nB)
    k1 = torch.where(kind_b == 0, va << 30,
                     torch.where(kind_b == 1, (1 << 60) | (e_lo << 30) | e_hi,
                                 (2 << 60) | (v0 << 30) | f_lo))
    k2 = torch.where(kind_b == 0, torch.zeros_like(va),
                     torch.where(kind_b == 1, e_pos, (f_hi << 16) | (f_P * n + f_Q)))
    del V, four, nA, nB, q1, q2, f_P, f_Q, f_lo, f_hi, e_lo, e_hi, e_pos
    gpt = (torch.arange(E, device=dev, dtype=torch.int64).view(E, 1) * nnn + lp.view(1, nb)).reshape(-1)
    return k1.reshape(-1), k2.reshape(-1), gpt


def build_gather_scatter(elements, coords, n, tol=None):
    """Bit-exact reference numbering (space.py:265-314) from topology + coordinates.

    elements: (E, 8) int64 device tensor of vertex ids; coords: (3, E, n, n, n).
    With ``tol`` (the reference's 1e-8 * max element diameter) the topological
    groups are cross-checked against the geometric tol-pairs (topology.py)."""
    dev = coords.device
    E = elements.shape[0]
    nnn = n ** 3
    P = E * nnn
    k1, k2, gpt = topo_keys(elements, n)
    # lexicographic sort by (k1, k2), ties by point index (stable sorts)
    o = torch.sort(k2, stable=True).indices
    o = o[torch.sort(k1[o], stable=True).indices]
    sk1, sk2 = k1[o], k2[o]
    newg = torch.ones_like(sk1, dtype=torch.bool)
    if newg.numel() > 1:
        newg[1:] = (sk1[1:] != sk1[:-1]) | (sk2[1:] != sk2[:-1])
    grp_sorted = torch.cumsum(newg.to(torch.int64), 0) - 1
    n_bgroups = int(grp_sorted[-1]) + 1 if grp_sorted.numel() else 0
    grp_of_b = torch.empty_like(grp_sorted)
    grp_of_b[o] = grp_sorted
    del o, sk1, sk2, newg, k1, k2, grp_sorted
    # group index of every local point: boundary groups first, then interior points
    group = torch.empty(P, dtype=torch.int64, device=dev)
    group[gpt] = grp_of_b
    is_int = torch.ones(P, dtype=torch.bool, device=dev)
    is_int[gpt] = False
    int_pts = torch.nonzero(is_int).view(-1)
    group[int_pts] = n_bgroups + torch.arange(int_pts.numel(), device=dev)
    n_groups = n_bgroups + int_pts.numel()
    del is_int, int_pts, grp_of_b, gpt
    gid = _number_groups(group, n_groups, coords)
    del group
    if tol is not None:
        # the reference groups GEOMETRICALLY (space.py:265-291): raise its
        # TopologyErrors, and where the topological groups differ from the
        # tol-graph components (duplicated vertex ids, non-matching curved
        # faces) number the components instead -- the reference's maps
        pairs = _topo.coincident_pairs(coords, tol)
        _topo.check_pairs(pairs, elements, nnn, tol)
        if not _topo.topology_agrees(gid, pairs, coords, tol):
            lab = _topo.components(pairs, P)
            uniq, group = torch.unique(lab, return_inverse=True)
            gid = _number_groups(group, uniq.numel(), coords)
            del uniq, group, lab
        del pairs
    perm = torch.sort(gid, stable=True).indices
    n_groups = int(gid.max()) + 1 if gid.numel() else 0
    counts = torch.bincount(gid, minlength=n_groups)
    offsets = torch.zeros(n_groups + 1, dtype=torch.int64, device=dev)
    offsets[1:] = torch.cumsum(counts, 0)
    return gid, perm, offsets


def _number_groups(group, n_groups, coords):
    """Global ids of point groups in the reference's order (space.py:294-303): the
    representative of a group is its lowest local point; groups are ordered by
    representative (the union-find root order), then stably by the exact
    coordinate bits of the representative, x primary."""
    dev = group.device
    P = group.numel()
    rep = torch.full((n_groups,), P, dtype=torch.int64, device=dev)
    rep.scatter_reduce_(0, group, torch.arange(P, device=dev), reduce="amin")
    flat = coords.reshape(3, -1)
    order = torch.sort(rep).indices
    for l in (2, 1, 0):
        key = flat[l][rep[order]] + 0.0            # + 0.0 folds -0.0 into +0.0
        order = order[torch.sort(key, stable=True).indices]
    rank = torch.empty_like(order)
    rank[order] = torch.arange(n_groups, device=dev)
    return rank[group]


# --------------------------------------------------------------------------- space

def _face_grids(n):
    base = np.arange(n ** 3, dtype=np.int64).reshape(n, n, n)
    return np.stack([base[0], base[-1], base[:, 0], base[:, -1], base[:, :, 0], base[:, :, -1]])


class FunctionSpace:
    """Device analogue of the reference FunctionSpace (space.py:102-180)."""

    def __init__(self, basis, mesh, coords, rx, jac, bm, geom, gs, facet_elem, facet_face,
                 facet_tag, facet_flat, facet_normal, facet_warea, comm=None, e_range=None):
        from . import dist as _dist

        self.comm = comm if comm is not None else _dist.single()
        self.e_range = e_range if e_range is not None else (0, coords.shape[1])
        self._coords_h = self._jac_h = None
        self.basis = basis
        self.mesh = mesh
        self.coords = coords
        self.rx = rx
        self.jac = jac
        self.bm = bm
        self.geom = geom
        self.gs = gs
        self.facet_elem = facet_elem
        self.facet_face = facet_face
        self.facet_tag = facet_tag
        self.facet_flat = facet_flat
        self.facet_normal = facet_normal
        self.facet_warea = facet_warea
        self.device = coords.device
        self.dmat = np.ascontiguousarray(basis.dmat, dtype=np.float64)
        self.volume = self.integral(torch.ones(self.shape, dtype=torch.float64, device=self.device))

    # coordinates and Jacobian are set-up fields: release_setup_fields() moves them
    # to host memory (4 fields of HBM) and they come back to the device on access
    coords = property(lambda self: self._coords if self._coords is not None else self._coords_h.to(self.device),
                      lambda self, v: setattr(self, "_coords", v))
    jac = property(lambda self: self._jac if self._jac is not None else self._jac_h.to(self.device),
                   lambda self, v: setattr(self, "_jac", v))

    def release_setup_fields(self):
        """Keep coords and jac in host memory only (a large run's device budget:
        they are read at set-up -- boundary values, initial fields -- not per step)."""
        if self._coords is not None:
            self._coords_h = self._coords.cpu()
            self._jac_h = self._jac.cpu()
            self._coords = self._jac = None
            torch.cuda.empty_cache()

    n = property(lambda self: self.basis.n)
    n_elements = property(lambda self: self.bm.shape[0])
    shape = property(lambda self: (self.n_elements, self.n, self.n, self.n))
    x = property(lambda self: self.coords[0])
    y = property(lambda self: self.coords[1])
    z = property(lambda self: self.coords[2])
    n_points = property(lambda self: self.n_elements * self.n ** 3)

    def zeros(self):
        return torch.zeros(self.shape, dtype=torch.float64, device=self.device)

    def zeros_vec(self):
        return torch.zeros((3,) + self.shape, dtype=torch.float64, device=self.device)

    def from_function(self, fn):
        """fn(x, y, z) on device tensors (use torch ops)."""
        return torch.as_tensor(fn(self.coords[0], self.coords[1], self.coords[2]),
                               dtype=torch.float64, device=self.device)

    def integral(self, u):
        """GLL quadrature sum(bm * u) (space.py:159-161), host float."""
        w = _device.workspace(self.device)
        _lib.call("sf_glsc3_f64", 1, ctypes_ptrs([self.bm]), ctypes_ptrs([u.contiguous()]), None,
                  self.n_points, *w.args(), _lib.ptr(w.slots[1:2]), _lib.stream_ptr(self.device))
        self.comm.sum_(w.slots[1:2])
        return w.read(1)[0]

    def l2_norm(self, u):
        return float(math.sqrt(max(self.integral(u * u), 0.0)))

    def mean(self, u):
        return self.integral(u) / self.volume

    def facet_sel(self, tag):
        if tag not in self.mesh.tag_names:
            raise KeyError(f"unknown boundary tag {tag!r}; have {self.mesh.tag_names}")
        return self.facet_tag == self.mesh.tag_names.index(tag)


def _wc(points):
    """Trilinear corner weights (8, n^3), reference space.py:183-189 arithmetic."""
    xi = np.asarray(points, dtype=np.float64)
    n = xi.size
    phi = np.stack([(1.0 - xi) / 2.0, (1.0 + xi) / 2.0])
    wc = np.empty((8, n, n, n))
    for c in range(8):
        cr, cs, ct = c & 1, (c >> 1) & 1, (c >> 2) & 1
        wc[c] = phi[cr][:, None, None] * phi[cs][None, :, None] * phi[ct][None, None, :]
    return wc.reshape(8, -1)


def _facets(mesh, basis, coords, dev):
    n = basis.n
    F = int(mesh.facet_elem.size)
    grids = _face_grids(n)
    fe = np.asarray(mesh.facet_elem, dtype=np.int64)
    ff = np.asarray(mesh.facet_face, dtype=np.int64)
    flat = fe[:, None, None] * n ** 3 + grids[ff]                     # (F, n, n)
    flat_t = torch.from_numpy(flat).to(dev)
    if F == 0:
        return flat_t, torch.zeros((0, n, n, 3), dtype=torch.float64, device=dev), \
            torch.zeros((0, n, n), dtype=torch.float64, device=dev)
    d = torch.tensor(np.asarray(basis.dmat), dtype=torch.float64, device=dev)
    w = torch.tensor(np.asarray(basis.weights), dtype=torch.float64, device=dev)
    fx = coords.reshape(3, -1)[:, flat_t]                              # (3, F, n, n)
    ta = torch.einsum("ab,lfbc->lfac", d, fx)
    tb = torch.einsum("ab,lfcb->lfca", d, fx)
    sign = torch.tensor(_FACE_NORMAL_SIGN, dtype=torch.float64, device=dev)[torch.from_numpy(ff).to(dev)]
    raw = sign.view(1, F, 1, 1) * torch.cross(ta, tb, dim=0)
    area = torch.linalg.vector_norm(raw, dim=0)
    if bool((area <= 0.0).any()):
        bad = int(torch.nonzero(area <= 0.0)[0, 0])
        raise GeometryError("degenerate boundary facet", element=int(fe[bad]))
    normal = (raw / area).permute(1, 2, 3, 0).contiguous()
    warea = area * (w[:, None] * w[None, :])
    return flat_t, normal, warea


def _coords(mesh, basis, elements, c0, c1, dev, st):
    """Trilinear GLL coordinates of elements c0..c1, curved records applied
    (space.py:182-192, 204-213): (3, c1 - c0, n, n, n)."""
    n = basis.n
    verts = torch.from_numpy(np.ascontiguousarray(mesh.vertices, dtype=np.float64)).to(dev)
    corners = verts[elements[c0:c1]].contiguous()                          # (Ec, 8, 3)
    wc = torch.from_numpy(_wc(basis.points)).to(dev)
    coords = torch.empty((3, c1 - c0, n, n, n), dtype=torch.float64, device=dev)
    _lib.call("sf_trilinear_coords_f64", _lib.ptr(corners), _lib.ptr(wc), n, c1 - c0, _lib.ptr(coords), st)
    del corners, verts
    curved = np.asarray(getattr(mesh, "curved_elem", np.zeros(0, dtype=np.int64)), dtype=np.int64)
    if curved.size:
        if mesh.geom_order != basis.order:
            raise ConfigError(
                f"mesh curved geometry order {mesh.geom_order} does not match basis order "
                f"{basis.order}; regenerate the mesh at the solver order")
        sel = np.nonzero((curved >= c0) & (curved < c1))[0]
        if sel.size:
            cc = torch.from_numpy(np.ascontiguousarray(mesh.curved_coords[sel], dtype=np.float64)).to(dev)
            ce = torch.from_numpy(curved[sel] - c0).to(dev)
            for l in range(3):
                coords[l][ce] = cc[..., l]
    return coords


def build_space(mesh, basis, device=None, comm=None):
    """Bind a basis to a mesh on the GPU (reference space.py:195-262).

    With a multi-rank ``comm`` (paper_2207_07098_b200.dist.Comm) the returned
    space holds this rank's contiguous element range only."""
    _lib.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise _lib.LibraryError("build_space needs a CUDA device (no CPU fallback)")
    _topo.validate_mesh(mesh, dev)                       # space.py:201
    n = basis.n
    E = int(mesh.n_elements)
    nnn = n ** 3
    st = _lib.stream_ptr(dev)
    elements = torch.from_numpy(np.ascontiguousarray(mesh.elements, dtype=np.int64)).to(dev)
    from . import dist as _dist

    comm = comm if comm is not None else _dist.single()
    starts = _dist.element_ranges(E, comm.world)
    e0, e1 = starts[comm.rank], starts[comm.rank + 1]
    El = e1 - e0
    # partitioned build: this rank's coordinates and numbering only (partition.py)
    parted = comm.world > 1 and _os.environ.get("SEMFLOW_B200_GLOBAL_BUILD", "0") != "1"
    c0, c1 = (e0, e1) if parted else (0, E)
    coords = _coords(mesh, basis, elements, c0, c1, dev, st)
    lcoords = coords[:, e0:e1].contiguous() if (comm.world > 1 and not parted) else coords
    rx = torch.empty((3, 3, El, n, n, n), dtype=torch.float64, device=dev)
    jac = torch.empty((El, n, n, n), dtype=torch.float64, device=dev)
    bm = torch.empty_like(jac)
    geom = torch.empty((6, El, n, n, n), dtype=torch.float64, device=dev)
    dh, dptr = _lib.host_f64(basis.dmat)
    wh, wptr = _lib.host_f64(basis.weights)
    _lib.call("sf_metrics_f64", dptr, wptr, n, _lib.ptr(lcoords), El, _lib.ptr(rx), _lib.ptr(jac),
              _lib.ptr(bm), _lib.ptr(geom), st)
    # the reference checks the Jacobian before it numbers the nodes (space.py:224-232)
    bad = jac <= 0.0
    if comm.any(bool(bad.any())):
        if bool(bad.any()):
            e, i, j, k = (int(v) for v in torch.nonzero(bad)[0])
            raise GeometryError(f"non-positive Jacobian determinant {float(jac[e, i, j, k]):.3e}",
                                element=e + e0,
                                ref_coords=(basis.points[i], basis.points[j], basis.points[k]))
        raise GeometryError("non-positive Jacobian determinant on another rank")
    tol = _topo.gs_tolerance(mesh)
    gs = None
    if parted:
        from . import partition as _part

        gid, plan, mult8, n_gid = _part.partitioned_numbering(elements, coords, n, comm, starts,
                                                              int(mesh.vertices.shape[0]))
        # geometric cross-check of this rank's points (topology.py); a mesh whose
        # topology and geometry disagree falls back to the global build
        pairs = _topo.coincident_pairs(coords, tol)
        _topo.check_pairs(pairs, elements[e0:e1], nnn, tol)
        _, lg = torch.unique(gid, return_inverse=True)
        agree = _topo.topology_agrees(lg, pairs, coords, tol)
        del pairs, lg
        if comm.any(not agree):
            parted = False
            coords = _coords(mesh, basis, elements, 0, E, dev, st)
        else:
            gs = GatherScatter(gid, None, None, (El, n, n, n), comm=comm, starts=starts, plan=plan,
                               mult8=mult8, n_gid=n_gid)
            del gid, plan, mult8
    if gs is None:
        # the gather-scatter numbering is global (every rank builds it; it depends on
        # the exact coordinates of all elements), everything else is per rank
        gid, perm, offsets = build_gather_scatter(elements, coords, n, tol=tol)
        if comm.world > 1:
            coords = coords[:, e0:e1].contiguous()
            torch.cuda.empty_cache()
        gs = GatherScatter(gid, perm, offsets, (El, n, n, n), comm=comm, starts=starts)
        del gid, perm, offsets
    del elements
    fe = np.asarray(mesh.facet_elem, dtype=np.int64)
    sel = (fe >= e0) & (fe < e1)
    lmesh = _LocalFacets(fe[sel] - e0, np.asarray(mesh.facet_face)[sel])
    flat, normal, warea = _facets(lmesh, basis, coords, dev)
    return FunctionSpace(
        basis=basis, mesh=mesh, coords=coords, rx=rx, jac=jac, bm=bm, geom=geom, gs=gs,
        facet_elem=fe[sel] - e0, facet_face=np.asarray(mesh.facet_face)[sel].copy(),
        facet_tag=np.asarray(mesh.facet_tag)[sel].copy(), facet_flat=flat, facet_normal=normal,
        facet_warea=warea, comm=comm, e_range=(e0, e1))


class _LocalFacets:
    def __init__(self, facet_elem, facet_face):
        self.facet_elem = facet_elem
        self.facet_face = facet_face


def from_reference(ref_space, device=None):
    """Upload a reference ``semflow.space.FunctionSpace`` (numpy) as-is."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt)
    g = ref_space.gs
    gs = GatherScatter(t(g.gid, torch.int64), t(g.perm, torch.int64), t(g.offsets, torch.int64),
                       ref_space.shape)
    return FunctionSpace(
        basis=ref_space.basis, mesh=ref_space.mesh, coords=t(ref_space.coords), rx=t(ref_space.rx),
        jac=t(ref_space.jac), bm=t(ref_space.bm), geom=t(ref_space.geom), gs=gs,
        facet_elem=np.asarray(ref_space.facet_elem).copy(),
        facet_face=np.asarray(ref_space.facet_face).copy(),
        facet_tag=np.asarray(ref_space.facet_tag).copy(),
        facet_flat=t(ref_space.facet_flat, torch.int64), facet_normal=t(ref_space.facet_normal),
        facet_warea=t(ref_space.facet_warea))
