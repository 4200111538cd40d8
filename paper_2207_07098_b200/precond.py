"""Preconditioners on device: block Jacobi (reference precond.py:27-59) and the
hybrid overlapping Schwarz method (precond.py:94-250).
"""

import ctypes

import numpy as np
import torch

from .errors import SolverBreakdownError


def assembled_diagonal(space, lam_visc, lam_mass):
    """Analytic diagonal of lam_visc D^T G D + lam_mass B, assembled (precond.py:27-40).

    The three einsum terms are accumulated over m in ascending order starting
    from 0.0 -- the order numpy's einsum uses -- so the result is bit-identical
    to the reference.
    """
    d = torch.tensor(space.dmat, dtype=torch.float64, device=space.device)
    g = space.geom
    n = space.n
    d2 = d * d
    dd = torch.diagonal(d).contiguous()
    # two field buffers + one product temporary (in place; same operation order)
    diag = torch.zeros(space.shape, dtype=torch.float64, device=space.device)
    tmp = torch.empty_like(diag)
    for m in range(n):        # einsum("mi,emjk->eijk", d2, g0)
        diag.add_(torch.mul(d2[m].view(1, n, 1, 1), g[0][:, m:m + 1, :, :], out=tmp))
    t = torch.zeros_like(diag)
    for m in range(n):        # einsum("mj,eimk->eijk", d2, g3)
        t.add_(torch.mul(d2[m].view(1, 1, n, 1), g[3][:, :, m:m + 1, :], out=tmp))
    diag.add_(t)
    t.zero_()
    for m in range(n):        # einsum("mk,eijm->eijk", d2, g5)
        t.add_(torch.mul(d2[m].view(1, 1, 1, n), g[5][:, :, :, m:m + 1], out=tmp))
    diag.add_(t)
    del t
    di = dd.view(1, n, 1, 1)
    dj = dd.view(1, 1, n, 1)
    dk = dd.view(1, 1, 1, n)
    for gi, a, b in ((g[1], di, dj), (g[2], di, dk), (g[4], dj, dk)):
        torch.mul(gi, 2.0, out=tmp)
        tmp.mul_(a).mul_(b)
        diag.add_(tmp)
    diag.mul_(lam_visc)
    torch.mul(space.bm, lam_mass, out=tmp)
    diag.add_(tmp)
    del tmp
    return space.gs.add_(diag)


class BlockJacobi:
    """Inverse assembled diagonal; masked rows are identity (precond.py:43-59)."""

    def __init__(self, space, lam_visc, lam_mass, mask=None):
        diag = assembled_diagonal(space, float(lam_visc), float(lam_mass))
        if mask is not None:
            m = torch.as_tensor(mask, dtype=torch.float64, device=space.device).view(space.shape)
            diag = torch.where(m == 0.0, torch.ones_like(diag), diag)
        if not bool((diag > 0.0).all()):
            flat = diag.reshape(-1)
            bad = int(torch.argmin(flat))
            raise SolverBreakdownError(
                f"non-positive operator diagonal {float(flat[bad]):.3e} at flat point {bad}")
        self.inv_diag = (1.0 / diag).contiguous()
        self.space = space

    def __call__(self, r):
        return self.inv_diag * r


# =========================================================================== hybrid Schwarz

def _face_layer(n, face):
    """Local indices of the first GLL layer inside a face (precond.py:62-68)."""
    base = np.arange(n * n * n).reshape(n, n, n)
    sl = [slice(None)] * 3
    axis, side = divmod(face, 2)
    sl[axis] = 1 if side == 0 else n - 2
    return base[tuple(sl)].ravel()


def element_matrices(space, lam_visc, lam_mass, batch=64, elems=None, geom=None, bm=None):
    """Dense element matrices A_e (len(elems), n^3, n^3) on the device: the
    identity basis pushed through the element kernel with the element's metric
    replicated (precond.py:71-91) -- the same arithmetic as the matrix-free
    operator.  ``elems``: element indices (default all) into ``geom`` (6, E, n^3)
    / ``bm`` (E, n^3) (default the space's own)."""
    from . import _lib
    from .operators import _ex

    n = space.n
    nn = n ** 3
    dev = space.device
    geom = space.geom.view(6, -1, nn) if geom is None else geom
    bm = space.bm.view(-1, nn) if bm is None else bm
    E = bm.shape[0]
    el = torch.arange(E, device=dev) if elems is None else torch.as_tensor(elems, device=dev).long()
    M = int(el.numel())
    mats = torch.empty((M, nn, nn), dtype=torch.float64, device=dev)
    eye = torch.eye(nn, dtype=torch.float64, device=dev)
    for i0 in range(0, M, batch):
        i1 = min(M, i0 + batch)
        B = i1 - i0
        sel = el[i0:i1]
        g = geom[:, sel].repeat_interleave(nn, dim=1).contiguous()
        b = bm[sel].repeat_interleave(nn, dim=0).contiguous()
        u = eye.repeat(B, 1).contiguous()
        w = torch.empty_like(u)
        _lib.call("sf_ax_helm_f64", space.dmat.ctypes.data, n, _lib.ptr(g), _lib.ptr(b), _lib.ptr(u), _lib.ptr(w),
                  B * nn, float(lam_visc), float(lam_mass), _ex(), _lib.stream_ptr(dev))
        mats[i0:i1] = w.view(B, nn, nn).transpose(1, 2)
    return mats


_HASH_SEED = 0x5EED5C4A


def _hash_weights(k, dev, salt):
    """Two independent rows of odd random int64 multipliers (a 128-bit linear hash)."""
    g = torch.Generator(device="cpu").manual_seed(_HASH_SEED + salt)
    # drawn as (k, 2) so a longer draw extends a shorter one (same prefix)
    w = torch.randint(-(2 ** 62), 2 ** 62, (k, 2), generator=g, dtype=torch.int64) | 1
    return w.T.contiguous().to(dev)


def _row_hash(x, w):
    """(rows, k) int64 -> (rows, 2) wrap-around linear hashes."""
    return torch.stack([(x * w[0]).sum(dim=1), (x * w[1]).sum(dim=1)], dim=1)


def _classes(h):
    """Class id per row of the (rows, 2) hash, representatives = first row of each
    class; the second hash word must agree inside a class (else: no sharing)."""
    uniq, inv = torch.unique(h[:, 0], return_inverse=True)
    rows = torch.arange(h.shape[0], device=h.device)
    rep = torch.full((uniq.numel(),), h.shape[0], dtype=torch.int64, device=h.device)
    rep.scatter_reduce_(0, inv, rows, reduce="amin")
    if not bool((h[rep[inv], 1] == h[:, 1]).all()):
        return rows.clone(), rows.clone()
    return inv, rep


def _lexsort2(a, b):
    """Permutation sorting by a, then b (stable)."""
    o = torch.sort(b, stable=True).indices
    return o[torch.sort(a[o], stable=True).indices]


def _segment_sums(keys, vals):
    """(unique keys ascending, sum of each key's values in input order)."""
    o = torch.sort(keys, stable=True).indices
    ks, vs = keys[o], vals[o]
    newk = torch.ones_like(ks, dtype=torch.bool)
    newk[1:] = ks[1:] != ks[:-1]
    seg = torch.cumsum(newk.to(torch.int64), 0) - 1
    nseg = int(seg[-1]) + 1 if seg.numel() else 0
    sstart = torch.nonzero(newk).view(-1)
    slen = torch.bincount(seg, minlength=nseg)
    out = torch.zeros(nseg, dtype=vals.dtype, device=vals.device)
    for j in range(int(slen.max()) if nseg else 0):
        m_ = slen > j
        out[m_] = out[m_] + vs[sstart[m_] + j]
    return ks[sstart], out


def _metric_classes(geom, bm, share_bits, chunk=4096):
    """(class id per element, representative element per class) for geom (6, E,
    nn) / bm (E, nn): equal within share_bits bits of the element's scale (or
    bitwise for None)."""
    dev = bm.device
    E, nn = bm.shape
    wr = (torch.rand(7 * nn, generator=torch.Generator().manual_seed(_HASH_SEED), dtype=torch.float64)
          + 0.5).to(dev)
    feats = torch.empty((E, 9), dtype=torch.float64, device=dev)
    for x0 in range(0, E, chunk):
        x1 = min(E, x0 + chunk)
        v = torch.cat([geom[:, x0:x1].permute(1, 0, 2).reshape(x1 - x0, 6 * nn), bm[x0:x1]], dim=1)
        feats[x0:x1, :7] = v.view(x1 - x0, 7, nn).sum(dim=2)
        feats[x0:x1, 7] = (v * wr).sum(dim=1)
        feats[x0:x1, 8] = v.abs().amax(dim=1)
    # one scale for all summaries: a plane of round-off (the off-diagonal G of an
    # affine box) quantises to 0 instead of to its own noise
    rng = float(feats.abs().max()) or 1.0
    q = torch.round(feats / rng * float(2 ** 28)).to(torch.int64)
    cls, rep = _classes(_row_hash(q, _hash_weights(9, dev, 7)))
    # verify every element against its class representative; split the misfits
    bad = torch.zeros(E, dtype=torch.bool, device=dev)
    for x0 in range(0, E, chunk):
        x1 = min(E, x0 + chunk)
        r_ = rep[cls[x0:x1]]
        a = torch.cat([geom[:, x0:x1].permute(1, 0, 2).reshape(x1 - x0, 6 * nn), bm[x0:x1]], dim=1)
        b = torch.cat([geom[:, r_].permute(1, 0, 2).reshape(x1 - x0, 6 * nn), bm[r_]], dim=1)
        if share_bits is None:
            bad[x0:x1] = (a.view(torch.int64) != b.view(torch.int64)).any(dim=1)
        else:
            tol = a.abs().amax(dim=1) * float(2.0 ** -int(share_bits))
            bad[x0:x1] = (a - b).abs().amax(dim=1) > tol
    if bool(bad.any()):
        nb = int(bad.sum())
        cls = cls.clone()
        cls[bad] = int(rep.numel()) + torch.arange(nb, device=dev)
        rep = torch.cat([rep, torch.nonzero(bad).view(-1)])
    return cls, rep


def _face_neighbours(mesh, dev):
    """(E, 6) neighbour element across each face (-1 on exterior faces) and the
    neighbour's face number: faces keyed by their vertex SET, exactly two owners
    (precond.py:113-124)."""
    from .mesh import FACE_CORNERS

    el = torch.as_tensor(np.ascontiguousarray(mesh.elements), dtype=torch.int64, device=dev)
    E = el.shape[0]
    fc = torch.as_tensor(np.array(FACE_CORNERS), device=dev)
    fv = torch.sort(el[:, fc.view(-1)].view(E * 6, 4), dim=1).values
    nv = int(mesh.vertices.shape[0])
    dup = torch.zeros_like(fv, dtype=torch.bool)
    dup[:, 1:] = fv[:, 1:] == fv[:, :-1]
    fv = torch.sort(torch.where(dup, torch.full_like(fv, nv), fv), dim=1).values
    o = torch.arange(E * 6, device=dev)
    for c in (3, 2, 1, 0):
        o = o[torch.sort(fv[o, c], stable=True).indices]
    sk = fv[o]
    same = (sk[1:] == sk[:-1]).all(dim=1)
    nbr = torch.full((E * 6,), -1, dtype=torch.int64, device=dev)
    nface = torch.full((E * 6,), -1, dtype=torch.int64, device=dev)
    # exactly two owners: equal to the next, and not part of a run of three
    two = same.clone()
    if two.numel() > 1:
        two[1:] &= ~same[:-1]
        two[:-1] &= ~same[1:]
    i = torch.nonzero(two).view(-1)
    a, b = o[i], o[i + 1]
    nbr[a], nbr[b] = b // 6, a // 6
    nface[a], nface[b] = b % 6, a % 6
    return nbr.view(E, 6), nface.view(E, 6)


class _SchwarzStruct(ctypes.Structure):
    _fields_ = [
        ("G", ctypes.c_longlong), ("P", ctypes.c_longlong), ("nv", ctypes.c_longlong),
        ("nnn", ctypes.c_int), ("S", ctypes.c_int),
        ("first", ctypes.c_void_p), ("gid", ctypes.c_void_p), ("wsqrt", ctypes.c_void_p),
        ("rg", ctypes.c_void_p), ("rw", ctypes.c_void_p),
        ("pt_ptr", ctypes.c_void_p), ("pt_ent", ctypes.c_void_p), ("tw", ctypes.c_void_p),
        ("vfixed", ctypes.c_void_p), ("rc_part", ctypes.c_void_p), ("rc", ctypes.c_void_p),
        ("ac_width", ctypes.c_int), ("ac_col", ctypes.c_void_p), ("ac_val", ctypes.c_void_p),
        ("ac_inv_diag", ctypes.c_void_p),
        ("xc", ctypes.c_void_p), ("cr", ctypes.c_void_p), ("cz", ctypes.c_void_p), ("cp", ctypes.c_void_p),
        ("cap", ctypes.c_void_p), ("cpart", ctypes.c_void_p), ("cbar", ctypes.c_void_p),
        ("coarse_iters", ctypes.c_int), ("coarse_blocks", ctypes.c_int),
        ("sub", ctypes.c_void_p), ("rwg", ctypes.c_void_p), ("sol", ctypes.c_void_p),
        ("sol_recv", ctypes.c_void_p), ("n_sol", ctypes.c_longlong),
        ("acc_off", ctypes.c_void_p), ("acc_pos", ctypes.c_void_p),
        ("cvert", ctypes.c_void_p), ("ccorn", ctypes.c_void_p), ("constrained", ctypes.c_void_p),
        ("z", ctypes.c_void_p), ("rflag", ctypes.c_void_p), ("se", ctypes.c_void_p),
        ("L", ctypes.c_longlong),
    ]


class _Plan:
    """Send/receive lists of one exchange (the fields dist.HaloIPC reads)."""

    def __init__(self, send_idx, n_recv, dev):
        self.send_idx = {q: t for q, t in send_idx.items() if t.numel()}
        self.n_recv = {q: int(k) for q, k in n_recv.items() if k}
        self.peers = sorted(set(self.send_idx) | set(self.n_recv))
        self.recv_off, off = {}, 0
        for q in self.peers:
            self.recv_off[q] = off
            off += self.n_recv.get(q, 0)
        self.n_recv_total = off
        self.send_off, so = {}, 0
        for q in self.peers:
            self.send_off[q] = so
            so += int(self.send_idx[q].numel()) if q in self.send_idx else 0
        self.send_all = (torch.cat([self.send_idx[q] for q in self.peers if q in self.send_idx]).to(torch.int32)
                         if self.send_idx else torch.zeros(0, dtype=torch.int32, device=dev))


def _alltoallv(comm, lists, width, dtype, dev):
    from .partition import alltoallv

    return alltoallv(comm, lists, width, dtype, dev)


class HybridSchwarz:
    """Overlapping Schwarz subdomain solves plus a trilinear coarse solve
    (precond.py:94-250), applied by hand-written kernels (csrc/schwarz.cu), on
    one rank or across ranks.

    Subdomain e = element e's global ids plus the first GLL layer inside each
    face neighbour (precond.py:126-139); its matrix sums the dense element
    matrices of every element touching it in ascending element order, Dirichlet
    rows/columns replaced by identity (:140-156).  Setup is vectorised on the
    device and DEDUPLICATED: every subdomain gets a 128-bit signature of what
    its matrix is made of (the metric class of each candidate element, the
    positions its points land on, the Dirichlet pattern, the size), subdomains
    with equal signatures share one assembled matrix and one explicit inverse.
    Elements are in one metric class when their geometric factors agree to
    ``share_bits`` bits relative to the element's scale (40: ~1e-12; np.linspace
    boxes differ in the last bits only); ``share_bits=None`` shares only
    bitwise-equal geometry.  A box mesh has <= 5^3 distinct subdomains whatever
    its size; an unstructured mesh stores one S x S inverse per element, the
    reference's O(E S^2).

    Across ranks (N > 1) every rank treats its own elements' subdomains.  The
    elements a subdomain reaches on other ranks are all vertex neighbours of the
    rank's elements: their gid rows, metrics and masks are fetched once.  Each
    application exchanges over NVLink (dist.HaloIPC): the weighted residual of
    the other ranks' first layers after the gather, the restriction partials
    (summed in rank order on every rank; the coarse solve is replicated), and the
    subdomain solutions on gids held by other ranks, which every holder adds in
    ascending global subdomain order -- the reference's order.

    One application (``apply_into``) is stream-ordered with no host
    synchronisation (CUDA-graph capturable; the fused GMRES captures it): the
    gather / restriction / coarse CG / overlap sums / scatter kernels are ours,
    and each subdomain class's solves are one FP64 GEMM (cuBLAS, the FP64 tensor
    cores) on the gathered residual slots.
    Subdomain solves use the explicit inverse instead of LU back-substitution and
    the 10-iteration coarse Jacobi-CG a sparse vertex matrix, so one application
    agrees with the reference to rounding (~1e-13) and Krylov iteration counts
    are the reference's.
    """

    TILE = 4

    def __init__(self, space, mask=None, lam_visc=1.0, lam_mass=0.0, coarse_iters=10, chunk=2048,
                 share_bits=40):
        from . import _lib
        from . import dist as _dist
        from .errors import ConfigError

        lib = _lib.load()
        gs = space.gs
        comm = space.comm
        W, rk = comm.world, comm.rank
        self.space = space
        self.coarse_iters = int(coarse_iters)
        dev = space.device
        n, El = space.n, space.n_elements
        nn = n ** 3
        P = El * nn
        mesh = space.mesh
        Eg = int(mesh.n_elements)
        e0, e1 = space.e_range
        nv = int(mesh.vertices.shape[0])
        elements = torch.as_tensor(np.ascontiguousarray(mesh.elements), dtype=torch.int64, device=dev)
        keep = (torch.ones(P, dtype=torch.bool, device=dev) if mask is None else
                torch.as_tensor(mask, device=dev).reshape(-1) != 0)
        starts = _dist.element_ranges(Eg, W)
        BIG = 1 << 62

        # ---- X: own elements + the other ranks' vertex neighbours, ascending global id
        if W == 1:
            gx = torch.arange(El, device=dev)
            i0 = 0
            gid_X = gs.gid.view(El, nn)
            geom_X = space.geom.view(6, El, nn)
            bm_X = space.bm.view(El, nn)
            keep_X = keep.view(El, nn)
            owner_X = torch.zeros(El, dtype=torch.int64, device=dev)
        else:
            vl = torch.zeros(nv, dtype=torch.bool, device=dev)
            vl[elements[e0:e1].reshape(-1)] = True
            touch = vl[elements].any(dim=1)
            touch[e0:e1] = True
            gx = torch.nonzero(touch).view(-1)
            i0 = int(torch.searchsorted(gx, torch.tensor([e0], device=dev)))
            st_t = torch.tensor(starts, dtype=torch.int64, device=dev)
            owner_X = torch.searchsorted(st_t, gx, right=True) - 1
            remote = owner_X != rk
            H = gx[remote]
            Ho = owner_X[remote]
            req = {q: H[Ho == q].view(-1, 1) for q in range(W) if q != rk}
            got = _alltoallv(comm, req, 1, torch.int64, dev)             # what the peers need from me
            lo = lambda t: (t.view(-1) - e0)
            rep_i = {q: gs.gid.view(El, nn)[lo(t)] for q, t in got.items()}
            rep_f = {q: torch.cat([space.geom.view(6, El, nn)[:, lo(t)].permute(1, 0, 2).reshape(-1, 6 * nn),
                                   space.bm.view(El, nn)[lo(t)],
                                   keep.view(El, nn)[lo(t)].to(torch.float64)], dim=1) for q, t in got.items()}
            ans_i = _alltoallv(comm, rep_i, nn, torch.int64, dev)
            ans_f = _alltoallv(comm, rep_f, 8 * nn, torch.float64, dev)
            NX = int(gx.numel())
            gid_X = torch.empty((NX, nn), dtype=torch.int64, device=dev)
            fX = torch.empty((NX, 8 * nn), dtype=torch.float64, device=dev)
            gid_X[i0:i0 + El] = gs.gid.view(El, nn)
            fX[i0:i0 + El] = torch.cat([space.geom.view(6, El, nn).permute(1, 0, 2).reshape(El, 6 * nn),
                                       space.bm.view(El, nn), keep.view(El, nn).to(torch.float64)], dim=1)
            ridx = torch.nonzero(remote).view(-1)
            for q in ans_i:
                sel = ridx[Ho == q]
                gid_X[sel] = ans_i[q]
                fX[sel] = ans_f[q]
            geom_X = fX[:, :6 * nn].reshape(NX, 6, nn).permute(1, 0, 2).contiguous()
            bm_X = fX[:, 6 * nn:7 * nn].contiguous()
            keep_X = fX[:, 7 * nn:] != 0.0
            del fX, rep_i, rep_f, ans_i, ans_f
        NX = int(gx.numel())

        # ---- subdomains (global gids): own gids + first layer inside each face neighbour
        nbr, nface = _face_neighbours(mesh, dev)
        nbr, nface = nbr[e0:e1], nface[e0:e1]
        layer = torch.as_tensor(np.stack([_face_layer(n, f) for f in range(6)]), device=dev)
        parts = [gid_X[i0:i0 + El]]
        for f in range(6):
            e2 = nbr[:, f]
            x2 = torch.searchsorted(gx, e2.clamp(min=0)).clamp(max=NX - 1)
            idx = layer[nface[:, f].clamp(min=0)]                        # (El, n^2)
            vals = torch.gather(gid_X[x2], 1, idx)
            parts.append(torch.where((e2 >= 0).view(El, 1), vals, torch.full_like(vals, BIG)))
        s_ = torch.sort(torch.cat(parts, dim=1), dim=1).values
        dup = torch.zeros_like(s_, dtype=torch.bool)
        dup[:, 1:] = s_[:, 1:] == s_[:, :-1]
        s_ = torch.sort(torch.where(dup, torch.full_like(s_, BIG), s_), dim=1).values
        size = (s_ < BIG).sum(dim=1)
        S = int(size.max())
        subg = s_[:, :S].contiguous()
        del s_, dup, parts
        self.S = S

        # ---- node space: gids with an own copy first (ascending), then the other
        #      ranks' layer gids grouped by the rank that provides them
        loc_nodes, loc_inv = torch.unique(gid_X[i0:i0 + El], return_inverse=True)
        Lloc = int(loc_nodes.numel())
        # own nodes are numbered in the order of their first local copy (element
        # major): the gather, the overlap sums and the scatter then walk memory in
        # element order instead of the gids' coordinate order
        fpt = torch.full((Lloc,), P, dtype=torch.int64, device=dev)
        fpt.scatter_reduce_(0, loc_inv.reshape(-1), torch.arange(P, device=dev), reduce="amin")
        loc_rank = torch.empty(Lloc, dtype=torch.int64, device=dev)
        loc_rank[torch.argsort(fpt)] = torch.arange(Lloc, device=dev)
        del fpt, loc_inv
        vsub = subg[subg < BIG]
        pos = torch.searchsorted(loc_nodes, vsub).clamp(max=Lloc - 1)
        rem = torch.unique(vsub[loc_nodes[pos] != vsub])
        Xflat = gid_X.reshape(-1)
        if rem.numel():
            # provider: the rank of the first X element holding the gid
            pr = torch.searchsorted(rem, Xflat).clamp(max=rem.numel() - 1)
            hit = rem[pr] == Xflat
            xmin = torch.full((rem.numel(),), NX, dtype=torch.int64, device=dev)
            xmin.scatter_reduce_(0, pr[hit], torch.arange(NX, device=dev).repeat_interleave(nn)[hit], reduce="amin")
            prov = owner_X[xmin]
            o = _lexsort2(prov, rem)
            rem, prov = rem[o], prov[o]
        else:
            prov = torch.zeros(0, dtype=torch.int64, device=dev)
        L = Lloc + int(rem.numel())
        self.G, self.L = Lloc, L
        if rem.numel():
            rem_sorted, rem_ord = torch.sort(rem)

        def node_of(g, unused):
            """global gid -> node index (``unused`` where it is not a node)."""
            g = g.contiguous()
            p1 = torch.searchsorted(loc_nodes, g).clamp(max=Lloc - 1)
            out = torch.where(loc_nodes[p1] == g, loc_rank[p1], torch.full_like(g, unused))
            if rem.numel():
                p2 = torch.searchsorted(rem_sorted, g).clamp(max=rem.numel() - 1)
                out = torch.where((out == unused) & (rem_sorted[p2] == g), Lloc + rem_ord[p2], out)
            return out

        valid = subg < BIG
        sub = torch.where(valid, node_of(subg.clamp(max=BIG - 1), L), torch.full_like(subg, L))
        sub = torch.sort(sub, dim=1).values                     # sorted node ids, pad L
        gidn_X = node_of(Xflat, L + 1).view(NX, nn)
        del Xflat, subg

        # constrained nodes: a copy (within X, which holds every copy) with mask 0
        con_n = torch.zeros(L + 2, dtype=torch.int64, device=dev)
        con_n.index_add_(0, gidn_X.reshape(-1), (~keep_X).reshape(-1).to(torch.int64))
        constrained = con_n[:L] > 0
        del con_n

        # ---- X elements touching each node (ascending X index), for the candidates
        key = torch.unique(gidn_X.reshape(-1) * NX + torch.arange(NX, device=dev).repeat_interleave(nn))
        ge_g, ge_e = key // NX, key % NX
        ge_off = torch.zeros(L + 3, dtype=torch.int64, device=dev)
        ge_off[1:] = torch.cumsum(torch.bincount(ge_g, minlength=L + 2), 0)
        del key, ge_g

        # ---- metric classes of the X elements: elements whose geometric factors
        #      agree to ``share_bits`` bits relative to the element's own scale
        #      (default 40: ~1e-12) share one element matrix -- np.linspace meshes
        #      differ elementwise only in the last bits; share_bits=None requires
        #      bitwise equality.  Candidates come from a hash of robust summaries
        #      (per-plane sums quantised to 2^-28 of their range: a last-bit
        #      difference does not move them), then every element is checked
        #      against its candidate representative and split off if it differs.
        ecls, erep = _metric_classes(geom_X, bm_X, share_bits)

        # ---- subdomain signatures (candidate classes, landing slots, Dirichlet, size)
        bmg = None
        cw = None
        sig = torch.empty((El, 2), dtype=torch.int64, device=dev)
        sub_canon = torch.empty_like(sub)
        for r0 in range(0, El, chunk):
            r1 = min(El, r0 + chunk)
            cand, bi, sub_c = self._candidates(sub[r0:r1], gidn_X, ge_off, ge_e, L, NX)
            sub_canon[r0:r1] = sub_c
            R, C = cand.shape
            if cw is None or cw.shape[1] < C * nn:
                cw = _hash_weights(max(C, 64) * nn, dev, 2)
                sw = [_hash_weights(max(C, 64), dev, 3), _hash_weights(S, dev, 4), _hash_weights(1, dev, 5)]
            con = (constrained[sub_c.clamp(max=L - 1)] & (sub_c < L)).to(torch.int64)
            cc = torch.where(cand >= 0, ecls[cand.clamp(min=0)] + 1, torch.zeros_like(cand))
            # fixed positions whatever the chunk's candidate count: padding
            # candidates and points outside the subdomain contribute 0
            h = (_row_hash((bi + 1).reshape(R, C * nn), cw[:, :C * nn])
                 + _row_hash(cc, sw[0][:, :C]) + _row_hash(con, sw[1][:, :S])
                 + size[r0:r1].view(R, 1) * sw[2][:, :1].view(1, 2))
            whole = (size[r0:r1] == gs.n_gid) & (con.sum(dim=1) == 0)
            if bool(whole.any()):       # the 1e-8 mass shift makes these unique
                if W > 1:
                    raise ConfigError("HybridSchwarz: a subdomain covering the whole mesh needs one rank")
                h[whole] += torch.arange(r0, r1, device=dev)[whole].view(-1, 1) * 0x9E3779B97F4A7C15
            sig[r0:r1] = h
        scls, srep = _classes(sig)
        U = int(srep.numel())
        self.n_classes = U
        del sig

        # ---- element matrices of the metric classes in use, the distinct subdomain
        #      matrices (assembled in ascending candidate order) and their inverses
        used = []
        for u0 in range(0, U, 256):
            cand_r, _, _ = self._candidates(sub[srep[u0:u0 + 256]], gidn_X, ge_off, ge_e, L, NX)
            used.append(torch.unique(ecls[cand_r[cand_r >= 0]]))
        used = torch.unique(torch.cat(used))
        emats_u = element_matrices(space, lam_visc, lam_mass, elems=erep[used], geom=geom_X, bm=bm_X)
        slot_of = torch.full((int(erep.numel()),), -1, dtype=torch.int64, device=dev)
        slot_of[used] = torch.arange(used.numel(), device=dev)
        inv = torch.empty((U, S, S), dtype=torch.float64, device=dev)
        ar = torch.arange(S, device=dev)
        for u0 in range(0, U, 64):
            u1 = min(U, u0 + 64)
            reps = srep[u0:u1]
            cand, bi, sub_r = self._candidates(sub[reps], gidn_X, ge_off, ge_e, L, NX)
            B = reps.numel()
            A = torch.zeros((B, S + 1, S + 1), dtype=torch.float64, device=dev)   # slot S: sink
            bix = torch.where(bi >= 0, bi, torch.full_like(bi, S))
            rows = torch.arange(B, device=dev).view(B, 1, 1)
            for k in range(cand.shape[1]):
                ok = cand[:, k] >= 0
                if not bool(ok.any()):
                    continue
                blk = emats_u[slot_of[ecls[cand[:, k].clamp(min=0)]]]             # (B, nn, nn)
                blk = torch.where(ok.view(B, 1, 1), blk, torch.zeros_like(blk))
                bk = bix[:, k]
                A.index_put_((rows, bk.view(B, nn, 1), bk.view(B, 1, nn)), blk, accumulate=True)
            A = A[:, :S, :S].contiguous()
            con = constrained[sub_r.clamp(max=L - 1)] & (sub_r < L)
            for b in range(B):
                sz = int(size[int(reps[b])])
                fx = torch.nonzero(con[b]).view(-1)
                if fx.numel():
                    A[b, fx, :] = 0.0
                    A[b, :, fx] = 0.0
                    A[b, fx, fx] = 1.0
                elif sz == gs.n_gid:
                    if bmg is None:
                        bmg = gs.gather_unique(gs.add(space.bm))
                    A[b, ar[:sz], ar[:sz]] += 1e-8 * bmg[sub_r[b, :sz]]
                if sz < S:
                    A[b, sz:, sz:] = torch.eye(S - sz, dtype=torch.float64, device=dev)
            inv[u0:u1] = torch.linalg.inv(A)
            del A
        del emats_u

        # ---- local solves: subdomain rows grouped by class; class c's solutions
        #      are one FP64 GEMM  sol[p0:p1] = rw[sub[p0:p1]] @ inv_c^T
        order = torch.sort(scls, stable=True).indices
        cls_sorted = scls[order]
        newc = torch.ones(El, dtype=torch.bool, device=dev)
        newc[1:] = cls_sorted[1:] != cls_sorted[:-1]
        cstart = torch.nonzero(newc).view(-1).tolist() + [El]
        self.blocks = [(int(cls_sorted[a]), a, b) for a, b in zip(cstart[:-1], cstart[1:])]
        self.invT = inv.transpose(1, 2).contiguous()
        del inv
        self.order = order
        self.row_cls = cls_sorted
        inv_order = torch.empty_like(order)
        inv_order[order] = torch.arange(El, device=dev)
        self.sub = sub_canon[order].to(torch.int32).contiguous()
        valid = sub_canon < L
        del sub, sub_canon
        if El * S >= 2 ** 31:
            raise ConfigError("HybridSchwarz: E * S exceeds int32 slot indexing; partition the mesh")

        def flat_pos(vi_):
            """canonical (subdomain, slot) flat index -> row of the class-ordered sol"""
            return inv_order[vi_ // S] * S + vi_ % S

        # ---- overlap accumulation: node -> (global subdomain, slot), ascending
        #      subdomain; on several ranks the other ranks' solutions on this rank's
        #      gids arrive through an exchange (plan "sol")
        vi = torch.nonzero(valid.view(-1)).view(-1)
        nsub = self.sub.view(-1)[flat_pos(vi)].long()
        gsub = vi // S + e0                                     # global subdomain id
        ent_node, ent_sub, ent_pos = [nsub], [gsub], [flat_pos(vi)]
        n_sol = El * S
        self.plan_sol = None
        gid_of_node = torch.empty(L, dtype=torch.int64, device=dev)
        gid_of_node[loc_rank] = loc_nodes
        gid_of_node[Lloc:] = rem
        if W > 1:
            has = torch.zeros((W, L + 2), dtype=torch.bool, device=dev)
            for q in range(W):
                has[q, gidn_X[owner_X == q].reshape(-1)] = True
            send_meta, send_flat = {}, {}
            for q in range(W):
                if q == rk:
                    continue
                m_ = has[q][nsub]
                if not bool(m_.any()):
                    continue
                gq, sq, fq = gid_of_node[nsub[m_]], gsub[m_], flat_pos(vi[m_])
                o = _lexsort2(gq, sq)
                send_meta[q] = torch.stack([gq[o], sq[o]], dim=1)
                send_flat[q] = fq[o]
            recv_meta = _alltoallv(comm, send_meta, 2, torch.int64, dev)
            self.plan_sol = _Plan(send_flat, {q: t.shape[0] for q, t in recv_meta.items()}, dev)
            for q, t in recv_meta.items():
                nd = node_of(t[:, 0], L)
                if bool((nd >= Lloc).any()):
                    raise ConfigError("HybridSchwarz: a received solution names a gid this rank does not hold")
                ent_node.append(nd)
                ent_sub.append(t[:, 1])
                ent_pos.append(n_sol + self.plan_sol.recv_off[q] + torch.arange(t.shape[0], device=dev))
            del has
        en, es, ep = torch.cat(ent_node), torch.cat(ent_sub), torch.cat(ent_pos)
        keep_e = en < Lloc
        en, es, ep = en[keep_e], es[keep_e], ep[keep_e]
        o = _lexsort2(en, es)
        if int(ep.max()) >= 2 ** 31 if ep.numel() else False:
            raise ConfigError("HybridSchwarz: solution slots exceed int32 indexing")
        self.acc_pos = ep[o].to(torch.int32).contiguous()
        cnt = torch.bincount(en, minlength=Lloc)
        self.acc_off = torch.zeros(Lloc + 1, dtype=torch.int64, device=dev)
        self.acc_off[1:] = torch.cumsum(cnt, 0)
        # 1/sqrt of the (small integer) overlap counts from a host table: IEEE sqrt
        # as numpy computes it (torch's CPU sqrt is not always correctly rounded)
        tab = 1.0 / np.sqrt(np.arange(1, int(cnt.max()) + 2, dtype=np.float64))
        self.wsqrt = torch.as_tensor(tab, device=dev)[cnt - 1].contiguous()      # every node is covered
        del vi, nsub, gsub, ent_node, ent_sub, ent_pos, en, es, ep, valid

        # ---- layer residuals from the other ranks (plan "layer"): rw of the
        #      remote-only nodes, provider by provider
        self.plan_layer = None
        if W > 1:
            req = {q: rem[prov == q].view(-1, 1) for q in range(W) if q != rk}
            asked = _alltoallv(comm, req, 1, torch.int64, dev)
            send = {}
            for q, t in asked.items():
                nd = node_of(t.view(-1), L)
                if bool((nd >= Lloc).any()):
                    raise ConfigError("HybridSchwarz: a peer asked for a gid this rank does not hold")
                send[q] = nd
            self.plan_layer = _Plan(send, {q: int((prov == q).sum()) for q in range(W) if q != rk}, dev)

        # ---- coarse space: one dof per vertex, trilinear embedding (:180-236)
        pts = torch.as_tensor(np.array(space.basis.points, dtype=np.float64), device=dev)
        phi = torch.stack([(1.0 - pts) / 2.0, (1.0 + pts) / 2.0])
        tw = torch.empty((nn, 8), dtype=torch.float64, device=dev)
        for c in range(8):
            tw[:, c] = (phi[c & 1].view(n, 1, 1) * phi[(c >> 1) & 1].view(1, n, 1)
                        * phi[(c >> 2) & 1].view(1, 1, n)).reshape(-1)
        self.tw = tw.contiguous()
        loc_el = elements[e0:e1]
        # first own copy of every own node; owned = the global first copy is here
        lnode = gidn_X[i0:i0 + El].reshape(-1)
        self.first = torch.full((Lloc,), P, dtype=torch.int64, device=dev)
        self.first.scatter_reduce_(0, lnode, torch.arange(P, device=dev), reduce="amin")
        gflat = (gx.view(NX, 1) * nn + torch.arange(nn, device=dev).view(1, nn)).reshape(-1)
        gfirst = torch.full((L + 2,), BIG, dtype=torch.int64, device=dev)
        gfirst.scatter_reduce_(0, gidn_X.reshape(-1), gflat, reduce="amin")
        owned = gfirst[:Lloc] == self.first + e0 * nn
        del gflat, gfirst
        cv, cc = torch.sort(loc_el, dim=1)
        self.cvert = cv.to(torch.int32).contiguous()
        self.ccorn = cc.to(torch.uint8).contiguous()
        # restriction rc = P^T rg (csrc/schwarz.cu): per element, the points that
        # carry their gid's owned first copy add tw[p, c] rg to corner c; per
        # vertex, the (element, corner) sums in ascending element order
        pts = torch.arange(P, device=dev)
        self.rflag = ((self.first[lnode] == pts) & owned[lnode]).to(torch.uint8).contiguous()
        vv = loc_el.reshape(-1)
        o = torch.sort(vv, stable=True).indices
        self.pt_ent = o.contiguous()                          # = element * 8 + corner
        self.pt_ptr = torch.zeros(nv + 1, dtype=torch.int64, device=dev)
        self.pt_ptr[1:] = torch.cumsum(torch.bincount(vv, minlength=nv), 0)
        del pts, vv, o
        # vertex blocks t^T A_e t of this rank's elements, summed per (i, j) in
        # element order; across ranks the partial sums add in rank order
        lcls = ecls[i0:i0 + El]
        ucls = torch.unique(lcls)
        em = element_matrices(space, lam_visc, lam_mass, elems=erep[ucls], geom=geom_X, bm=bm_X)
        blocks_c = tw.T.unsqueeze(0) @ em @ tw.unsqueeze(0)                     # (nc, 8, 8)
        del em
        cslot = torch.full((int(erep.numel()),), -1, dtype=torch.int64, device=dev)
        cslot[ucls] = torch.arange(ucls.numel(), device=dev)
        bl = blocks_c[cslot[lcls]]                                              # (El, 8, 8)
        ri = loc_el.view(El, 8, 1).expand(El, 8, 8).reshape(-1)
        ci = loc_el.view(El, 1, 8).expand(El, 8, 8).reshape(-1)
        kv, vs = _segment_sums(ri * nv + ci, bl.reshape(-1))
        corners_loc = torch.tensor([((c & 1) * (n - 1) * n + ((c >> 1) & 1) * (n - 1)) * n + ((c >> 2) & 1) * (n - 1)
                                    for c in range(8)], device=dev)
        vfixed = torch.zeros(nv, dtype=torch.bool, device=dev)
        vfixed[loc_el[constrained[gidn_X[i0:i0 + El][:, corners_loc]]]] = True
        if W > 1:
            from .partition import all_gather_cat

            cnts = all_gather_cat(comm, torch.tensor([kv.numel()], dtype=torch.int64, device=dev)).cpu()
            mx = int(cnts.max())
            pk = torch.full((mx,), -1, dtype=torch.int64, device=dev)
            pv = torch.zeros(mx, dtype=torch.float64, device=dev)
            pk[:kv.numel()], pv[:vs.numel()] = kv, vs
            ak, av = all_gather_cat(comm, pk), all_gather_cat(comm, pv)
            okk = ak >= 0
            kv, vs = _segment_sums(ak[okk], av[okk])                    # rank order = element order
            vfixed = all_gather_cat(comm, vfixed.to(torch.int32)).view(W, nv).amax(dim=0) > 0
        krow, kcol = kv // nv, kv % nv
        fr, fcn = vfixed[krow], vfixed[kcol]
        val = torch.where(fr | fcn, torch.zeros_like(vs), vs)
        val = torch.where(fr & (krow == kcol), torch.ones_like(val), val)
        diag = torch.zeros(nv, dtype=torch.float64, device=dev)
        dm = krow == kcol
        diag[krow[dm]] = val[dm]
        dc = torch.where(diag <= 0.0, torch.ones_like(diag), diag)
        self.coarse_inv_diag = (1.0 / dc).contiguous()
        rcnt = torch.bincount(krow, minlength=nv)
        width = int(rcnt.max())
        rstart = torch.zeros(nv + 1, dtype=torch.int64, device=dev)
        rstart[1:] = torch.cumsum(rcnt, 0)
        slot = torch.arange(kv.numel(), device=dev) - rstart[krow]
        self.ac_col = torch.arange(nv, device=dev, dtype=torch.int32).view(nv, 1).repeat(1, width).contiguous()
        self.ac_val = torch.zeros((nv, width), dtype=torch.float64, device=dev)
        self.ac_col[krow, slot] = kcol.to(torch.int32)
        self.ac_val[krow, slot] = val
        self.vfixed = vfixed.to(torch.uint8).contiguous()
        self.constrained = constrained[:Lloc].to(torch.uint8).contiguous()
        self.nv = nv
        self.gid = lnode.contiguous()                            # node of every own point
        self.gid_of_node = gid_of_node

        # ---- work buffers, the exchanges (N > 1) and the C struct
        f64 = lambda k: torch.zeros(k, dtype=torch.float64, device=dev)
        self.rg, self.rw = f64(Lloc), f64(L + 1)                # rw[L] = 0: the padding slot
        self.rc_part = f64(nv)
        self.rc = self.rc_part if W == 1 else f64(nv)
        self.xc, self.cr, self.cz, self.cp, self.cap = (f64(nv) for _ in range(5))
        nblk = int(lib.sf_schwarz_coarse_blocks())
        self.cpart = f64(2 * nblk)
        self.cbar = torch.zeros(2, dtype=torch.int32, device=dev)
        self.sol = f64(n_sol)
        self.rwg = f64(n_sol)
        self.se = f64(El * 8)
        self.z = f64(Lloc)
        self.sol_recv = f64(max(self.plan_sol.n_recv_total, 1)) if self.plan_sol is not None else None
        self._ipc = {}
        if W > 1:
            allv = torch.arange(nv, dtype=torch.int32, device=dev)
            self.plan_rc = _Plan({q: allv for q in range(W) if q != rk}, {q: nv for q in range(W) if q != rk}, dev)
            self.rc_recv = f64(max(self.plan_rc.n_recv_total, 1))
            if dev.type == "cuda":
                if comm.peer is None:
                    raise ConfigError("HybridSchwarz across ranks needs the NVLink peer path")
                for name, plan in (("layer", self.plan_layer), ("rc", self.plan_rc), ("sol", self.plan_sol)):
                    self._ipc[name] = _dist.HaloIPC(comm, plan)
        st = _SchwarzStruct()
        pt = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        st.G, st.P, st.nv, st.nnn, st.S = Lloc, P, nv, nn, S
        st.first, st.gid, st.wsqrt, st.rg, st.rw = (pt(t) for t in (self.first, self.gid, self.wsqrt, self.rg,
                                                                      self.rw))
        st.pt_ptr, st.pt_ent, st.tw, st.vfixed = (pt(t) for t in (self.pt_ptr, self.pt_ent, self.tw, self.vfixed))
        st.rc_part, st.rc = pt(self.rc_part), pt(self.rc)
        st.ac_width = width
        st.ac_col, st.ac_val, st.ac_inv_diag = pt(self.ac_col), pt(self.ac_val), pt(self.coarse_inv_diag)
        st.xc, st.cr, st.cz, st.cp, st.cap = (pt(t) for t in (self.xc, self.cr, self.cz, self.cp, self.cap))
        st.cpart, st.cbar = pt(self.cpart), pt(self.cbar)
        st.coarse_iters, st.coarse_blocks = self.coarse_iters, nblk
        st.sub, st.rwg, st.sol = pt(self.sub), pt(self.rwg), pt(self.sol)
        st.sol_recv, st.n_sol = pt(self.sol_recv), n_sol
        st.acc_off, st.acc_pos = pt(self.acc_off), pt(self.acc_pos)
        st.cvert, st.ccorn, st.constrained, st.z = pt(self.cvert), pt(self.ccorn), pt(self.constrained), pt(self.z)
        st.rflag, st.se = pt(self.rflag), pt(self.se)
        st.L = L
        self._st = st
        self.launches = 0

    def _exchange_into(self, name, src, dst):
        """NVLink exchange `name` of src's listed entries; the received values are
        copied (the current inbox bank) to dst."""
        from . import _lib

        ipc = self._ipc[name]
        recv = ipc.exchange(src)
        if recv is not None and ipc.plan.n_recv_total:
            _lib.call("sf_halo_unbank_f64", recv.data_ptr(), recv.seq_ptr, recv.bank, ipc.plan.n_recv_total,
                      _lib.ptr(dst), _lib.stream_ptr(self.space.device))

    @staticmethod
    def _candidates(sub, gid_e, ge_off, ge_e, G, E):
        """Candidate elements of each subdomain row (every element touching one of
        its gids, ascending; -1 padded) and, per candidate, the subdomain slot of
        each of its points (-1 outside): the reference's cand / li / bi
        (precond.py:136-151)."""
        dev = sub.device
        R, S = sub.shape
        nn = gid_e.shape[1]
        ok = sub < G
        row = torch.arange(R, device=dev).view(R, 1).expand(R, S)[ok]
        g = sub[ok]
        cnt = ge_off[g + 1] - ge_off[g]
        rr = torch.repeat_interleave(row, cnt)
        start = torch.repeat_interleave(ge_off[g], cnt)
        within = torch.arange(int(cnt.sum()), device=dev) - torch.repeat_interleave(
            torch.cumsum(cnt, 0) - cnt, cnt)
        ee = ge_e[start + within]
        key = torch.unique(rr * E + ee)
        kr, ke = key // E, key % E
        kc = torch.bincount(kr, minlength=R)
        C = int(kc.max()) if R else 0
        ks = torch.zeros(R + 1, dtype=torch.int64, device=dev)
        ks[1:] = torch.cumsum(kc, 0)
        cand = torch.full((R, C), -1, dtype=torch.int64, device=dev)
        cand[kr, torch.arange(key.numel(), device=dev) - ks[kr]] = ke
        vals = gid_e[cand.clamp(min=0)].view(R, C * nn)
        pos = torch.searchsorted(sub.contiguous(), vals)
        hit = torch.gather(sub, 1, pos.clamp(max=S - 1)) == vals
        bi = torch.where(hit & (cand >= 0).repeat_interleave(nn, dim=1), pos, torch.full_like(pos, -1))
        # canonical slot order = first appearance scanning the candidates in
        # ascending order and their points in local order.  The reference orders
        # a subdomain by gid (space-filling, so translated subdomains of a
        # linspace box order their points differently at ulp-level ties); the
        # canonical order makes equivalent subdomains identical, and the matrix
        # is the reference's up to a symmetric permutation (same entries).
        big = C * nn
        first = torch.full((R, S + 1), big, dtype=torch.int64, device=dev)
        flat = torch.arange(C * nn, device=dev).view(1, -1).expand(R, -1)
        first.scatter_reduce_(1, torch.where(bi >= 0, bi, torch.full_like(bi, S)), flat, reduce="amin")
        order = torch.sort(first[:, :S], dim=1, stable=True).indices        # canonical slot -> sorted slot
        canon = torch.empty_like(order)
        canon.scatter_(1, order, torch.arange(S, device=dev).view(1, S).expand(R, S))
        bi_c = torch.where(bi >= 0, torch.gather(canon, 1, bi.clamp(min=0)), bi)
        sub_c = torch.gather(sub, 1, order)
        return cand, bi_c.view(R, C, nn), sub_c

    def apply_into(self, r, out):
        """out <- M^-1 r (HybridSchwarz.__call__, precond.py:239-250); r, out: fields.
        Stream-ordered, no host synchronisation (capturable in a CUDA graph)."""
        from . import _lib

        st = ctypes.addressof(self._st)
        stream = _lib.stream_ptr(self.space.device)
        comm = self.space.comm
        multi = bool(self._ipc)
        _lib.call("sf_schwarz_gather_f64", st, _lib.ptr(r.contiguous()), stream)
        if multi:
            self._exchange_into("layer", self.rw, self.rw[self.G:])
        _lib.call("sf_schwarz_restrict_f64", st, stream)
        if multi:
            self._exchange_into("rc", self.rc_part, self.rc_recv)
            _lib.call("sf_schwarz_rank_sum_f64", st, _lib.ptr(self.rc_recv), comm.rank, comm.world, stream)
        _lib.call("sf_schwarz_coarse_f64", st, stream)
        _lib.call("sf_schwarz_gather_rw_f64", st, stream)
        S = self.S
        rwg, sol = self.rwg.view(-1, S), self.sol.view(-1, S)
        for c, a, b in self.blocks:                 # one FP64 GEMM per subdomain class
            torch.matmul(rwg[a:b], self.invT[c], out=sol[a:b])
        if multi:
            self._exchange_into("sol", self.sol, self.sol_recv)
        _lib.call("sf_schwarz_finalize_f64", st, stream)
        _lib.call("sf_schwarz_scatter_f64", st, _lib.ptr(out), stream)
        self.launches += 6 + len(self.blocks) + (8 if multi else 0)
        return out

    def __call__(self, r):
        from . import _lib

        _lib.require_cuda(r)
        return self.apply_into(r, torch.empty_like(r))
