"""Mesh validation and the geometric cross-check of the gather-scatter numbering.

Two reference checks, restated as sort/scan passes on the device (setup only):

* :func:`validate_mesh` -- ``Mesh.validate`` (reference mesh.py:95-147): index
  ranges, conformity (a face is owned by one element, exterior, or two,
  interior) and facet tagging (every exterior face tagged once, no interior
  face tagged).  The reference walks a dict of ``frozenset`` face keys in
  element order; here the faces are sorted by their vertex set and the FIRST
  offending face in that dict order is reported, with the reference's message.
* :func:`coincident_pairs` / :func:`reconcile` -- ``_build_gather_scatter``'s
  geometric grouping (space.py:265-314): GLL points closer than
  ``tol = 1e-8 * max element diameter`` are one global node, the union of all
  such pairs (cKDTree ``query_pairs(r=tol)``).  The device builder
  (space.build_gather_scatter) groups points TOPOLOGICALLY (shared vertex ids),
  which equals the geometric grouping on conforming meshes whose coincident
  points share vertex ids.  Here every point is hashed into a uniform grid of
  cells >= tol, the tol-pairs are found among the 14 forward neighbour cells,
  and (1) the reference's ``TopologyError`` cases are raised (two points of one
  element coincide; coincident points in elements sharing no vertex), (2) if any
  pair crosses two topological groups, or a group is not within tol of its
  representative, the groups are recomputed as the connected components of the
  pair graph (label propagation + pointer jumping), i.e. the reference's own
  definition, so the maps are the reference's on every mesh.
"""

import numpy as np
import torch

from .errors import TopologyError

FACE_CORNERS = ((0, 2, 4, 6), (1, 3, 5, 7), (0, 1, 4, 5), (2, 3, 6, 7), (0, 1, 2, 3), (4, 5, 6, 7))


def _t(a, dev, dtype=torch.int64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)


def validate_mesh(mesh, device=None):
    """Raise TopologyError exactly where the reference's Mesh.validate does
    (mesh.py:95-147); returns the mesh."""
    dev = torch.device(device) if device is not None else torch.device("cpu")
    nv = int(mesh.vertices.shape[0])
    E = int(mesh.elements.shape[0])
    el = np.asarray(mesh.elements)
    fe_np, ff_np, ft_np = (np.asarray(a) for a in (mesh.facet_elem, mesh.facet_face, mesh.facet_tag))
    if el.size and (el.min() < 0 or el.max() >= nv):
        raise TopologyError("element vertex index out of range")
    if fe_np.size:
        if fe_np.min() < 0 or fe_np.max() >= E:
            raise TopologyError("facet element index out of range")
        if ff_np.min() < 0 or ff_np.max() > 5:
            raise TopologyError("facet local face index out of range")
        if ft_np.min() < 0 or ft_np.max() >= len(mesh.tag_names):
            raise TopologyError("facet tag index out of range")
    if E:
        elements = _t(el, dev)
        fc = _t(np.array(FACE_CORNERS), dev)
        # face key = the SET of its 4 vertex ids (reference frozenset): sort, blank
        # repeats, sort again so the distinct ids lead
        fv = torch.sort(elements[:, fc.view(-1)].view(E * 6, 4), dim=1).values
        dup = torch.zeros_like(fv, dtype=torch.bool)
        dup[:, 1:] = fv[:, 1:] == fv[:, :-1]
        fv = torch.sort(torch.where(dup, torch.full_like(fv, nv), fv), dim=1).values
        # group equal keys; the dict order of the reference is first occurrence
        o = torch.arange(E * 6, device=dev)
        for c in (3, 2, 1, 0):
            o = o[torch.sort(fv[o, c], stable=True).indices]
        sk = fv[o]
        new = torch.ones(E * 6, dtype=torch.bool, device=dev)
        new[1:] = (sk[1:] != sk[:-1]).any(dim=1)
        grp_sorted = torch.cumsum(new.to(torch.int64), 0) - 1
        G = int(grp_sorted[-1]) + 1
        grp = torch.empty_like(grp_sorted)
        grp[o] = grp_sorted
        cnt = torch.bincount(grp, minlength=G)
        first = torch.full((G,), E * 6, dtype=torch.int64, device=dev)
        first.scatter_reduce_(0, grp, o, reduce="amin")
        # 1. non-conforming: first (dict-order) face owned by more than two elements
        big = cnt > 2
        if bool(big.any()):
            g = int(torch.argmin(torch.where(big, first, torch.full_like(first, E * 6))))
            lst = sorted((int(i) // 6, int(i) % 6) for i in torch.nonzero(grp == g).view(-1).tolist())
            raise TopologyError(f"face shared by {len(lst)} elements (non-conforming): {lst}")
        # 2. a facet tagged twice (the first repeat in facet order)
        ef = fe_np.astype(np.int64) * 6 + ff_np.astype(np.int64)
        if ef.size:
            eft = _t(ef, dev)
            so = torch.sort(eft, stable=True)
            rep = torch.zeros(ef.size, dtype=torch.bool, device=dev)
            rep[so.indices[1:]] = so.values[1:] == so.values[:-1]
            if bool(rep.any()):
                i = int(torch.nonzero(rep)[0])
                raise TopologyError(f"facet ({int(fe_np[i])}, {int(ff_np[i])}) tagged more than once")
        tagged = torch.zeros(E * 6, dtype=torch.bool, device=dev)
        if ef.size:
            tagged[_t(ef, dev)] = True
        # 3. walk the faces in dict order: an untagged exterior face or a tagged
        #    interior face, whichever comes first (mesh.py:125-133)
        ext = cnt[grp] == 1
        bad_face = (ext & ~tagged) | (~ext & tagged)
        if bool(bad_face.any()):
            gbad = torch.zeros(G, dtype=torch.bool, device=dev)
            gbad[grp[bad_face]] = True
            g = int(torch.argmin(torch.where(gbad, first, torch.full_like(first, E * 6))))
            members = torch.nonzero(grp == g).view(-1).tolist()    # ascending = list order
            if len(members) == 1:
                i = members[0]
                raise TopologyError(f"exterior face {(i // 6, i % 6)} carries no boundary tag")
            for i in members:
                if bool(tagged[i]):
                    raise TopologyError(f"interior face {(i // 6, i % 6)} carries a boundary tag")
    curved = np.asarray(getattr(mesh, "curved_elem", np.zeros(0)))
    if curved.size:
        if mesh.geom_order is None:
            raise TopologyError("curved records present but geom_order unset")
        ng1 = mesh.geom_order + 1
        if tuple(mesh.curved_coords.shape) != (curved.size, ng1, ng1, ng1, 3):
            raise TopologyError("curved_coords shape inconsistent with geom_order")
        if curved.min() < 0 or curved.max() >= E:
            raise TopologyError("curved element index out of range")
    return mesh


def gs_tolerance(mesh):
    """tol = 1e-8 * max element corner-box diagonal (space.py:268-271), host numpy
    arithmetic as in the reference."""
    corner = np.asarray(mesh.vertices)[np.asarray(mesh.elements)]
    if corner.shape[0] == 0:
        return 0.0
    diam = np.linalg.norm(corner.max(axis=1) - corner.min(axis=1), axis=1)
    return 1e-8 * float(diam.max())


# 13 forward neighbour offsets (plus the own cell, handled separately): each
# unordered pair of cells is visited once
_FWD = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
        if (dx, dy, dz) > (0, 0, 0)]


def coincident_pairs(coords, tol, chunk=1 << 24):
    """All pairs (i < j) of local points with |x_i - x_j| <= tol (the reference's
    cKDTree.query_pairs(r=tol) set, unordered), as a (K, 2) int64 device tensor."""
    dev = coords.device
    pts = coords.reshape(3, -1)
    P = pts.shape[1]
    if P < 2 or tol <= 0.0:
        return torch.zeros((0, 2), dtype=torch.int64, device=dev)
    lo = pts.min(dim=1).values
    ext = (pts.max(dim=1).values - lo).cpu().numpy()
    # cell size >= tol, grown until the cell grid index fits 62 bits
    h = float(tol)
    while np.prod(np.floor(ext / h) + 3.0) >= 2.0 ** 62:
        h *= 2.0
    dims = [int(np.floor(e / h)) + 3 for e in ext]
    cell = torch.floor((pts - lo.view(3, 1)) / h).to(torch.int64) + 1         # (3, P), >= 1
    key = (cell[0] * dims[1] + cell[1]) * dims[2] + cell[2]
    del cell
    skey, order = torch.sort(key)
    del key
    spts = pts[:, order]
    out = []
    offs = [0] + [(dx * dims[1] + dy) * dims[2] + dz for dx, dy, dz in _FWD]
    tol2 = tol * tol
    for c0 in range(0, P, chunk):
        c1 = min(P, c0 + chunk)
        kq = skey[c0:c1]
        xq = spts[:, c0:c1]
        iq = torch.arange(c0, c1, device=dev)
        for off in offs:
            kk = kq + off
            a = torch.searchsorted(skey, kk, side="left")
            b = torch.searchsorted(skey, kk, side="right")
            if off == 0:
                a = iq + 1           # own cell: only later entries (each pair once)
            n = (b - a).clamp_min(0)
            m = int(n.max()) if n.numel() else 0
            for j in range(m):
                sel = torch.nonzero(n > j).view(-1)
                if sel.numel() == 0:
                    break
                cand = a[sel] + j
                d = spts[:, cand] - xq[:, sel]
                close = (d * d).sum(0).sqrt() <= tol
                if bool(close.any()):
                    s = sel[close]
                    out.append(torch.stack([order[c0 + s], order[cand[close]]], dim=1))
    if not out:
        return torch.zeros((0, 2), dtype=torch.int64, device=dev)
    pr = torch.cat(out)
    return torch.stack([pr.min(dim=1).values, pr.max(dim=1).values], dim=1)


def check_pairs(pairs, elements, nnn, tol):
    """The reference's TopologyError checks on the coincident pairs (space.py:274-291)."""
    if pairs.numel() == 0:
        return
    ep = pairs[:, 0] // nnn
    eq = pairs[:, 1] // nnn
    same = ep == eq
    if bool(same.any()):
        k = int(torch.nonzero(same)[0])
        p = pairs[k].tolist()
        raise TopologyError(
            f"two GLL points of element {int(ep[k])} coincide within tolerance {tol:.3e} "
            f"(degenerate element?): local points {p}")
    va = elements[ep]                       # (K, 8)
    vb = elements[eq]
    share = (va.unsqueeze(2) == vb.unsqueeze(1)).flatten(1).any(dim=1)
    if not bool(share.all()):
        k = int(torch.nonzero(~share)[0])
        raise TopologyError(
            f"coincident points in non-adjacent elements {int(ep[k])} and {int(eq[k])} "
            f"(tolerance {tol:.3e})")


def components(pairs, P):
    """Connected components of the pair graph on P points: group label = lowest
    point index of the component (label propagation + pointer jumping)."""
    dev = pairs.device
    lab = torch.arange(P, device=dev)
    if pairs.numel() == 0:
        return lab
    i, j = pairs[:, 0], pairs[:, 1]
    while True:
        m = torch.minimum(lab[i], lab[j])
        new = lab.clone()
        new.scatter_reduce_(0, i, m, reduce="amin")
        new.scatter_reduce_(0, j, m, reduce="amin")
        while True:                      # pointer jumping to the current roots
            nxt = new[new]
            if torch.equal(nxt, new):
                break
            new = nxt
        if torch.equal(new, lab):
            return lab
        lab = new


def topology_agrees(gid, pairs, coords, tol):
    """True when the topological groups ARE the tol-graph components: no pair
    joins two groups and every copy lies within tol of its group's lowest copy."""
    if pairs.numel() and bool((gid[pairs[:, 0]] != gid[pairs[:, 1]]).any()):
        return False
    P = gid.numel()
    n_g = int(gid.max()) + 1 if P else 0
    rep = torch.full((n_g,), P, dtype=torch.int64, device=gid.device)
    rep.scatter_reduce_(0, gid, torch.arange(P, device=gid.device), reduce="amin")
    pts = coords.reshape(3, -1)
    d = pts - pts[:, rep[gid]]
    return bool(((d * d).sum(0).sqrt() <= tol).all())
