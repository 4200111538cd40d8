"""Preconditioners on device: block Jacobi (reference precond.py:27-59) and the
hybrid overlapping Schwarz method (precond.py:94-250).
"""

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
    diag = torch.zeros(space.shape, dtype=torch.float64, device=space.device)
    for m in range(n):        # einsum("mi,emjk->eijk", d2, g0)
        diag = diag + d2[m].view(1, n, 1, 1) * g[0][:, m:m + 1, :, :]
    t = torch.zeros_like(diag)
    for m in range(n):        # einsum("mj,eimk->eijk", d2, g3)
        t = t + d2[m].view(1, 1, n, 1) * g[3][:, :, m:m + 1, :]
    diag = diag + t
    t = torch.zeros_like(diag)
    for m in range(n):        # einsum("mk,eijm->eijk", d2, g5)
        t = t + d2[m].view(1, 1, 1, n) * g[5][:, :, :, m:m + 1]
    diag = diag + t
    di = dd.view(1, n, 1, 1)
    dj = dd.view(1, 1, n, 1)
    dk = dd.view(1, 1, 1, n)
    diag = diag + ((2.0 * g[1]) * di) * dj
    diag = diag + ((2.0 * g[2]) * di) * dk
    diag = diag + ((2.0 * g[4]) * dj) * dk
    diag = lam_visc * diag + lam_mass * space.bm
    return space.gs.add(diag)


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


def element_matrices(space, lam_visc, lam_mass, batch=64):
    """Dense element matrices A_e (E, n^3, n^3) on the device: the identity basis
    pushed through the element kernel with the element's metric replicated
    (precond.py:71-91) -- the same arithmetic as the matrix-free operator."""
    from . import _lib
    from .operators import _ex

    n, E = space.n, space.n_elements
    nn = n ** 3
    dev = space.device
    mats = torch.empty((E, nn, nn), dtype=torch.float64, device=dev)
    eye = torch.eye(nn, dtype=torch.float64, device=dev)
    for e0 in range(0, E, batch):
        e1 = min(E, e0 + batch)
        B = e1 - e0
        g = space.geom.view(6, E, nn)[:, e0:e1].repeat_interleave(nn, dim=1).contiguous()
        bm = space.bm.view(E, nn)[e0:e1].repeat_interleave(nn, dim=0).contiguous()
        u = eye.repeat(B, 1).contiguous()
        w = torch.empty_like(u)
        _lib.call("sf_ax_helm_f64", space.dmat.ctypes.data, n, _lib.ptr(g), _lib.ptr(bm), _lib.ptr(u), _lib.ptr(w),
                  B * nn, float(lam_visc), float(lam_mass), _ex(), _lib.stream_ptr(dev))
        mats[e0:e1] = w.view(B, nn, nn).transpose(1, 2)
    return mats


class HybridSchwarz:
    """Overlapping Schwarz subdomain solves plus a trilinear coarse solve
    (precond.py:94-250), on the device.

    Subdomain e = element e's global ids plus the first GLL layer inside each
    face neighbour; its matrix is assembled from the dense element matrices of
    every element touching it (candidates added in ascending order, as the
    reference does), Dirichlet rows/columns replaced by identity, and LU-factored
    as one padded batch (torch.linalg.lu_factor).  An application gathers one
    value per global id, solves all subdomains in one batched triangular solve,
    accumulates the overlapping corrections in ascending subdomain order
    (deterministic, no atomics), adds the coarse correction from a fixed number
    of Jacobi-CG iterations on the assembled vertex problem, and scatters back.
    Results agree with the reference to rounding (LU pivoting and the element
    matrices' summation order differ at the last bit).  Single-rank only; the
    memory is the reference's O(E (n^3 + 6 n^2)^2).
    """

    def __init__(self, space, mask=None, lam_visc=1.0, lam_mass=0.0, coarse_iters=10):
        from .errors import ConfigError
        from .mesh import FACE_CORNERS

        gs = space.gs
        if space.comm.world > 1:
            raise ConfigError("the hybrid Schwarz preconditioner is single-rank on the device path")
        self.space = space
        self.coarse_iters = int(coarse_iters)
        dev = space.device
        n, E = space.n, space.n_elements
        nn = n ** 3
        G = gs.n_gid
        gid_e = gs.gid.view(E, nn).cpu().numpy()
        constrained = np.zeros(G, dtype=bool)
        if mask is not None:
            m = torch.as_tensor(mask, dtype=torch.float64, device=dev).reshape(-1).cpu().numpy()
            constrained[gs.gid.cpu().numpy()[m == 0.0]] = True
        mats = element_matrices(space, lam_visc, lam_mass)

        mesh = space.mesh
        faces = {}
        for e in range(E):
            for f, corners in enumerate(FACE_CORNERS):
                faces.setdefault(frozenset(int(mesh.elements[e, c]) for c in corners), []).append((e, f))
        neighbors = [[] for _ in range(E)]
        for pairs in faces.values():
            if len(pairs) == 2:
                (e0, f0), (e1, f1) = pairs
                neighbors[e0].append((e1, f1))
                neighbors[e1].append((e0, f0))
        layer = [_face_layer(n, f) for f in range(6)]
        # elements touching each gid, ascending
        order = np.argsort(gid_e.ravel(), kind="stable")
        g_sorted = gid_e.ravel()[order]
        e_sorted = order // nn
        starts = np.searchsorted(g_sorted, np.arange(G + 1))

        subs = []
        for e in range(E):
            parts = [gid_e[e]] + [gid_e[e2][layer[f2]] for e2, f2 in neighbors[e]]
            subs.append(np.unique(np.concatenate(parts)))
        S = max(s.size for s in subs)
        self.S = S
        overlap = np.zeros(G)
        for s in subs:
            overlap[s] += 1.0

        # assembly by candidate rank: pass k adds every subdomain's k-th candidate
        cands = []
        for e, s in enumerate(subs):
            cs = np.unique(np.concatenate([e_sorted[starts[g]:starts[g + 1]] for g in s]))
            cands.append(cs)
        A = torch.zeros((E, S + 1, S + 1), dtype=torch.float64, device=dev)   # slot S: padding sink
        kmax = max(c.size for c in cands)
        for k in range(kmax):
            es = [e for e in range(E) if cands[e].size > k]
            li_l, bi_l = [], []
            for e in es:
                e2 = cands[e][k]
                s = subs[e]
                pos = np.searchsorted(s, gid_e[e2])
                inside = s[np.minimum(pos, s.size - 1)] == gid_e[e2]
                li_l.append(np.nonzero(inside)[0])
                bi_l.append(pos[inside])
            L = max(x.size for x in li_l)
            li = np.zeros((len(es), L), dtype=np.int64)
            bi = np.full((len(es), L), S, dtype=np.int64)
            valid = np.zeros((len(es), L), dtype=bool)
            for r, (a_, b_) in enumerate(zip(li_l, bi_l)):
                li[r, :a_.size], bi[r, :b_.size], valid[r, :a_.size] = a_, b_, True
            e2s = torch.as_tensor([cands[e][k] for e in es], device=dev)
            li_t = torch.as_tensor(li, device=dev)
            bi_t = torch.as_tensor(bi, device=dev)
            vm = torch.as_tensor(valid, device=dev)
            blk = mats[e2s[:, None, None], li_t[:, :, None], li_t[:, None, :]]
            blk = torch.where(vm[:, :, None] & vm[:, None, :], blk, torch.zeros_like(blk))
            A.index_put_((torch.as_tensor(es, device=dev)[:, None, None], bi_t[:, :, None], bi_t[:, None, :]),
                          blk, accumulate=True)
            del blk
        A = A[:, :S, :S].contiguous()
        ar = torch.arange(S, device=dev)
        for e, s in enumerate(subs):
            fixed = np.nonzero(constrained[s])[0]
            if fixed.size:
                fx = torch.as_tensor(fixed, device=dev)
                A[e, fx, :] = 0.0
                A[e, :, fx] = 0.0
                A[e, fx, fx] = 1.0
            elif s.size == G:
                bmg = gs.gather_unique(gs.add(space.bm))
                A[e, ar[:s.size], ar[:s.size]] += 1e-8 * bmg[torch.as_tensor(s, device=dev)]
            if s.size < S:
                A[e, s.size:, s.size:] = torch.eye(S - s.size, dtype=torch.float64, device=dev)
        self.lu, self.piv = torch.linalg.lu_factor(A)
        del A
        sub_pad = np.full((E, S), G, dtype=np.int64)          # index G: a zero right-hand side
        for e, s in enumerate(subs):
            sub_pad[e, :s.size] = s
        self.sub_pad = torch.as_tensor(sub_pad, device=dev)
        # accumulation passes: contribution (e, i) goes to pass = rank of e among
        # the subdomains holding that gid, so each pass has no repeated target
        flat_g = sub_pad.ravel()
        ok = flat_g < G
        fe = np.repeat(np.arange(E), S)[ok]
        fg = flat_g[ok]
        fpos = np.nonzero(ok)[0]
        o = np.lexsort((fe, fg))
        fg_s = fg[o]
        first = np.r_[True, fg_s[1:] != fg_s[:-1]]
        grp = np.cumsum(first) - 1
        rank = np.arange(fg_s.size) - np.nonzero(first)[0][grp]
        self.passes = []
        for r in range(int(rank.max()) + 1 if rank.size else 0):
            sel = o[rank == r]
            self.passes.append((torch.as_tensor(fpos[sel], device=dev), torch.as_tensor(fg[sel], device=dev)))
        self.wsqrt = torch.as_tensor(1.0 / np.sqrt(overlap), device=dev)
        self.constrained = torch.as_tensor(constrained, device=dev)

        # coarse space: one dof per mesh vertex, trilinear embedding
        pts = space.basis.points
        phi = np.stack([(1.0 - pts) / 2.0, (1.0 + pts) / 2.0])
        t = np.empty((nn, 8))
        for c in range(8):
            t[:, c] = (phi[c & 1][:, None, None] * phi[(c >> 1) & 1][None, :, None]
                       * phi[(c >> 2) & 1][None, None, :]).ravel()
        nv = mesh.vertices.shape[0]
        tt = torch.as_tensor(t, device=dev)
        blocks = (tt.T.unsqueeze(0) @ mats @ tt.unsqueeze(0)).cpu().numpy()     # (E, 8, 8)
        del mats
        ac = np.zeros((nv, nv))
        for e in range(E):
            verts = mesh.elements[e]
            ac[np.ix_(verts, verts)] += blocks[e]
        rows = np.repeat(gid_e.reshape(-1), 8)
        cols = np.repeat(mesh.elements[:, None, :], nn, axis=1).reshape(-1)
        vals = np.tile(t.ravel(), E)
        key = rows.astype(np.int64) * np.int64(nv) + cols
        _, firsti = np.unique(key, return_index=True)
        r_, c_, v_ = rows[firsti], cols[firsti], vals[firsti]
        # the sparse embedding as padded row lists (deterministic fixed-order sums;
        # library SpMV may reduce in a run-dependent order)
        self.P_idx, self.P_val = self._padded_rows(r_, c_, v_, G, dev)
        self.PT_idx, self.PT_val = self._padded_rows(c_, r_, v_, nv, dev)
        vfixed = np.zeros(nv, dtype=bool)
        for e in range(E):
            for c in range(8):
                i, j, k = (c & 1) * (n - 1), ((c >> 1) & 1) * (n - 1), ((c >> 2) & 1) * (n - 1)
                if constrained[gid_e[e, (i * n + j) * n + k]]:
                    vfixed[mesh.elements[e, c]] = True
        if vfixed.any():
            ac[vfixed, :] = 0.0
            ac[:, vfixed] = 0.0
            ac[vfixed, vfixed] = 1.0
        dc = np.diag(ac).copy()
        dc[dc <= 0.0] = 1.0
        self.a_coarse = torch.as_tensor(ac, device=dev)
        self.coarse_inv_diag = torch.as_tensor(1.0 / dc, device=dev)
        self.v_fixed = torch.as_tensor(vfixed, device=dev)
        self.G = G

    @staticmethod
    def _padded_rows(rows, cols, vals, nrows, dev):
        """(nrows, width) column indices / values of a sparse matrix, rows padded
        with weight 0 (column order ascending within a row)."""
        o = np.lexsort((cols, rows))
        rows, cols, vals = rows[o], cols[o], vals[o]
        cnt = np.bincount(rows, minlength=nrows)
        width = max(1, int(cnt.max()) if cnt.size else 1)
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        slot = np.arange(rows.size) - start[rows]
        idx = np.zeros((nrows, width), dtype=np.int64)
        val = np.zeros((nrows, width))
        idx[rows, slot] = cols
        val[rows, slot] = vals
        return torch.as_tensor(idx, device=dev), torch.as_tensor(val, device=dev)

    @staticmethod
    def _spmv(idx, val, x):
        return (val * x[idx]).sum(dim=1)

    def _coarse_solve(self, rc):
        """Fixed-iteration Jacobi-CG on the vertex problem from zero (precond.py:205-230)."""
        x = torch.zeros_like(rc)
        r = rc.clone()
        z = self.coarse_inv_diag * r
        p = z.clone()
        rz = float(torch.dot(r, z))
        if rz <= 0.0:
            return x
        for _ in range(self.coarse_iters):
            ap = self.a_coarse @ p
            pap = float(torch.dot(p, ap))
            if pap <= 0.0:
                break
            alpha = rz / pap
            x += alpha * p
            r -= alpha * ap
            z = self.coarse_inv_diag * r
            rz_new = float(torch.dot(r, z))
            if rz_new <= 0.0:
                break
            p = z + (rz_new / rz) * p
            rz = rz_new
        return x

    def __call__(self, r):
        gs = self.space.gs
        rg = gs.gather_unique(r)
        rw = torch.cat([self.wsqrt * rg, rg.new_zeros(1)])
        sol = torch.linalg.lu_solve(self.lu, self.piv, rw[self.sub_pad].unsqueeze(-1)).squeeze(-1).reshape(-1)
        z = torch.zeros_like(rg)
        for pos, g in self.passes:
            z.index_add_(0, g, sol[pos])
        z *= self.wsqrt
        rc = self._spmv(self.PT_idx, self.PT_val, rg)
        rc[self.v_fixed] = 0.0
        z += self._spmv(self.P_idx, self.P_val, self._coarse_solve(rc))
        z[self.constrained] = rg[self.constrained]
        return gs.scatter_unique(z, r.shape)
