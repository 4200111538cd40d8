"""Partitioned gather-scatter construction (partition.py) against the global
build, on CPU over gloo: every rank builds only its element range's numbering
and halo plan, and must get exactly what the global build gives it
(dist.build_halo_plan over the reference-order global maps) -- gid slice,
multiplicities, shared maps, send lists and receive counts, and the
gather_unique / scatter_unique helpers -- on a perturbed
box (2, 3, 4 and 8 ranks) and on the curved cylinder mini-rotor mesh (2, 3, 4).
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, payload, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2207_07098_b200 import partition
        from paper_2207_07098_b200.dist import Comm, build_halo_plan, element_ranges

        elements, coords, n, nv, gid, perm, off = payload
        comm = Comm()
        E = elements.shape[0]
        starts = element_ranges(E, world)
        e0, e1 = starts[rank], starts[rank + 1]
        g_loc, plan, mult8, n_gid = partition.partitioned_numbering(
            elements, coords[:, e0:e1].contiguous(), n, comm, starts, nv)
        nnn = n ** 3
        ref = build_halo_plan(gid, perm, off, starts, rank, nnn)
        counts = off[1:] - off[:-1]
        g_ref = gid[e0 * nnn:e1 * nnn]
        ok = {
            "gid": bool(torch.equal(g_loc, g_ref)),
            "n_gid": n_gid == int(off.numel() - 1),
            "mult": bool(torch.equal(mult8.long(), counts[g_ref])),
            "sh_off": bool(torch.equal(plan.sh_off, ref.sh_off)),
            "sh_perm": bool(torch.equal(plan.sh_perm, ref.sh_perm)),
            "peers": plan.peers == ref.peers,
            "n_recv": plan.n_recv == ref.n_recv,
            "send": all(torch.equal(plan.send_idx[p], ref.send_idx[p]) for p in ref.send_idx)
            and set(plan.send_idx) == set(ref.send_idx),
        }
        # gather_unique / scatter_unique on the partitioned space (space.py:62-70):
        # the reference's first-copy values, every rank the whole vector, bitwise
        from paper_2207_07098_b200.space import GatherScatter

        gsp = GatherScatter(g_loc, None, None, (e1 - e0, n, n, n), comm=comm, starts=starts, plan=plan,
                            mult8=mult8, n_gid=n_gid)
        u_full = torch.randn(E * nnn, generator=torch.Generator().manual_seed(7), dtype=torch.float64)
        u_full[::5] = -0.0
        want = u_full[perm[off[:-1]]]
        got = gsp.gather_unique(u_full[e0 * nnn:e1 * nnn].view(e1 - e0, n, n, n))
        ok["gather_unique"] = bool(torch.equal(got.view(torch.int64), want.view(torch.int64)))
        ok["scatter_unique"] = bool(torch.equal(gsp.scatter_unique(want, (e1 - e0, n, n, n)).reshape(-1),
                                                want[gid[e0 * nnn:e1 * nnn]]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _box(oracle):
    m = oracle.gen_box_mesh((0.0, 1.0, 0.0, 1.3, 0.0, 0.9), (3, 4, 5))
    rng = np.random.default_rng(3)
    v = m.vertices
    inner = np.all((v > 1e-9) & (v < np.array([1.0, 1.3, 0.9]) - 1e-9), axis=1)
    v[inner] += 0.05 * rng.uniform(-1, 1, (int(inner.sum()), 3))
    return m, 4


def _rotor():
    from conftest import load_npz, mesh_from_golden

    return mesh_from_golden(load_npz("spaces.npz"), "rotor"), 5


@pytest.mark.parametrize("world,case", [(2, "box"), (3, "box"), (4, "box"), (8, "box"),
                                        (2, "rotor"), (3, "rotor"), (4, "rotor")])
def test_partitioned_numbering_equals_global(oracle, world, case):
    mesh, order = _box(oracle) if case == "box" else _rotor()
    osp = oracle.build_space(mesh, oracle.make_basis(order))
    g = osp.gs
    payload = (torch.from_numpy(np.ascontiguousarray(mesh.elements, dtype=np.int64)),
               torch.from_numpy(np.ascontiguousarray(osp.coords)), osp.n, int(mesh.vertices.shape[0]),
               torch.from_numpy(g.gid), torch.from_numpy(g.perm), torch.from_numpy(g.offsets))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, payload, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, ok = q.get(timeout=300)
        res[r] = ok
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert all(res[r].values()), (r, res[r])
