"""Multi-rank host logic on CPU: halo plans, exchange over gloo, deterministic reductions.

The partitioned dssum must be bitwise identical to the single-rank (reference)
dssum for every rank count: each rank sums all copies of an interface gid in
global order from its own values plus the raw values received from its peers.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_07098_b200.dist import Comm, build_halo_plan, dssum_reference_cpu, element_ranges


def _space(oracle, counts=(3, 4, 5), order=4, perturb=True):
    m = oracle.gen_box_mesh((0.0, 1.0, 0.0, 1.3, 0.0, 0.9), counts)
    if perturb:
        rng = np.random.default_rng(3)
        v = m.vertices
        inner = np.all((v > 1e-9) & (v < np.array([1.0, 1.3, 0.9]) - 1e-9), axis=1)
        v[inner] += 0.05 * rng.uniform(-1, 1, (int(inner.sum()), 3))
    return oracle.build_space(m, oracle.make_basis(order))


@pytest.mark.parametrize("world", [2, 3, 5, 8])
@pytest.mark.parametrize("mode", [0, 1])
def test_partitioned_dssum_is_bitwise_single_rank(oracle, world, mode):
    sp = _space(oracle)
    E = sp.shape[0]
    nnn = sp.n ** 3
    gs = sp.gs
    u = np.random.default_rng(7).standard_normal(E * nnn)
    want = (gs.add if mode == 0 else gs.avg)(u.reshape(sp.shape)).reshape(-1)
    starts = element_ranges(E, world)
    gid, perm, off = (torch.from_numpy(a) for a in (gs.gid, gs.perm, gs.offsets))
    plans = [build_halo_plan(gid, perm, off, starts, r, nnn) for r in range(world)]
    parts = [u[starts[r] * nnn:starts[r + 1] * nnn] for r in range(world)]
    outs = dssum_reference_cpu(parts, plans, mode=mode)
    got = np.concatenate(outs)
    assert np.array_equal(got, want)
    # every interface value a rank receives is one it needs; send and receive sizes agree
    for r in range(world):
        for q in plans[r].peers:
            assert plans[r].n_recv[q] == int(plans[q].send_idx[r].numel())


def test_plan_single_rank_has_no_peers(oracle):
    sp = _space(oracle, perturb=False)
    nnn = sp.n ** 3
    gid, perm, off = (torch.from_numpy(a) for a in (sp.gs.gid, sp.gs.perm, sp.gs.offsets))
    plan = build_halo_plan(gid, perm, off, element_ranges(sp.shape[0], 1), 0, nnn)
    assert plan.peers == [] and plan.n_recv_total == 0
    counts = np.diff(sp.gs.offsets)
    assert plan.n_shared == int((counts > 1).sum())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, payload, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gid, perm, off, nnn, u = payload
        E = gid.numel() // nnn
        starts = element_ranges(E, world)
        comm = Comm()
        plan = build_halo_plan(gid, perm, off, starts, rank, nnn)
        v = torch.from_numpy(u[starts[rank] * nnn:starts[rank + 1] * nnn].copy())
        send = {p: v[plan.send_idx[p].long()].clone() for p in plan.send_idx}
        recv = {p: torch.empty(plan.n_recv[p], dtype=torch.float64) for p in plan.n_recv}
        comm.exchange(send, recv)
        rb = np.zeros(plan.n_recv_total)
        for p in plan.peers:
            rb[plan.recv_off[p]:plan.recv_off[p] + plan.n_recv[p]] = recv[p].numpy()
        # the kernel's arithmetic, on the received raw copies
        src = np.concatenate([v.numpy(), rb])
        out = v.numpy().copy()
        so, sperm = plan.sh_off.numpy(), plan.sh_perm.numpy()
        for g in range(plan.n_shared):
            acc = 0.0
            for o in range(so[g], so[g + 1]):
                acc = acc + src[sperm[o]]
            for o in range(so[g], so[g + 1]):
                if sperm[o] < plan.P_loc:
                    out[sperm[o]] = acc
        # deterministic rank-order reduction
        part = torch.tensor([float(rank + 1), 0.5 * rank], dtype=torch.float64)
        comm.sum_(part)
        # checkpoint gather of element slices (uneven ranges)
        n = round(nnn ** (1.0 / 3.0))
        full = torch.from_numpy(np.stack([u, 2.0 * u, -u]).reshape(3, E, n, n, n))
        mine = full[:, starts[rank]:starts[rank + 1]].contiguous()
        got = comm.gather_elements(mine, starts)
        root = comm.gather_to_root(mine, starts)   # checkpoint path: rank 0 only, host numpy
        ok_root = (root is None) if rank else bool(np.array_equal(root, full.numpy()))
        q.put((rank, out, part.numpy(), bool(torch.equal(got, full)) and ok_root))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_halo_exchange(oracle, world):
    sp = _space(oracle, counts=(2, 3, 4), order=3)
    gs = sp.gs
    nnn = sp.n ** 3
    u = np.random.default_rng(11).standard_normal(gs.gid.size)
    want = gs.add(u.reshape(sp.shape)).reshape(-1)
    payload = (torch.from_numpy(gs.gid), torch.from_numpy(gs.perm), torch.from_numpy(gs.offsets), nnn, u)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, payload, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, out, part, gathered = q.get(timeout=120)
        assert gathered
        res[r] = (out, part)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    E = gs.gid.size // nnn
    starts = element_ranges(E, world)
    got = np.concatenate([res[r][0] for r in range(world)])
    assert np.array_equal(got, want)
    for r in range(world):
        assert np.array_equal(res[r][1], np.array([world * (world + 1) / 2, 0.25 * world * (world - 1)]))
    assert starts[-1] == E


def test_interior_run():
    """Element range computed while the halo travels (space.interior_run)."""
    from paper_2207_07098_b200.space import interior_run

    E = 64
    # z-slab middle rank: first and last 16-element layers hold interface copies
    iface = list(range(0, 16)) + list(range(48, 64))
    assert interior_run(iface, E) == (16, 48)
    assert interior_run(list(range(48, 64)), E) == (0, 48)          # first rank
    assert interior_run(list(range(0, 16)), E) == (16, 64)          # last rank
    assert interior_run([3, 50], E) == (4, 50)                       # even bounds
    assert interior_run(list(range(E)), E) is None
    assert interior_run([0, 2], 3) is None


def test_abort_grace_hook_reports_then_waits():
    """A rank that dies with peer memory mapped keeps its process alive past the
    peer kernels' poll timeout (dist.ABORT_GRACE_S) after reporting the error."""
    import time

    from paper_2207_07098_b200 import dist as sfdist

    seen = []
    hook = sfdist._abort_grace_hook(lambda tp, val, tb: seen.append((tp, time.perf_counter())), grace=0.2)
    t0 = time.perf_counter()
    hook(RuntimeError, RuntimeError("x"), None)
    assert seen and seen[0][0] is RuntimeError and seen[0][1] - t0 < 0.1
    assert time.perf_counter() - t0 >= 0.2
    assert sfdist.ABORT_GRACE_S > 5.0          # the peer poll timeout (csrc/peer.cuh)
