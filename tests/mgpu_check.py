"""Multi-GPU parity check, run under torchrun (one rank per GPU):

    torchrun --standalone --nproc-per-node 2 tests/mgpu_check.py [ne] [steps]

0. the partitioned build's gid slice, multiplicities and global id count equal the
   single-GPU build's (TGV box and the curved mini-rotor mesh);
1. partitioned dssum (add / avg / masked Poisson operator) on a random field is
   bitwise identical to the single-GPU result, on every rank;
2. partitioned glsc3 equals the single-GPU value to rounding;
3. the TGV step on the partitioned mesh reproduces the reference's iteration
   counts and kinetic energy (tests/golden/solvers.json) when ne is 4 or 8 --
   with the look-ahead GMRES replaying its Arnoldi steps from CUDA graphs that
   contain the fused NVLink reductions and halo exchanges;
4. stress: 10^4 back-to-back fused MGS reductions, a pseudo-random third of them
   gated off on the device, no halo exchange and no host sync in between, with
   integer-valued data so every sum is exact: each result equals the 1-GPU value
   bit for bit (the mailbox banks follow the executed calls only);
5. a graph-captured dssum with its halo exchange, replayed 64 times on changing
   input, bitwise equal to the single-GPU dssum;
6. the hybrid Schwarz preconditioner across ranks (schwarz_checks).
Rank 0 prints one JSON line and exits nonzero on failure.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2207_07098_b200 import dist, operators as ops
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space
    from paper_2207_07098_b200.timestep import enstrophy, kinetic_energy, tgv_problem

    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    comm = dist.init_from_env()
    dev = torch.device("cuda", torch.cuda.current_device())
    r, W = comm.rank, comm.world
    L = 2 * np.pi
    mesh = gen_box_mesh((0, L, 0, L, 0, L), (ne, ne, ne))
    basis = make_basis(7)
    full = build_space(mesh, basis, device=dev)                 # single-GPU reference on each rank
    _FULL["space"] = full
    part = build_space(mesh, basis, device=dev, comm=comm)
    e0, e1 = part.e_range
    nnn = basis.n ** 3
    # the partitioned build (partition.py, default for N > 1) gives this rank
    # exactly the single-GPU build's gid slice and multiplicities
    ok = {}
    ok["partitioned_gid"] = bool(torch.equal(part.gs.gid, full.gs.gid[e0 * nnn:e1 * nnn]))
    ok["partitioned_mult"] = bool(torch.equal(part.gs.mult8, full.gs.mult8[e0 * nnn:e1 * nnn]))
    ok["partitioned_n_gid"] = part.gs.n_gid == full.gs.n_gid
    g = torch.Generator(device="cpu").manual_seed(5)
    u_full = torch.randn(full.shape, generator=g, dtype=torch.float64).to(dev)
    u = u_full[e0:e1].contiguous()
    ok["dssum_add"] = bool(torch.equal(part.gs.add(u), full.gs.add(u_full)[e0:e1]))
    ok["dssum_avg"] = bool(torch.equal(part.gs.avg(u), full.gs.avg(u_full)[e0:e1]))
    mask_f = torch.ones(full.shape, dtype=torch.float64, device=dev)
    mask_f.view(-1)[full.facet_flat.reshape(-1)] = 0.0
    mask_p = mask_f[e0:e1].contiguous()
    a_f = ops.make_global_op(full, 1.0 / 1600, 183.3, mask_f)(u_full)[e0:e1]
    a_p = ops.make_global_op(part, 1.0 / 1600, 183.3, mask_p)(u)
    ok["masked_op"] = bool(torch.equal(a_p, a_f))
    d_f = full.gs.dot(u_full, ops.make_global_op(full, 1.0, 0.0)(u_full))
    d_p = part.gs.dot(u, ops.make_global_op(part, 1.0, 0.0)(u))
    ok["glsc3"] = abs(d_p - d_f) <= 1e-13 * abs(d_f)
    # many back-to-back exchanges without host syncs (double-banked halo inboxes)
    outs = [part.gs.add(u * float(k + 1)) for k in range(64)]
    ok["dssum_repeat"] = all(bool(torch.equal(o, full.gs.add(u_full * float(k + 1))[e0:e1]))
                             for k, o in enumerate(outs))
    ok["halo_path"] = "ipc" if getattr(part.gs, "_ipc", None) is not None else "nccl"
    # unstructured: the curved mini-rotor mesh (multiplicities up to 10, odd class sizes)
    from paper_2207_07098_b200.mesh import gen_cylinder_box_mesh

    rm = gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                               n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5)
    rfull = build_space(rm, make_basis(5), device=dev)
    rpart = build_space(rm, make_basis(5), device=dev, comm=comm)
    q0, q1 = rpart.e_range
    ok["rotor_partitioned_gid"] = bool(torch.equal(rpart.gs.gid, rfull.gs.gid[q0 * 216:q1 * 216]))
    ru = torch.randn(rfull.shape, generator=g, dtype=torch.float64).to(dev)
    ok["rotor_dssum"] = bool(torch.equal(rpart.gs.add(ru[q0:q1].contiguous()), rfull.gs.add(ru)[q0:q1]))
    del rfull, rpart
    ok.update(schwarz_checks(full, part, mask_f, mask_p, u_full, u, dev, comm, e0, e1))
    del full
    torch.cuda.empty_cache()
    ok.update(stress_checks(part, dev, comm))
    res = {"world": W, "ne": ne, "checks": ok}
    if ne in (4, 8):
        with open(os.path.join(ROOT, "tests", "golden", "solvers.json")) as fh:
            rows = json.load(fh)[f"tgv{ne}"]
        sp, st, state = tgv_problem(ne, device=dev, comm=comm)
        its, kes = [], []
        for row in rows[1:steps + 1]:
            state, d = st.step(state)
            ke = kinetic_energy(sp, state.vel)
            ens = enstrophy(sp, state.vel)
            its.append((d.p_iterations, list(d.v_iterations), row["p_it"], row["v_it"]))
            kes.append((ke, row["ke"], ens, row["ens"]))
        ok["tgv_counts"] = all(a == c and b == dd for a, b, c, dd in its)
        ok["tgv_ke"] = all(abs(k - kr) <= 1e-9 * abs(kr) and abs(e - er) <= 1e-9 * abs(er) for k, kr, e, er in kes)
        res["tgv"] = {"iterations": its, "ke": kes}
    res["ok"] = all(ok.values())
    if r == 0:
        print(json.dumps(res), flush=True)
    torch.distributed.destroy_process_group()
    sys.exit(0 if res["ok"] else 1)


def schwarz_checks(full, part, mask_f, mask_p, u_full, u, dev, comm, e0, e1):
    """Section 6: the hybrid Schwarz preconditioner across ranks -- one application
    equals the single-GPU one to rounding (the coarse restriction adds rank
    partials), the Schwarz-preconditioned GMRES takes the single-GPU iteration
    count, and the reference's TGV 4^3 Schwarz steps keep their counts."""
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.precond import HybridSchwarz
    from paper_2207_07098_b200.timestep import tgv_problem

    ok = {}
    Mf = HybridSchwarz(full, mask=mask_f)
    Mp = HybridSchwarz(part, mask=mask_p)
    # a continuous field (every copy of a gid equal), as the Krylov vectors are:
    # the gather reads one copy per gid
    uc_full = full.gs.avg(u_full)
    zf = Mf(uc_full)[e0:e1]
    zp = Mp(uc_full[e0:e1].contiguous())
    err = float((zp - zf).abs().max() / zf.abs().max())
    ok["schwarz_apply"] = err <= 1e-12
    ok["schwarz_apply_err"] = f"{err:.2e}"
    ok["schwarz_classes"] = Mp.n_classes
    x, y, z = full.coords
    f = 3.0 * np.pi ** 2 * torch.sin(x) * torch.sin(y) * torch.sin(z)
    rhs_f = mask_f * full.gs.add(full.bm * f)
    rhs_p = rhs_f[e0:e1].contiguous()
    Af = ops.make_global_op(full, 1.0, 0.0, mask_f)
    Ap = ops.make_global_op(part, 1.0, 0.0, mask_p)
    i_f = krylov.gmres(Af, rhs_f, tol=1e-8, max_iter=200, restart=20, precond=Mf, dot=full.gs.dot)
    i_p = krylov.gmres(Ap, rhs_p, tol=1e-8, max_iter=200, restart=20, precond=Mp, dot=part.gs.dot)
    ok["schwarz_gmres_its"] = i_p.iterations == i_f.iterations
    ok["schwarz_gmres_x"] = float((i_p.x - i_f.x[e0:e1]).abs().max() / i_f.x.abs().max()) <= 1e-8
    with open(os.path.join(ROOT, "tests", "golden", "schwarz.json")) as fh:
        rows = json.load(fh)["tgv4"]
    sp, st, state = tgv_problem(4, device=dev, comm=comm, precond="schwarz")
    its = []
    for row in rows:
        state, d = st.step(state)
        its.append((d.p_iterations, list(d.v_iterations), row["p_it"], row["v_it"]))
    ok["schwarz_tgv4_counts"] = all(a == c and b == dd for a, b, c, dd in its)
    # the mini-rotor case with its default Schwarz preconditioner on the curved,
    # unstructured mesh (every subdomain distinct), partitioned across the ranks
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.bc import BoundarySet
    from paper_2207_07098_b200.mesh import gen_cylinder_box_mesh
    from paper_2207_07098_b200.space import build_space
    from paper_2207_07098_b200.timestep import SolverOptions, Stepper

    with open(os.path.join(ROOT, "tests", "golden", "rotor_schwarz_steps.json")) as fh:
        rrows = json.load(fh)["rows"]
    specs = {"inflow": {"kind": "inflow", "u_cl": 1.0, "h": 2.0}, "outflow": {"kind": "outflow"},
             "bottom": {"kind": "noslip"}, "top": {"kind": "symmetry"}, "span": {"kind": "symmetry"},
             "cylinder": {"kind": "rotor", "u_cl": 1.0, "alpha": 3.0, "delta": 0.25}}
    rm = gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                               n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5)
    rsp = build_space(rm, make_basis(5), device=dev, comm=comm)
    rst = Stepper(rsp, BoundarySet(rsp, specs), nu=1.0 / 100.0, dt=2e-3, scheme_order=3,
                  pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="schwarz"),
                  velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    v0 = torch.zeros((3,) + rsp.shape, dtype=torch.float64, device=dev)
    v0[0] = 1.0
    rstate = rst.initial_state(v0)
    rits = []
    for row in rrows:
        rstate, d = rst.step(rstate)
        rits.append((d.p_iterations, list(d.v_iterations), row["p_it"], row["v_it"]))
    ok["schwarz_rotor_counts"] = all(a == c and b == dd for a, b, c, dd in rits)
    ok["schwarz_rotor_its"] = rits
    return ok


def stress_checks(part, dev, comm, n_calls=10000):
    """Sections 4 and 5 of the module docstring."""
    from paper_2207_07098_b200 import _device, _lib

    ok = {}
    r, W = comm.rank, comm.world
    P = 1 << 15
    g = torch.Generator(device="cpu").manual_seed(11)
    # global integer data; rank r owns rows [r*P, (r+1)*P)
    wg = torch.randint(-8, 9, (W * P,), generator=g, dtype=torch.int64).to(torch.float64)
    vg = torch.randint(-8, 9, (4, W * P), generator=g, dtype=torch.int64).to(torch.float64)
    w = wg[r * P:(r + 1) * P].contiguous().to(dev)
    V = vg[:, r * P:(r + 1) * P].contiguous().to(dev)
    mult = torch.ones(P, dtype=torch.uint8, device=dev)
    gates = torch.rand(n_calls, generator=g) > 1.0 / 3.0            # same pattern on every rank
    gate_dev = gates.to(torch.float64).to(dev)
    out = torch.full((n_calls, 2), -1.0, dtype=torch.float64, device=dev)
    wk = _device.workspace(dev).args()
    st = _lib.stream_ptr(dev)
    peer = comm.peer
    torch.cuda.synchronize()
    for k in range(n_calls):
        _lib.call("sf_mgs_step_peer_f64", _lib.ptr(w), None, None, _lib.ptr(V[k % 4]), None, None, _lib.ptr(mult),
                  1, P, *wk, out.data_ptr() + 16 * k, *peer.fused_args(), gate_dev.data_ptr() + 8 * k, st)
    got = out.cpu()
    want = torch.full((n_calls, 2), -1.0, dtype=torch.float64)
    dots = (vg * wg).sum(dim=1)                                      # exact: |values| < 2^53
    nrm = (wg * wg).sum()
    for k in range(n_calls):
        if gates[k]:
            want[k, 0] = dots[k % 4]
            want[k, 1] = nrm
    ok["stress_gated_reductions"] = bool(torch.equal(got, want))
    ok["stress_calls"] = n_calls
    ok["stress_executed"] = int(gates.sum())
    ok["stress_seq"] = int(peer.seq.item())
    ok["stress_seq_ok"] = ok["stress_seq"] >= ok["stress_executed"]
    # graph-captured dssum + halo exchange, replayed on changing input
    if part.gs._ipc is not None:
        u_static = torch.empty(part.shape, dtype=torch.float64, device=dev)
        u_static.copy_(torch.randn(part.shape, generator=g, dtype=torch.float64).to(dev))
        part.gs.add(u_static)                      # warm-up (eager)
        gr = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream(dev)
        s2.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s2):
            part.gs.add(u_static)
        torch.cuda.current_stream(dev).wait_stream(s2)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr):
            res_static = part.gs.add(u_static)
        good = True
        e0, e1 = part.e_range
        for k in range(64):
            ug = torch.randn(_FULL["space"].shape, generator=g, dtype=torch.float64)
            u_static.copy_(ug[e0:e1].to(dev))
            gr.replay()
            want_k = _single_dssum(ug, dev)[e0:e1]
            good &= bool(torch.equal(res_static, want_k))
        ok["graph_halo_dssum"] = good
    comm.check()
    return ok


_FULL = {}


def _single_dssum(ug, dev):
    sp = _FULL["space"]
    return sp.gs.add(ug.to(dev))


if __name__ == "__main__":
    main()
