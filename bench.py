"""Benchmark of the SEM hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload tgv|poisson|channel|cylinder]
                    [--ne N] [--impl ours|reference]

Workloads (BASELINE.json configs):
  poisson  config 2: Jacobi-PCG on the 32^3-element lx=8 box, Dirichlet walls;
           one step = one PCG solve (42 iterations, tol 1e-8, identical to the
           reference's count); metric value = P * iterations / t (GDOF/s of
           operator work).
  tgv      configs 1/3 (default): BDF3/EXT3 Taylor-Green step, 64^3 (--ne).
  channel  config 4: 48x32x48 channel box (--ne scales it).
  cylinder config 5: cylinder-in-box (Flettner rotor) mesh, counts / --ne
           (default 2: 252 928 curved elements, 129 M points).

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
synchronize, timed with CUDA events on the launching stream, max over ranks.
Inputs are larger than L2 (126 MB): at 32^3 one field is 134 MB and the
geometric factors 805 MB, so every step streams from HBM.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- helpers

def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        # NCCL prints its version banner on stdout at the VERSION and WARN levels;
        # the driver expects exactly one JSON line there
        if os.environ.get("NCCL_DEBUG", "WARN").upper() in ("WARN", "VERSION"):
            os.environ["NCCL_DEBUG"] = "NONE"
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier_max(value, world):
    """max over ranks of a host float (timing rule: max over ranks)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum(values, world):
    """sum over ranks of a list of host floats"""
    if world == 1:
        return list(values)
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def step_traffic(bytes_sum, gate, t, steps, world, peak):
    """Step-level roofline (SURVEY 8(d) "Time step"): the algorithmic bytes of every
    library call in the timed steps (traffic.py; gated second-sweep MGS passes
    credited with the measured fire fraction), summed over ranks, per step and
    divided by the step time.  torch's own elementwise kernels are not credited."""
    from paper_2207_07098_b200 import traffic

    fire = gate[0] / gate[1] if gate[1] else 1.0
    per_step = (bytes_sum[0] + fire * bytes_sum[1]) / steps
    ach = per_step / (t / steps) / 1e9
    return {"algorithmic_bytes_per_step": per_step, "achieved": ach, "peak": peak * world, "unit": "GB/s",
            "frac": ach / (peak * world), "second_sweep_fire_fraction": fire,
            "uncredited": sorted(traffic.UNMODELED) + ["torch elementwise kernels"]}


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def poisson_space(ne, dev):
    import torch

    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space

    sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (ne, ne, ne)), make_basis(7), device=dev)
    mask = torch.ones(sp.shape, dtype=torch.float64, device=dev)
    mask.view(-1)[sp.facet_flat.reshape(-1)] = 0.0
    x, y, z = sp.coords
    f = 3.0 * math.pi ** 2 * torch.sin(math.pi * x) * torch.sin(math.pi * y) * torch.sin(math.pi * z)
    return sp, mask, f


def ax_dssum_bytes(sp, masked, helmholtz=False):
    """Algorithmic bytes of one Ax+dssum application."""
    P = sp.n_points
    gs = sp.gs
    b = P * (8 + 48 + 8) + (P * 8 if helmholtz else 0)
    b += gs.shared_local_points * (8 + 8 + 4) + gs.n_shared * 4
    return b


def time_kernels(sp, op, u, reps=20):
    """Average CUDA-event durations of the Ax kernel and the dssum kernel on the
    launching stream (inputs > L2 at >= 32^3)."""
    import torch

    from paper_2207_07098_b200 import _lib
    from paper_2207_07098_b200.operators import _ex

    st = torch.cuda.current_stream()
    stp = st.cuda_stream
    w = torch.empty_like(u)
    gs = sp.gs
    E = sp.n_elements

    def ax():
        if op.masked:
            _lib.call("sf_ax_masked_f64", sp.dmat.ctypes.data, sp.n, _lib.ptr(sp.geom), _lib.ptr(sp.bm),
                      _lib.ptr(u), _lib.ptr(w), E, op.lam_visc, op.lam_mass, _lib.ptr(op.inmask),
                      _lib.ptr(op.outsel), _ex(), stp)
        else:
            _lib.call("sf_ax_helm_f64", sp.dmat.ctypes.data, sp.n, _lib.ptr(sp.geom), _lib.ptr(sp.bm),
                      _lib.ptr(u), _lib.ptr(w), E, op.lam_visc, op.lam_mass, _ex(), stp)

    def dss():
        if op.masked:
            gs.dssum_into(w, 2, u=u, perm=op.sh_perm)
        else:
            gs.dssum_into(w, 0)

    jobs = [("ax", ax), ("dssum", dss)]
    res = {}
    for name, fn in jobs:
        for _ in range(3):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in evs:
            a.record(st)
            fn()
            b.record(st)
        torch.cuda.synchronize()
        res[name] = float(np.mean([a.elapsed_time(b) for a, b in evs])) * 1e-3
    return res


#: dram__bytes_read.sum + dram__bytes_write.sum per launch of the MGS pass, from
#: the ncu --set full capture committed under profiles/ (keyed by mesh size)
def _sum_or_none(*xs):
    return None if any(x is None for x in xs) else sum(xs)


def ncu_traffic(kernel, ne):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` on the
    ne^3 lx=8 box, from the committed ncu --set full summary
    (profiles/r2_ncu_traffic.json, tools/kernel_probe.py under ncu); None when that
    size was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")) as fh:
            tab = json.load(fh)["bytes_per_launch"]
        return tab.get(kernel, {}).get(str(ne))
    except (OSError, ValueError, KeyError):
        return None


def time_mgs(sp, w0, reps=20):
    """CUDA-event time of one GMRES MGS pass (w -= h v_prev; <w, v_next>_1/mult)
    on full-size fields; returns (seconds, algorithmic bytes = P * 33)."""
    import torch

    from paper_2207_07098_b200 import _device, _lib

    st = torch.cuda.current_stream()
    w = w0.clone()
    vp = torch.randn_like(w0)
    vn = torch.randn_like(w0)
    h = torch.tensor([1e-9, 0.0], dtype=torch.float64, device=w0.device)
    out = torch.zeros(2, dtype=torch.float64, device=w0.device)
    wk = _device.workspace(w0.device)
    P = sp.n_points

    def fn():
        _lib.call("sf_mgs_step_f64", _lib.ptr(w), _lib.ptr(vp), _lib.ptr(h), _lib.ptr(vn), None, None,
                  _lib.ptr(sp.gs.mult8), 0, P, *wk.args(), _lib.ptr(out), None, st.cuda_stream)

    for _ in range(3):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in evs:
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in evs])) * 1e-3, P * 33


# ----------------------------------------------------------------------------- CPU baseline

def cpu_poisson_sample():
    """Oracle (CPU port of the reference) Jacobi-PCG on the 8^3 lx=8 Poisson box."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import semflow_oracle as O

    sp = O.build_space(O.gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (8, 8, 8)), O.make_basis(7))
    mask = np.ones(sp.shape)
    mask.reshape(-1)[sp.facet_flat.ravel()] = 0.0
    x, y, z = sp.coords
    f = 3.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    rhs = mask * sp.gs.add(sp.bm * f)
    A = O.make_global_op(sp, 1.0, 0.0, mask)
    M = O.block_jacobi(sp, 1.0, 0.0, mask)[0]
    O.pcg(A, rhs, 1e-8, 500, M, sp.gs.dot)       # warm
    t0 = time.perf_counter()
    reps = 0
    its = 0
    while True:
        info = O.pcg(A, rhs, 1e-8, 500, M, sp.gs.dot)
        reps += 1
        its += info.iterations
        if time.perf_counter() - t0 > 10.0:
            break
    dt = time.perf_counter() - t0
    P = int(np.prod(sp.shape))
    return {"value": P * its / dt / 1e9, "unit": "GDOF/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"oracle Jacobi-PCG, 8^3 lx=8 Poisson box ({P} points), {reps} solves x "
                      f"{its // reps} iterations in {dt:.1f} s"}


# ----------------------------------------------------------------------------- workloads

def bench_poisson(args, world, rank, dev):
    import torch

    from paper_2207_07098_b200 import _lib, krylov, operators as ops
    from paper_2207_07098_b200.precond import BlockJacobi

    ne = args.ne or 32
    sp, mask, f = poisson_space(ne, dev)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    M = BlockJacobi(sp, 1.0, 0.0, mask)
    rhs = mask * sp.gs.add(sp.bm * f)
    P = sp.n_points
    solve = lambda b: krylov.pcg(A, b, tol=1e-8, max_iter=500, precond=M, dot=sp.gs.dot)
    for _ in range(args.warmup):
        info = solve(rhs)
    st = torch.cuda.current_stream()
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    barrier(world)
    torch.cuda.synchronize()
    l0 = _lib.LAUNCHES
    _lib.BYTES[:] = [0, 0]
    _lib.ACCOUNT = True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    its = 0
    for _ in range(args.steps):
        info = solve(rhs)
        its += info.iterations
    e1.record(st)
    _lib.ACCOUNT = False
    torch.cuda.synchronize()
    barrier(world)
    launches = _lib.LAUNCHES - l0
    traffic_sum = all_sum(list(_lib.BYTES), world)
    clk.stop()
    t = barrier_max(e0.elapsed_time(e1) * 1e-3, world)
    value = world * P * its / t / 1e9
    # end to end through the public API with host buffers: H2D of the rhs, solve, D2H of x
    rhs_h = rhs.cpu().pin_memory()
    x_h = torch.empty_like(rhs_h).pin_memory()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_its = 0
    for _ in range(args.steps):
        b = rhs_h.to(dev, non_blocking=True)
        info = solve(b)
        x_h.copy_(info.x, non_blocking=True)
        torch.cuda.synchronize()
        e_its += info.iterations
    te = barrier_max(time.perf_counter() - t0, world)
    e2e = {"value": world * P * e_its / te / 1e9, "unit": "GDOF/s",
           "h2d_bytes_per_step": rhs_h.numel() * 8, "d2h_bytes_per_step": x_h.numel() * 8}
    kt = time_kernels(sp, A, torch.randn(sp.shape, dtype=torch.float64, device=dev))
    pk, src = peaks()
    nbytes = ax_dssum_bytes(sp, True)
    t_op = kt["ax"] + kt["dssum"]
    achieved = nbytes / t_op / 1e9
    line = {
        "metric": "GDOF/s per PCG iteration (config 2: Poisson Ax+dssum+Jacobi-CG, 32^3 lx=8)",
        "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"poisson {ne}^3 lx=8 Dirichlet box, Jacobi-PCG tol 1e-8 (config 2)",
                   "points": P, "iterations_per_step": its // args.steps, "l2": "inputs larger than L2",
                   "parallelism": f"replicas x{world}" if world > 1 else "single"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"],
                     "traffic": _sum_or_none(ncu_traffic("ax8t_kernel<0,1,0,0>", ne),
                                             ncu_traffic("dssum_blk_kernel<2>", ne)),
                     "kernel": "ax8t_kernel (masked) + dssum_blk_kernel",
                     "algorithmic_bytes": nbytes, "us": t_op * 1e6, "ax_us": kt["ax"] * 1e6,
                     "dssum_us": kt["dssum"] * 1e6, "peak_source": src,
                     "step": step_traffic(traffic_sum, [0, 0], t, args.steps, world, pk["hbm_gbs"])},
        "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
    }
    return line


def cpu_tgv_sample(steps=None, warmup=None, budget=20.0):
    """Oracle (CPU port of the reference) TGV Re=1600 on the 8^3 lx=8 box: mean step time
    over the first steps (config 1, the reference's own CPU-runnable case)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import semflow_oracle as O

    sp, st, state = O.tgv_setup(8)
    P = int(np.prod(sp.shape))
    for _ in range(warmup or 0):
        state, _d = st.step(state)
    times, its = [], []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        state, d = st.step(state)
        times.append(time.perf_counter() - t0)
        its.append(d.p_iterations)
        if (steps is not None and len(times) >= steps) or (steps is None and time.perf_counter() - t_all > budget):
            break
    t = float(np.mean(times))
    first = (warmup or 0) + 1
    return {"value": P / t / 1e9, "unit": "GDOF/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"oracle TGV Re=1600 8^3 lx=8 ({P} points), steps {first}-{first + len(times) - 1} "
                      f"(pressure its {its}), mean {t:.2f} s/step"}


def cpu_channel_sample(budget=20.0):
    """Oracle channel (config-4 set-up) on a 12x8x12 lx=8 box: mean step time over
    the first steps within the budget (the full 48x32x48 case needs ~40 min per
    step on the CPU reference)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import semflow_oracle as O

    sp, st, state = O.channel_setup((12, 8, 12))
    P = int(np.prod(sp.shape))
    times, its = [], []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        state, d = st.step(state)
        times.append(time.perf_counter() - t0)
        its.append(d.p_iterations)
        if time.perf_counter() - t_all > budget:
            break
    t = float(np.mean(times))
    return {"value": P / t / 1e9, "unit": "GDOF/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"oracle channel 12x8x12 lx=8 ({P} points), steps 1-{len(times)} "
                      f"(pressure its {its}), mean {t:.2f} s/step"}


def cpu_cylinder_sample(budget=20.0):
    """Oracle on the config-5 set-up at counts / 16 (456 curved elements, lx=8):
    mean step time over the first steps within the budget.  The mesh comes from
    the package's generator, which is bit-identical to the reference's."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import semflow_oracle as O

    from paper_2207_07098_b200.mesh import gen_cylinder_box_mesh
    from paper_2207_07098_b200.timestep import cylinder_params

    prm = cylinder_params(16)
    sp = O.build_space(gen_cylinder_box_mesh(**prm), O.make_basis(7))
    bc = O.Boundary(sp, {"inflow": {"kind": "inflow", "u_cl": 1.0, "h": prm["height"]}, "outflow": {"kind": "outflow"},
                         "bottom": {"kind": "noslip"}, "top": {"kind": "symmetry"}, "span": {"kind": "symmetry"},
                         "cylinder": {"kind": "rotor", "u_cl": 1.0, "alpha": 3.0, "delta": 0.25}})
    st = O.Stepper(sp, bc, 1.0 / 100.0, 2e-3)
    v0 = np.zeros((3,) + sp.shape)
    v0[0] = 1.0
    state = st.initial_state(v0)
    P = int(np.prod(sp.shape))
    times, its = [], []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        state, d = st.step(state)
        times.append(time.perf_counter() - t0)
        its.append(d.p_iterations)
        if time.perf_counter() - t_all > budget:
            break
    t = float(np.mean(times))
    return {"value": P / t / 1e9, "unit": "GDOF/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"oracle cylinder config-5 counts/16 ({sp.shape[0]} elements, {P} points), steps "
                      f"1-{len(times)} (pressure its {its}), mean {t:.2f} s/step"}


def bench_tgv(args, world, rank, dev):
    import torch

    from paper_2207_07098_b200 import _lib
    from paper_2207_07098_b200.timestep import FlowState, kinetic_energy, tgv_problem

    from paper_2207_07098_b200 import dist as sfdist

    # config 3 is TGV 64^3 (134 M points).  The reference's projection spaces add
    # 8 fields (1.07 GB each at 64^3) per step up to 20 solves, so one B200
    # (180 GB) holds 64^3 for at most 8 warm-up + timed steps; longer runs use
    # 48^3 at every GPU count so the strong-scaling series stays one workload.
    comm = sfdist.init_from_env()
    if args.workload == "channel":
        from paper_2207_07098_b200.timestep import channel_problem

        counts = (48, 32, 48) if not args.ne else (args.ne, max(1, 2 * args.ne // 3), args.ne)
        ne = counts
        sp, st, state = channel_problem(counts, device=dev, comm=comm, precond=args.precond)
        P = counts[0] * counts[1] * counts[2] * sp.n ** 3
    elif args.workload == "cylinder":
        from paper_2207_07098_b200.timestep import cylinder_problem

        ne = args.ne or 2                    # scale divisor of the config-5 counts
        sp, st, state = cylinder_problem(ne, device=dev, comm=comm, projection=args.projection == "on",
                                         restart=args.restart, recycle=True)
        sp.release_setup_fields()          # coords / jac: set-up only (4 fields of HBM)
        P = sp.mesh.n_elements * sp.n ** 3
    else:
        ne = args.ne or (64 if args.warmup + args.steps <= 8 else 48)
        sp, st, state = tgv_problem(ne, device=dev, comm=comm, precond=args.precond,
                                    projection=args.projection == "on", dealias=args.dealias,
                                    **({"dt": args.dt} if args.dt > 0 else {}))
        P = ne ** 3 * sp.n ** 3            # global points: strong scaling, fixed total work
    for k in range(args.warmup):
        # the projection bases grow by one (x, Ax) pair per solve: reserve the
        # slots of the last warm-up step and the timed steps up front (setup-time
        # allocation, as Neko's projection init; the same memory the last warm-up
        # step would have taken anyway), then run that step so the allocator's
        # cache holds every field a step allocates and frees
        if k == args.warmup - 1 and not args.no_reserve:
            st.reserve_projection(args.steps + 1)
        state, d = st.step(state)
    stream = torch.cuda.current_stream()
    # one timed loop gives both numbers over the SAME K steps:
    #   value: device time of each step (CUDA events on the launching stream),
    #   e2e:   wall time of each step through the public API with host buffers --
    #          the caller's velocity field is copied in from pinned host memory and
    #          the new velocity is read back (the reference's Stepper works on host
    #          arrays); the rest of the FlowState stays resident on the device.
    #          The read-back of step k's velocity and the upload of step k+1's
    #          input (the caller hands the result back) run chunk by chunk on the
    #          two copy directions at once; step 0's input is uploaded whole.
    vel_h = state.vel.cpu().pin_memory()
    out_h = torch.empty_like(vel_h).pin_memory()
    s_d2h, s_h2d = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    n_chunk = 16
    nel = vel_h.numel()
    cuts = [nel * c // n_chunk for c in range(n_chunk + 1)]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clk = ClockSampler(torch.cuda.current_device())
    # setup objects (meshes, maps, operators) are long-lived: move them out of the
    # collector's generations so a full collection during a step stays cheap
    import gc

    if os.environ.get("SEMFLOW_B200_GC_FREEZE", "1") != "0":
        gc.collect()
        gc.freeze()
    from paper_2207_07098_b200 import krylov as _kry

    clk.start()
    barrier(world)
    torch.cuda.synchronize()
    l0 = _lib.LAUNCHES
    _lib.BYTES[:] = [0, 0]
    _kry.GATE_STATS[:] = [0, 0]
    _lib.ACCOUNT = True
    p_its, v_its, cfls = [], [], []
    allocs0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    t0 = time.perf_counter()
    v = vel_h.to(dev, non_blocking=True)
    for k in range(args.steps):
        state = FlowState(state.time, state.nsteps, [v] + state.vel_hist[1:], state.curl_hist,
                          state.nl_hist, state.prs, state.primed)
        evs[k][0].record(stream)
        state, d = st.step(state)
        evs[k][1].record(stream)
        # result -> caller (D2H), caller's next input -> device (H2D), pipelined
        v = torch.empty_like(state.vel) if k + 1 < args.steps else None
        src, hb = state.vel.view(-1), out_h.view(-1)
        s_d2h.wait_event(evs[k][1])
        for c in range(n_chunk):
            lo, hi = cuts[c], cuts[c + 1]
            with torch.cuda.stream(s_d2h):
                hb[lo:hi].copy_(src[lo:hi], non_blocking=True)
            if v is not None:
                s_h2d.wait_stream(s_d2h)
                with torch.cuda.stream(s_h2d):
                    v.view(-1)[lo:hi].copy_(hb[lo:hi], non_blocking=True)
        torch.cuda.synchronize()
        del src                          # the result buffer leaves with the state it belongs to
        vel_h, out_h = out_h, vel_h      # the result is the caller's next input (no host copy)
        p_its.append(d.p_iterations)
        v_its.append(list(d.v_iterations))
        cfls.append(round(d.cfl, 4))
    te_local = time.perf_counter() - t0
    device_allocs = torch.cuda.memory_stats().get("num_device_alloc", 0) - allocs0
    _lib.ACCOUNT = False
    torch.cuda.synchronize()
    barrier(world)
    launches = _lib.LAUNCHES - l0
    traffic_sum = all_sum(list(_lib.BYTES) + list(_kry.GATE_STATS), world)
    clk.stop()
    t = barrier_max(sum(a.elapsed_time(b) for a, b in evs) * 1e-3, world)
    te = barrier_max(te_local, world)
    value = P * args.steps / t / 1e9
    ke = kinetic_energy(sp, state.vel)
    e2e = {"value": P * args.steps / te / 1e9, "unit": "GDOF/s",
           "h2d_bytes_per_step": P * 3 * 8, "d2h_bytes_per_step": P * 3 * 8}
    op = st.apply_p
    probe = torch.randn(sp.shape, dtype=torch.float64, device=dev)
    kt = time_kernels(sp, op, probe)
    pk, src = peaks()
    nbytes = ax_dssum_bytes(sp, op.masked)
    t_op = kt["ax"] + kt["dssum"]
    achieved = nbytes / t_op / 1e9
    # dominant kernel of the step: the GMRES modified-Gram-Schmidt pass
    # (w -= h v_{i-1}; <w, v_i>) -- ~70 % of the step at 64^3 (profiles/)
    t_mgs, mgs_bytes = time_mgs(sp, probe)
    mgs_gbs = mgs_bytes / t_mgs / 1e9
    if args.workload == "channel":
        wl_name = (f"channel {ne[0]}x{ne[1]}x{ne[2]} elements lx=8 (config 4{'' if ne == (48, 32, 48) else ' analogue'}),"
                   " Poiseuille inflow/outflow/no-slip/symmetry, nu=1/2800 dt=2e-3,"
                   f" {'Schwarz' if args.precond == 'schwarz' else 'Jacobi'}-GMRES(20) p 1e-5,"
                   f" Jacobi-PCG v 1e-8, projection {args.projection}")
        metric = "GDOF/s per time step (channel, lx=8)"
    elif args.workload == "cylinder":
        wl_name = (f"cylinder-in-box (Flettner-rotor) {sp.mesh.n_elements} curved/unstructured hex elements lx=8"
                   f" (config 5{'' if ne == 1 else f' counts / {ne}'}), rotor wall, power-law inflow, Re=100"
                   f" dt=2e-3, Jacobi-GMRES({args.restart}) p 1e-5, Jacobi-PCG v 1e-8, projection {args.projection}")
        metric = "GDOF/s per time step (cylinder, lx=8)"
    else:
        wl_name = (f"TGV Re=1600 {ne}^3 elements lx=8 (config {'3' if ne == 64 else '1' if ne == 8 else '1/3 analogue'}),"
                   f" symmetry box, {'Schwarz' if args.precond == 'schwarz' else 'Jacobi'}-GMRES(20) p 1e-5,"
                   f"{' dealiased convection (3/2 rule),' if args.dealias else ''}"
                   f" Jacobi-PCG v 1e-8, projection {args.projection}")
        metric = "GDOF/s per time step (TGV, lx=8)"
    return {
        "metric": metric,
        "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl_name,
                   "points": P, "steps_timed": f"{args.warmup + 1}-{args.warmup + args.steps}",
                   "p_iterations": p_its, "v_iterations": v_its, "ke_end": ke, "cfl": cfls,
                   "dt": st.dt, "capped_p_solves": sum(1 for q in p_its if q >= st.p_opt.max_iter),
                   "device_allocs_timed_rank0": int(device_allocs),
                   "peak_mem_gb_rank0": torch.cuda.max_memory_allocated() / 1e9,
                   "alloc_retries_rank0": int(torch.cuda.memory_stats().get("num_alloc_retries", 0)),
                   "l2": "inputs larger than L2" if P * 8 * 6 / world > 126e6 else "working set may be L2-resident",
                   "parallelism": (f"element partition x{world} (contiguous element ranges), "
                                   + ("NVLink IPC halo exchange + peer-memory glsc3 allreduce fused into the "
                                      "Krylov kernels" if sp.comm.peer is not None else
                                      "NCCL halo exchange + all-gather dots")
                                   if world > 1 else "single")},
        "roofline": {"bound": "hbm", "achieved": mgs_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": mgs_gbs / pk["hbm_gbs"], "traffic": ncu_traffic("mgs2_kernel<1,1,0,0>", ne),
                     "kernel": "mgs2_kernel<true,true,false,false> (GMRES MGS pass, rank 0)",
                     "algorithmic_bytes": mgs_bytes, "us": t_mgs * 1e6, "peak_source": src,
                     "ax_dssum": {"achieved": achieved, "frac": achieved / pk["hbm_gbs"],
                                  "algorithmic_bytes": nbytes, "us": t_op * 1e6, "ax_us": kt["ax"] * 1e6,
                                  "dssum_us": kt["dssum"] * 1e6,
                                  "traffic": _sum_or_none(ncu_traffic("ax8t_kernel<0,0,0,0>", ne),
                                                          ncu_traffic("dssum_blk_kernel<0>", ne)),
                                  "kernel": "ax8t_kernel + dssum_blk_kernel (pressure Poisson operator)"},
                     "step": step_traffic(traffic_sum[:2], traffic_sum[2:], t, args.steps, world,
                                          pk["hbm_gbs"])},
        "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
    }


def _arm_workload(args):
    """The GPU arm's workload name for the same flags (the reference arm reports it)."""
    if args.workload == "poisson":
        return f"poisson {args.ne or 32}^3 lx=8 Dirichlet box, Jacobi-PCG tol 1e-8 (config 2)"
    if args.workload == "channel":
        return "channel 48x32x48 elements lx=8 (config 4)" if not args.ne else f"channel analogue ne={args.ne}"
    if args.workload == "cylinder":
        return f"cylinder-in-box (Flettner rotor), config 5 counts / {args.ne or 2}, lx=8"
    ne = args.ne or (64 if args.warmup + args.steps <= 8 else 48)
    return f"TGV Re=1600 {ne}^3 elements lx=8 (config {'3' if ne == 64 else '1' if ne == 8 else '1/3 analogue'})"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-reserve", action="store_true",
                    help="grow the projection bases inside the timed steps (A/B of the slot reservation)")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="tgv", choices=("tgv", "poisson", "channel", "cylinder"))
    ap.add_argument("--ne", type=int, default=0)
    ap.add_argument("--dealias", action="store_true",
                    help="TGV: over-integrated convection (operators.Dealias, 3/2 rule)")
    ap.add_argument("--restart", type=int, default=20,
                    help="cylinder: pressure GMRES restart (20 as the reference; 10 frees 10 fields)")
    ap.add_argument("--projection", default="on", choices=("on", "off"),
                    help="solution projection (the reference's default: on); off frees its bases")
    ap.add_argument("--precond", default="jacobi", choices=("jacobi", "schwarz"),
                    help="TGV pressure preconditioner (schwarz: the reference's default, small meshes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dt", type=float, default=0.0,
                    help="TGV time step (default: the config's literal 1e-2)")
    ap.add_argument("--no-cfl-matched", action="store_true",
                    help="skip the second TGV run at the paper's CFL (~0.4)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        if args.workload == "tgv":
            base = cpu_tgv_sample(steps=args.steps, warmup=args.warmup)
            metric = "GDOF/s per time step (TGV, lx=8)"
        elif args.workload == "channel":
            base = cpu_channel_sample()
            metric = "GDOF/s per time step (channel, lx=8)"
        elif args.workload == "cylinder":
            base = cpu_cylinder_sample()
            metric = "GDOF/s per time step (cylinder, lx=8)"
        else:
            base = cpu_poisson_sample()
            metric = "GDOF/s per PCG iteration (config 2: Poisson Ax+dssum+Jacobi-CG, 32^3 lx=8)"
        line = {"impl": "reference", "metric": metric,
                "value": base["value"], "unit": "GDOF/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
                "config": {"workload": _arm_workload(args),
                           "timed_on": "a bounded CPU sample of that workload (cpu_baseline.sample): the "
                                       "full-size case needs minutes to hours per step on the host"},
                "cpu_baseline": base, "e2e": {"value": base["value"], "unit": "GDOF/s",
                                              "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    import torch

    world, rank, local = dist_setup()
    dev = torch.device("cuda", torch.cuda.current_device())
    line = (bench_poisson if args.workload == "poisson" else bench_tgv)(args, world, rank, dev)
    if args.workload == "tgv" and not args.no_cfl_matched and args.dt <= 0:
        # The literal config fixes dt = 1e-2 at every mesh size (CFL 0.2 at 8^3,
        # ~1.2 at 48^3, ~1.6 at 64^3: past the explicit EXT3 limit, so GMRES hits
        # its cap).  The same workload at the paper's CFL ~0.4,
        # dt scaled with the element size, is reported beside it.
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        ne = args.ne or (64 if args.warmup + args.steps <= 8 else 48)
        a2 = argparse.Namespace(**vars(args))
        a2.dt = 1e-2 * (0.4 / 0.1985) * 8.0 / ne       # CFL = 0.1985 at 8^3, dt = 1e-2 (golden)
        l2 = bench_tgv(a2, world, rank, dev)
        c2 = l2["config"]
        line["cfl_matched"] = {
            "dt": a2.dt, "value": l2["value"], "unit": l2["unit"], "ms_per_step": l2["ms_per_step"],
            "e2e": l2["e2e"], "cfl": c2["cfl"], "p_iterations": c2["p_iterations"],
            "v_iterations": c2["v_iterations"], "capped_p_solves": c2["capped_p_solves"],
            "device_allocs_timed_rank0": c2["device_allocs_timed_rank0"], "ke_end": c2["ke_end"],
            "step_roofline_frac": l2["roofline"]["step"]["frac"], "clocks": l2["clocks"],
            "note": "same mesh, solver settings and step numbers at dt scaled to CFL ~0.4 (the paper's)"}
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            # the same step numbers as the GPU's timed steps, on the 8^3 mesh the
            # CPU port finishes in seconds (config 1)
            line["cpu_baseline"] = {"tgv": lambda: cpu_tgv_sample(steps=args.steps, warmup=args.warmup),
                                    "channel": lambda: cpu_channel_sample(),
                                    "cylinder": lambda: cpu_cylinder_sample(),
                                    "poisson": cpu_poisson_sample}[args.workload]()
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
