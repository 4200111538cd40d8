"""Per-kernel device-time breakdown of TGV time steps (torch.profiler / CUPTI).

    python tools/step_profile.py [ne] [warmup] [steps]

Prints, for the profiled steps, total device time per kernel name, launch counts
and the share of the step; used to decide which kernel to optimise next.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    from paper_2207_07098_b200.timestep import tgv_problem

    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    from paper_2207_07098_b200 import dist

    comm = dist.init_from_env()          # torchrun: one rank per GPU, rank 0 reports
    dev = torch.device("cuda", torch.cuda.current_device())
    sp, st, state = tgv_problem(ne, device=dev, comm=comm)
    for _ in range(warm):
        state, d = st.step(state)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            state, d = st.step(state)
            if comm.rank == 0:
                print("step", d.step, "p_it", d.p_iterations, "v_it", d.v_iterations, "wall", round(d.wall_time, 4))
        torch.cuda.synchronize()
    if comm.rank != 0:
        return
    agg = {}
    total = 0.0
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        name = ev.name.split("(")[0][:70]
        t = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        c = agg.setdefault(name, [0.0, 0])
        c[0] += t
        c[1] += 1
        total += t
    print(f"total device time {total / 1e3:.2f} ms over {steps} step(s), {sum(v[1] for v in agg.values())} kernels")
    for name, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"{t / 1e3:10.3f} ms {100 * t / total:6.1f}%  {n:6d}x  {t / n:9.1f} us  {name}")


if __name__ == "__main__":
    main()
