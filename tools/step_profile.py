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
    sp, st, state = tgv_problem(ne, device=dev, comm=comm, precond=os.environ.get("PRECOND", "jacobi"))
    for k in range(warm):
        if k == warm - 1 and os.environ.get("RESERVE", "1") == "1":
            st.reserve_projection(steps + 1)     # as bench.py does before its last warm-up step
        state, d = st.step(state)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_stats()
    if os.environ.get("MEMHIST", "0") == "1":
        torch.cuda.memory._record_memory_history(max_entries=200000)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            state, d = st.step(state)
            if comm.rank == 0:
                print("step", d.step, "p_it", d.p_iterations, "v_it", d.v_iterations, "wall", round(d.wall_time, 4))
        torch.cuda.synchronize()
    if comm.rank != 0:
        return
    m1 = torch.cuda.memory_stats()
    if os.environ.get("MEMHIST", "0") == "1":
        snap = torch.cuda.memory._snapshot()
        for tr in snap["device_traces"]:
            for e in tr:
                if e["action"] == "segment_alloc":
                    fr = [f"{f['filename'].split('/')[-1]}:{f['line']}:{f['name']}" for f in e.get("frames", [])
                          if "paper_2207" in f["filename"] or "step_profile" in f["filename"]]
                    print(f"segment_alloc {e['size'] / 2**30:.3f} GiB <- {' < '.join(fr[:6])}")
    print("allocator over the profiled steps:", {k: m1.get(k, 0) - m0.get(k, 0) for k in
          ("num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams")})
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
    if os.environ.get("CPU_TABLE", "0") == "1":
        print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=20))
    # device idle gaps between consecutive kernels (host-side stalls)
    spans = sorted((ev.time_range.start, ev.time_range.end, ev.name.split("(")[0][:50])
                   for ev in prof.events() if ev.device_type.name == "CUDA")
    gaps = []
    for a, b in zip(spans, spans[1:]):
        g = b[0] - max(a[1], 0)
        if g > 0:
            gaps.append((g, a[2], b[2]))
    if spans:
        busy_span = spans[-1][1] - spans[0][0]
        print(f"device span {busy_span / 1e3:.2f} ms, idle {sum(g for g, _, _ in gaps) / 1e3:.2f} ms "
              f"in {len(gaps)} gaps ({sum(g for g, _, _ in gaps if g > 100) / 1e3:.2f} ms in gaps > 100 us)")
        by = {}
        for g, a, b in gaps:
            k = (a, b)
            c = by.setdefault(k, [0.0, 0])
            c[0] += g
            c[1] += 1
        for (a, b), (t, n) in sorted(by.items(), key=lambda kv: -kv[1][0])[:15]:
            print(f"  gap {t / 1e3:8.2f} ms {n:5d}x  after {a}  before {b}")


if __name__ == "__main__":
    main()
