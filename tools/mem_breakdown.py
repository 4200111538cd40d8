"""Device memory of a running step, by owner, in units of one scalar field.

    python tools/mem_breakdown.py <workload tgv|cylinder> <size> [projection on|off] [steps] [jacobi|schwarz]

Builds the problem on cuda:0, runs the steps, then attributes every live tensor
it can reach (space geometry and maps, FieldWork buffers, stepper state and
preconditioners, GMRES graph buffers, projection bases) and prints one JSON
line with the totals, the allocator's current and peak figures.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def nbytes(obj, seen):
    import torch

    if isinstance(obj, torch.Tensor):
        if not obj.is_cuda:
            return 0
        key = obj.untyped_storage().data_ptr()
        if key in seen:
            return 0
        seen.add(key)
        return obj.untyped_storage().nbytes()
    if isinstance(obj, (list, tuple)):
        return sum(nbytes(o, seen) for o in obj)
    if isinstance(obj, dict):
        return sum(nbytes(o, seen) for o in obj.values())
    return 0


def main():
    import torch

    from paper_2207_07098_b200 import _device
    from paper_2207_07098_b200.timestep import cylinder_problem, tgv_problem

    wl = sys.argv[1] if len(sys.argv) > 1 else "cylinder"
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    proj = (sys.argv[3] if len(sys.argv) > 3 else "off") == "on"
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    precond = sys.argv[5] if len(sys.argv) > 5 else "jacobi"
    dev = torch.device("cuda", 0)
    if wl == "cylinder":
        sp, st, state = cylinder_problem(size, device=dev, projection=proj)
    else:
        sp, st, state = tgv_problem(size, device=dev, projection=proj, precond=precond)
    after_setup = torch.cuda.memory_allocated(dev)
    for _ in range(steps):
        state, _d = st.step(state)
    torch.cuda.synchronize()
    F = sp.n_points * 8
    seen = set()
    rows = {}
    rows["geometry (coords rx jac bm geom)"] = nbytes([sp.coords, sp.rx, sp.jac, sp.bm, sp.geom], seen)
    g = sp.gs
    rows["gather-scatter maps"] = nbytes([v for v in vars(g).values() if isinstance(v, torch.Tensor)], seen)
    fw = _device.field_work(sp)
    for (name, shape), t in sorted(fw._bufs.items(), key=lambda kv: -kv[1].numel()):
        rows[f"work {name} {tuple(shape)}"] = nbytes(t, seen)
    rows["state (vel/curl/nl hist, prs)"] = nbytes([state.vel_hist, state.curl_hist, state.nl_hist, state.prs], seen)
    for k, v in vars(st).items():
        b = nbytes(v, seen)
        if b:
            rows[f"stepper.{k}"] = b
        for kk, vv in (vars(v).items() if hasattr(v, "__dict__") else []):
            b = nbytes(vv, seen)
            if b:
                rows[f"stepper.{k}.{kk}"] = b
    pc = getattr(st, "p_precond", None)
    if pc is not None and hasattr(pc, "__dict__"):
        for kk, vv in vars(pc).items():
            b = nbytes(vv, seen)
            if b:
                rows[f"p_precond.{kk}"] = b
    gb = getattr(getattr(st, "apply_p", None), "_gmres_graphs", None)
    if gb is not None:
        rows["gmres graph buffers (V, Z, z)"] = nbytes([gb.V, gb.Z, gb.z], seen)
    for name, pr in getattr(st, "_proj", {}).items():
        rows[f"projection {name}"] = nbytes([pr.xs, pr.axs], seen)
    total = torch.cuda.memory_allocated(dev)
    rows["unattributed"] = total - sum(rows.values())
    out = {"workload": wl, "size": size, "projection": proj, "points": sp.n_points, "field_gb": F / 1e9,
           "allocated_gb": total / 1e9, "after_setup_gb": after_setup / 1e9,
           "peak_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
           "fields": {k: round(v / F, 2) for k, v in rows.items() if v}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
