"""Per-rank set-up cost of build_space under torchrun: wall time and peak device
memory of the partitioned build (default) and of the global build
(SEMFLOW_B200_GLOBAL_BUILD=1), on the config-5 cylinder mesh at a given scale.

    torchrun --standalone --nproc-per-node N tools/setup_mem.py <scale> [global]

Rank 0 prints one JSON line with every rank's numbers.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2207_07098_b200 import dist
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_cylinder_box_mesh
    from paper_2207_07098_b200.space import build_space
    from paper_2207_07098_b200.timestep import cylinder_params

    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    if len(sys.argv) > 2 and sys.argv[2] == "global":
        os.environ["SEMFLOW_B200_GLOBAL_BUILD"] = "1"
    comm = dist.init_from_env()
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    mesh = gen_cylinder_box_mesh(**cylinder_params(scale))
    t_mesh = time.perf_counter() - t0
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base = torch.cuda.memory_allocated(dev)
    t0 = time.perf_counter()
    sp = build_space(mesh, make_basis(7), device=dev, comm=comm)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    peak = torch.cuda.max_memory_allocated(dev) - base
    held = torch.cuda.memory_allocated(dev) - base
    row = {"rank": comm.rank, "elements": sp.n_elements, "points": sp.n_points, "build_s": round(t_build, 2),
           "peak_gb": round(peak / 1e9, 2), "held_gb": round(held / 1e9, 2), "n_gid": sp.gs.n_gid}
    rows = [None] * comm.world
    torch.distributed.all_gather_object(rows, row)
    if comm.rank == 0:
        print(json.dumps({"scale": scale, "E": int(mesh.n_elements), "world": comm.world,
                          "build": "global" if os.environ.get("SEMFLOW_B200_GLOBAL_BUILD") == "1" else "partitioned",
                          "mesh_gen_s": round(t_mesh, 1), "ranks": rows}), flush=True)
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
