"""Partitioned vs global build of the gather-scatter numbering on the config-5
cylinder mesh, under torchrun (one rank per GPU):

    torchrun --standalone --nproc-per-node N tools/partition_check.py [analogue] [<scale> ...]

For the 9 728-element config-5 analogue (tests/golden/make_golden.py
CYL_MESHES) and each scale of cylinder_params (2: 252 928 elements) every rank builds its space twice -- SEMFLOW_B200_GLOBAL_BUILD=1 (every
rank numbers the whole mesh) and the default partitioned build -- and compares
its gid slice, multiplicities, shared maps and halo send lists bit for bit.
Rank 0 prints one JSON line.
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

    comm = dist.init_from_env()
    dev = torch.device("cuda", torch.cuda.current_device())
    out = []
    analogue = dict(diameter=1.0, xlim=(-50.0, 120.0), zlim=(-25.0, 25.0), height=10.0, n_azimuthal=32,
                    n_radial=8, n_axial=4, n_upstream=16, n_downstream=32, n_front=16, n_back=16, geom_order=7)
    for scale in sys.argv[1:] or ["analogue", "2"]:
        mesh = gen_cylinder_box_mesh(**(analogue if scale == "analogue" else cylinder_params(int(scale))))
        sps, times = {}, {}
        for mode in ("global", "partitioned"):
            os.environ["SEMFLOW_B200_GLOBAL_BUILD"] = "1" if mode == "global" else "0"
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sp = build_space(mesh, make_basis(7), device=dev, comm=comm)
            torch.cuda.synchronize()
            times[mode] = round(time.perf_counter() - t0, 2)
            g = sp.gs
            sps[mode] = {"gid": g.gid.clone(), "mult": g.mult8.clone(), "sh_off": g.sh_off.clone(),
                         "sh_perm": g.sh_perm.clone(), "n_gid": g.n_gid,
                         "send": {q: t.clone() for q, t in g.plan.send_idx.items()},
                         "n_recv": dict(g.plan.n_recv)}
            del sp, g
            torch.cuda.empty_cache()
        a, b = sps["global"], sps["partitioned"]
        ok = {k: bool(torch.equal(a[k], b[k])) for k in ("gid", "mult", "sh_off", "sh_perm")}
        ok["n_gid"] = a["n_gid"] == b["n_gid"]
        ok["halo"] = (a["n_recv"] == b["n_recv"] and set(a["send"]) == set(b["send"])
                      and all(torch.equal(a["send"][q], b["send"][q]) for q in a["send"]))
        rows = [None] * comm.world
        torch.distributed.all_gather_object(rows, {"rank": comm.rank, "ok": ok, "build_s": times})
        out.append({"scale": scale, "E": int(mesh.n_elements), "ranks": rows,
                    "all_equal": all(all(r["ok"].values()) for r in rows)})
    if comm.rank == 0:
        print(json.dumps({"world": comm.world, "meshes": out}), flush=True)
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
