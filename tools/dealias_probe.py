"""Run the fused over-integrated convection (sf_dealias_advect_f64) twice on an
ne^3 lx=8 box and time one call with CUDA events (ncu target):

    python tools/dealias_probe.py <ne>
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2207_07098_b200 import operators as ops
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space

    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    dev = torch.device("cuda", 0)
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0, L, 0, L, 0, L), (ne, ne, ne)), make_basis(7), device=dev)
    dl = ops.Dealias(sp)
    g = torch.Generator().manual_seed(1)
    c = torch.randn((3,) + sp.shape, generator=g, dtype=torch.float64).to(dev)
    out = torch.empty_like(c)
    for _ in range(2):
        dl.advect_vec(c, c, sign=-1.0, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        dl.advect_vec(c, c, sign=-1.0, out=out)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 5 * 1e3
    E = sp.n_elements
    # HBM bytes: c, v (6 fields), rx (9), wjac_f (m^3/n^3 = 3.375), bm (1), out (3)
    gb = E * 512 * 8 * (6 + 9 + 3.375 + 1 + 3) / 1e9
    print(json.dumps({"ne": ne, "points": sp.n_points, "us": round(us, 1), "hbm_gb": round(gb, 3),
                      "gbs": round(gb / us * 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
