"""Apply the hybrid Schwarz preconditioner of the TGV pressure operator on an
ne^3 lx=8 box twice (ncu captures of the sch_* kernels) and time one
application with CUDA events:

    python tools/schwarz_probe.py <ne>
    ncu --set full -k regex:sch_ -c 12 -o out python tools/schwarz_probe.py 32
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.precond import HybridSchwarz
    from paper_2207_07098_b200.space import build_space

    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    dev = torch.device("cuda", 0)
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0, L, 0, L, 0, L), (ne, ne, ne)), make_basis(7), device=dev)
    t0 = time.perf_counter()
    M = HybridSchwarz(sp)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    r = torch.randn(sp.shape, dtype=torch.float64, generator=torch.Generator().manual_seed(2)).to(dev)
    z = torch.empty_like(r)
    for _ in range(2):
        M.apply_into(r, z)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    reps = 10
    for _ in range(reps):
        M.apply_into(r, z)
    ev[1].record()
    torch.cuda.synchronize()
    us = ev[0].elapsed_time(ev[1]) / reps * 1e3
    # per-stage device time of one application (CUDA events around each stage)
    from paper_2207_07098_b200 import _lib
    import ctypes

    st = ctypes.addressof(M._st)
    stream = _lib.stream_ptr(dev)
    stages = {}

    def tick(name, fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        stages[name] = round(a.elapsed_time(b) * 1e3, 1)

    tick("gather", lambda: _lib.call("sf_schwarz_gather_f64", st, _lib.ptr(r), stream))
    tick("restrict", lambda: _lib.call("sf_schwarz_restrict_f64", st, stream))
    tick("coarse", lambda: _lib.call("sf_schwarz_coarse_f64", st, stream))
    tick("gather_rw", lambda: _lib.call("sf_schwarz_gather_rw_f64", st, stream))

    def gemms():
        rwg, sol = M.rwg.view(-1, M.S), M.sol.view(-1, M.S)
        for c, a_, b_ in M.blocks:
            torch.matmul(rwg[a_:b_], M.invT[c], out=sol[a_:b_])
    tick("class_gemms", gemms)
    tick("finalize", lambda: _lib.call("sf_schwarz_finalize_f64", st, stream))
    tick("scatter", lambda: _lib.call("sf_schwarz_scatter_f64", st, _lib.ptr(z), stream))
    E, S, U = sp.n_elements, M.S, M.n_classes
    print(json.dumps({"ne": ne, "points": sp.n_points, "setup_s": round(t_setup, 2), "classes": U, "S": S,
                      "apply_us": round(us, 1), "stages_us": stages,
                      "local_solve_gflop": round(2.0 * E * S * S / 1e9, 2),
                      "mem_gb": round(torch.cuda.max_memory_allocated(dev) / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
