"""A/B of the two n = 8 Ax kernels (sf_set_ax_kernel 0 = register prefetch,
1 = bulk-copy ring): bitwise agreement on every variant, then CUDA-event timings.

    python tools/ax_ab.py [ne] [--exact]     # on the GPU box

Prints one line per variant: both kernels' median us over 20 back-to-back
launches (inputs larger than L2 from ne = 32), the algorithmic GB/s of the new
kernel and whether the outputs are bit-identical; then the masked Poisson
operator (Ax + dssum) on the config-2 mesh.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from bench import poisson_space
    from paper_2207_07098_b200 import _lib
    from paper_2207_07098_b200.operators import GlobalOp

    ne = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 32
    exact = 1 if "--exact" in sys.argv else 0
    dev = torch.device("cuda", 0)
    sp, mask, f = poisson_space(ne, dev)
    L = _lib.load()
    op = GlobalOp(sp, 1.0, 0.0, mask)
    g = torch.Generator(device="cpu").manual_seed(3)
    u = torch.randn(sp.shape, generator=g, dtype=torch.float64).to(dev)
    pre = (torch.rand(sp.shape, generator=g, dtype=torch.float64) + 0.5).to(dev)
    w = torch.empty_like(u)
    st = torch.cuda.current_stream().cuda_stream
    P = sp.n_points
    E = sp.n_elements
    D = sp.dmat.ctypes.data
    im, os_ = op.inmask.data_ptr(), op.outsel.data_ptr()
    # (name, call, algorithmic bytes per point)
    variants = {
        "plain": (lambda: L.sf_ax_helm_f64(D, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(), w.data_ptr(),
                                           E, 1.0, 0.0, exact, st), 64),
        "masked": (lambda: L.sf_ax_masked_f64(D, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(), w.data_ptr(),
                                              E, 1.0, 0.0, im, os_, exact, st), 64),
        "helm_masked": (lambda: L.sf_ax_masked_f64(D, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(),
                                                   w.data_ptr(), E, 1.0 / 1600, 183.3, im, os_, exact, st), 72),
        "pre": (lambda: L.sf_ax_pre_f64(D, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(), pre.data_ptr(),
                                        w.data_ptr(), E, 1.0, 0.0, None, None, exact, st), 72),
        "pre_masked": (lambda: L.sf_ax_pre_f64(D, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(),
                                               pre.data_ptr(), w.data_ptr(), E, 1.0, 0.0, im, os_, exact, st), 72),
        "range_mid": (lambda: L.sf_ax_range_f64(D, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(), None,
                                                w.data_ptr(), E, 2 * (E // 8), 2 * (E // 4), 1.0, 0.0, im, os_,
                                                exact, st), 64),
    }

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in ev:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3

    rows = []
    for name, (fn, bpp) in variants.items():
        out = {}
        t = {}
        for kern in (0, 1):
            _lib.call("sf_set_ax_kernel", kern)
            w.fill_(float("nan"))
            fn()
            torch.cuda.synchronize()
            err = L.sf_last_error()
            out[kern] = w.clone()
            t[kern] = timed(fn)
        npts = P if name != "range_mid" else (2 * (E // 4) - 2 * (E // 8)) * 512
        same = bool(torch.equal(out[0].nan_to_num(7.0), out[1].nan_to_num(7.0)))
        diff = float((out[0] - out[1]).abs().nan_to_num(1e300).max())
        row = {"variant": name, "us_reg": round(t[0], 1), "us_bulk": round(t[1], 1),
               "GBps_bulk": round(npts * bpp / (t[1] * 1e-6) / 1e9), "bitwise": same, "maxdiff": diff,
               "err": err.decode() if err else ""}
        rows.append(row)
        print(json.dumps(row), flush=True)
    # the masked Poisson operator (config 2): Ax + dssum through the library
    for kern in (0, 1):
        _lib.call("sf_set_ax_kernel", kern)
        ta = timed(lambda: op.apply_into(u, w))
        print(json.dumps({"operator": "masked Poisson Ax+dssum", "ax_kernel": kern, "us": round(ta, 1),
                          "GBps_alg": round(1279.6e6 * (ne / 32) ** 3 / (ta * 1e-6) / 1e9)}), flush=True)
    _lib.call("sf_set_ax_kernel", 1)


if __name__ == "__main__":
    main()
