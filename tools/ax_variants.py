"""Build and time Ax_helm kernel variants (register bound / unroll) and dssum at 32^3.

    python tools/ax_variants.py build      # here (nvcc), writes paper_2207_07098_b200/variants/*.so
    python tools/ax_variants.py run [ne]   # on the GPU box
"""
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2207_07098_b200", "variants")
# e.g. {"minb5": "-DSF_AX8S_MINB=5"}: MINB 3/5 and unroll 1/4 measured slower; so
# was a register-resident r-flux (f1 contracted into 8 per-thread accumulators as
# each layer is formed, bit-identical output): 275 / 255 (unroll 1) vs 234 us
# masked at 32^3, 2141 vs 1774 us at 64^3; storing the pass-through value of
# masked unshared points at load time instead of re-loading it: 234.0 vs 234.0 us
VARIANTS = {}


def build():
    from concurrent.futures import ThreadPoolExecutor

    from paper_2207_07098_b200 import build as b

    os.makedirs(VDIR, exist_ok=True)
    srcs = b.sources()

    def one(item):
        name, flags = item
        out = os.path.join(VDIR, f"lib_{name}.so")
        cmd = ["nvcc", *b.NVCC_FLAGS, "-shared", *flags.split(), "-o", out, *srcs]
        subprocess.run(cmd, check=True)
        return out

    with ThreadPoolExecutor(4) as ex:
        print(list(ex.map(one, VARIANTS.items())))


def run(ne):
    import numpy as np
    import torch

    from paper_2207_07098_b200 import _lib
    from bench import poisson_space

    dev = torch.device("cuda", 0)
    sp, mask, f = poisson_space(ne, dev)
    from paper_2207_07098_b200.operators import GlobalOp

    op = GlobalOp(sp, 1.0, 0.0, mask)
    u = torch.randn(sp.shape, dtype=torch.float64, device=dev)
    w = torch.empty_like(u)
    st = torch.cuda.current_stream().cuda_stream
    P = sp.n_points
    gs = sp.gs
    paths = [_lib.LIB_PATH] if os.environ.get("AX_MAIN_ONLY") else \
        [_lib.LIB_PATH] + sorted(glob.glob(os.path.join(VDIR, "lib_*.so")))
    ref_out = {}   # the main library's outputs: every variant must match them bit for bit
    for path in paths:
        L = ctypes.CDLL(path)
        for name, args in _lib._SIGS.items():
            getattr(L, name).argtypes = args
        L.sf_last_error.restype = ctypes.c_char_p
        res = {}
        for kind in ("masked", "plain", "dssum", "dssum_blk", "helm"):
            def fn():
                if kind == "masked":
                    L.sf_ax_masked_f64(sp.dmat.ctypes.data, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(),
                                       w.data_ptr(), sp.n_elements, 1.0, 0.0, op.inmask.data_ptr(),
                                       op.outsel.data_ptr(), 0, st)
                elif kind == "plain":
                    L.sf_ax_helm_f64(sp.dmat.ctypes.data, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(),
                                     w.data_ptr(), sp.n_elements, 1.0, 0.0, 0, st)
                elif kind == "helm":
                    L.sf_ax_masked_f64(sp.dmat.ctypes.data, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(),
                                       w.data_ptr(), sp.n_elements, 1.0 / 1600, 183.3, op.inmask.data_ptr(),
                                       op.outsel.data_ptr(), 0, st)
                elif kind == "dssum_blk":
                    if not hasattr(gs, "cls_nb"):
                        gs._build_classes()
                    n2, n4, n8 = gs.cls_n
                    L.sf_dssum_blk_f64(w.data_ptr(), op.sh_perm.data_ptr(), n2, n4, n8, gs.cls_gen_off.data_ptr(),
                                       gs.cls_bstart.data_ptr(), gs.cls_nb, 2, u.data_ptr(), None, None, 0, st)
                else:
                    if hasattr(L, "sf_dssum_cls_f64"):
                        n2, n4, n8 = gs.cls_n
                        L.sf_dssum_cls_f64(w.data_ptr(), op.sh_perm.data_ptr(), n2, n4, n8,
                                           gs.cls_gen_off.data_ptr(), gs.cls_n_gen, 2, u.data_ptr(), None, 0, st)
                    else:   # CSR layout (older builds): the plain shared maps
                        L.sf_dssum_f64(w.data_ptr(), gs.sh_off.data_ptr(), gs.masked_perm_csr.data_ptr(),
                                       gs.n_shared, 2, u.data_ptr(), None, 0, st)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            if kind in ("masked", "plain", "helm"):
                if kind not in ref_out:
                    ref_out[kind] = w.clone()
                elif not torch.equal(ref_out[kind], w):
                    print("   ", kind, "MISMATCH vs main library, max diff",
                          float((ref_out[kind] - w).abs().max()), flush=True)
            err = L.sf_last_error()
            if err:
                print("   ", kind, "error:", err)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
            torch.cuda.synchronize()
            for a, b in ev:
                a.record()
                fn()
                b.record()
            torch.cuda.synchronize()
            res[kind] = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3
        if hasattr(L, "sf_ax_dssum8_f64"):
            for cpl in os.environ.get("AX_CHUNKS", "592").split(","):
                cp, lag = (int(x) for x in (cpl.split(":") + ["1"])[:2])
                plans = {"fmasked": gs.fused_plan(op.sh_perm, chunk_pairs=cp, lag=lag),
                         "fplain": gs.fused_plan(None, chunk_pairs=cp, lag=lag)}
                for kind, pl in plans.items():
                    m = kind == "fmasked"

                    def fn():
                        L.sf_ax_dssum8_f64(sp.dmat.ctypes.data, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(),
                                           w.data_ptr(), sp.n_elements, 1.0, 0.0,
                                           op.inmask.data_ptr() if m else None, op.outsel.data_ptr() if m else None,
                                           2 if m else 0, *pl.launch_args(), 0, st)
                    for _ in range(3):
                        fn()
                    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
                    torch.cuda.synchronize()
                    for a, b in ev:
                        a.record()
                        fn()
                        b.record()
                    torch.cuda.synchronize()
                    res[f"{kind}{cpl}"] = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3
        gbs = P * 64 / (res["masked"] * 1e-6) / 1e9
        print(f"{os.path.basename(path):24s} masked {res['masked']:8.1f} us ({gbs:6.0f} GB/s)  plain {res['plain']:8.1f} us"
              f"  dssum {res['dssum']:7.1f} us  dssum_blk {res['dssum_blk']:7.1f} us  helm {res['helm']:7.1f} us",
              flush=True)
        fk = {k: round(v, 1) for k, v in res.items() if k.startswith("f")}
        if fk:
            print("   fused:", fk, flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 32)
