"""Bandwidth of the Krylov vector kernels at a given size vs a torch elementwise reference.

    python tools/vec_bench.py [P_millions]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e-3


def main():
    from paper_2207_07098_b200 import _device, _lib

    P = int(float(sys.argv[1]) * 1e6) if len(sys.argv) > 1 else 134217728
    dev = torch.device("cuda", 0)
    _lib.load(os.environ.get("SF_LIB", _lib.LIB_PATH))
    print("library:", os.environ.get("SF_LIB", _lib.LIB_PATH))
    w = torch.randn(P, dtype=torch.float64, device=dev)
    v1 = torch.randn(P, dtype=torch.float64, device=dev)
    v2 = torch.randn(P, dtype=torch.float64, device=dev)
    m8 = torch.randint(1, 9, (P,), dtype=torch.uint8, device=dev)
    h = torch.tensor([1e-3, 0.0], dtype=torch.float64, device=dev)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    wk = _device.workspace(dev)
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    res["torch w.add_(v,-h) (24 B/pt)"] = (timeit(lambda: w.add_(v1, alpha=-1e-3)), 24)
    res["torch copy (16 B/pt)"] = (timeit(lambda: w.copy_(v1)), 16)
    res["mgs prev+next (33 B/pt)"] = (timeit(lambda: _lib.call(
        "sf_mgs_step_f64", w.data_ptr(), v1.data_ptr(), h.data_ptr(), v2.data_ptr(), None, None, m8.data_ptr(),
        0, P, *wk.args(), out.data_ptr(), None, st)), 33)
    res["mgs next+norm (17 B/pt)"] = (timeit(lambda: _lib.call(
        "sf_mgs_step_f64", w.data_ptr(), None, None, v2.data_ptr(), None, None, m8.data_ptr(),
        1, P, *wk.args(), out.data_ptr(), None, st)), 17)
    pa = (ctypes.c_void_p * 1)(w.data_ptr())
    pb = (ctypes.c_void_p * 1)(v1.data_ptr())
    res["glsc3 (17 B/pt)"] = (timeit(lambda: _lib.call(
        "sf_glsc3_f64", 1, pa, pb, m8.data_ptr(), P, *wk.args(), out.data_ptr(), st)), 17)
    h[0] = 2.0
    res["scale_div (16 B/pt)"] = (timeit(lambda: _lib.call(
        "sf_scale_div_f64", v2.data_ptr(), v1.data_ptr(), None, None, h.data_ptr(), P, st)), 16)
    h[0] = 1.0
    res["scale_div in place (16 B/pt)"] = (timeit(lambda: _lib.call(
        "sf_scale_div_f64", w.data_ptr(), w.data_ptr(), None, None, h.data_ptr(), P, st)), 16)
    for k, (t, b) in res.items():
        print(f"{k:32s} {t * 1e6:9.1f} us  {P * b / t / 1e9:7.0f} GB/s")


if __name__ == "__main__":
    main()
