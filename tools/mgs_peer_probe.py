"""Cost of the fused NVLink allreduce in the GMRES MGS pass (torchrun, N ranks):

    python -m torch.distributed.run --standalone --nproc-per-node N tools/mgs_peer_probe.py [P_millions]

Each rank holds P/N points (P defaults to config 3's 134.2 M).  Times 50
back-to-back passes (w -= h v_prev; <w, v_next>) with CUDA events, twice each:
the local pass alone (sf_mgs_step_f64, no collective) and the fused pass
(sf_mgs_step_peer_f64, rank partials summed over NVLink in its last block).
Rank 0 prints one JSON line (max over ranks of the per-pass us).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2207_07098_b200 import _device, _lib, dist

    comm = dist.init_from_env()
    dev = torch.device("cuda", torch.cuda.current_device())
    P = int(float(sys.argv[1]) * 1e6) if len(sys.argv) > 1 else 64 ** 3 * 512
    Pl = (P // comm.world) & ~1
    g = torch.Generator(device="cpu").manual_seed(comm.rank)
    w = torch.randn(Pl, generator=g, dtype=torch.float64).to(dev)
    vp = torch.randn(Pl, generator=g, dtype=torch.float64).to(dev)
    vn = torch.randn(Pl, generator=g, dtype=torch.float64).to(dev)
    mult = torch.ones(Pl, dtype=torch.uint8, device=dev)
    h = torch.tensor([1e-12], dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    wk = _device.workspace(dev)
    st = _lib.stream_ptr(dev)
    peer = comm.peer
    args = (_lib.ptr(w), _lib.ptr(vp), _lib.ptr(h), _lib.ptr(vn), None, None, _lib.ptr(mult), 0, Pl)

    def local():
        _lib.call("sf_mgs_step_f64", *args, *wk.args(), _lib.ptr(out), None, st)

    def fused():
        _lib.call("sf_mgs_step_peer_f64", *args, *wk.args(), _lib.ptr(out), *peer.fused_args(), None, st)

    def time(fn, reps=50):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        if comm.world > 1:
            comm.dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([1000.0 * a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        comm.max_(t)
        return float(t.item())

    res = {"world": comm.world, "points_per_rank": Pl, "local_us": time(local)}
    if peer is not None:
        res["fused_us"] = time(fused)
        res["local_us_2"] = time(local)
        res["fused_us_2"] = time(fused)
    bytes_ = Pl * 33
    res["local_GBps"] = bytes_ / (res["local_us"] * 1e3)
    if comm.rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
