"""Time the strong-form derivative kernels at ne^3 (CUDA events)."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2207_07098_b200 import operators as ops  # noqa: E402
from paper_2207_07098_b200.timestep import tgv_problem  # noqa: E402


def main():
    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    sp, st, state = tgv_problem(ne, device=torch.device("cuda", 0))
    v = state.vel
    for name, fn in (("grad", lambda: ops.grad(sp, v[0])), ("div", lambda: ops.div(sp, v)),
                     ("curl", lambda: ops.curl(sp, v)), ("advect", lambda: ops.advect_vec(sp, v, v, sign=-1.0)),
                     ("cdtp", lambda: ops.weak_grad_dot(sp, v))):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{name:7s} {a.elapsed_time(b) / 10 * 1e3:9.1f} us", flush=True)


if __name__ == "__main__":
    main()
