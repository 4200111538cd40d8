"""Run the n=8 Ax kernels a few times at ne^3 (for ncu captures)."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from bench import poisson_space  # noqa: E402
from paper_2207_07098_b200.operators import GlobalOp  # noqa: E402


def main():
    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    dev = torch.device("cuda", 0)
    sp, mask, f = poisson_space(ne, dev)
    op = GlobalOp(sp, 1.0, 0.0, mask)
    u = torch.randn(sp.shape, dtype=torch.float64, device=dev)
    w = torch.empty_like(u)
    for _ in range(3):
        op.apply_into(u, w)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
