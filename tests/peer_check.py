"""NVLink peer allreduce check (torchrun, one rank per GPU):

    torchrun --standalone --nproc-per-node 2 tests/peer_check.py

Every rank reduces [rank + 1, 0.5 * rank, -rank, 7] many times, with in-place
and separate in/out buffers, and compares with the expected rank-order sums.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    from paper_2207_07098_b200 import dist

    comm = dist.init_from_env()
    r, W = comm.rank, comm.world
    dev = torch.device("cuda", torch.cuda.current_device())
    assert comm.peer is not None, "peer reducer not set up"
    want = torch.tensor([sum(q + 1.0 for q in range(W)), sum(0.5 * q for q in range(W)),
                         sum(-float(q) for q in range(W)), 7.0 * W], dtype=torch.float64)
    bad = 0
    for it in range(200):
        t = torch.tensor([r + 1.0, 0.5 * r, -float(r), 7.0], dtype=torch.float64, device=dev)
        comm.sum_(t)
        got = t.cpu()
        if not torch.equal(got, want):
            bad += 1
            if bad < 4:
                print(f"rank {r} iter {it}: got {got.tolist()} want {want.tolist()}", flush=True)
    comm.peer.check()
    print(f"rank {r}: {200 - bad}/200 ok, error flag {int(comm.peer.error.item())}", flush=True)
    comm.close()
    torch.distributed.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
