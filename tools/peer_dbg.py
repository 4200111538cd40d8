import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2207_07098_b200 import dist, _lib
comm = dist.init_from_env()
r = comm.rank
dev = torch.device("cuda", torch.cuda.current_device())
p = comm.peer
for trial in range(3):
    a = torch.tensor([r + 1.0, 0.5 * r, -float(r), 7.0], dtype=torch.float64, device=dev)
    b = torch.zeros(4, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    print("rank", r, "before", a.tolist(), flush=True)
    p.seq += 1
    _lib.call("sf_peer_allreduce_f64", p.boxes, comm.world, r, p.seq, _lib.ptr(p.error), _lib.ptr(a), 4, _lib.ptr(b), _lib.stream_ptr(dev))
    torch.cuda.synchronize()
    print("rank", r, "in after", a.tolist(), "out", b.tolist(), flush=True)
torch.distributed.destroy_process_group()
