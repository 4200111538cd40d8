import os, time, torch, torch.distributed as dist
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
r, w = dist.get_rank(), dist.get_world_size()
for nbytes in (8 * 147456, 8 * 1024 * 1024):
    n = nbytes // 8
    s = torch.randn(n, device="cuda", dtype=torch.float64); rcv = torch.empty_like(s)
    q = 1 - r
    for it in range(30):
        if it == 10:
            torch.cuda.synchronize(); dist.barrier(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
        ops = [dist.P2POp(dist.irecv, rcv, q), dist.P2POp(dist.isend, s, q)]
        for wk in dist.batch_isend_irecv(ops): wk.wait()
    e1.record(); torch.cuda.synchronize()
    if r == 0: print("bytes", nbytes, "us per exchange", e0.elapsed_time(e1) * 1e3 / 20, flush=True)
dist.destroy_process_group()
