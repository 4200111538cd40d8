"""Multi-GPU parity on the GPU box (driver-visible): runs tests/mgpu_check.py under
torchrun on 2 GPUs (and 4 when visible) and requires every check to pass --
partitioned dssum / masked operator bitwise equal to one GPU, the reference's TGV
iteration counts with graph-captured multi-rank GMRES, 10^4 gated fused NVLink
reductions exact, and a graph-replayed halo dssum bitwise.  Skipped with fewer
than two GPUs.  Each run's JSON line is kept in gpurun_out/mgpu_<N>.json."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_mgpu_parity(world):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs (have {_gpus()})")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(world),
           os.path.join(ROOT, "tests", "mgpu_check.py"), "8", "10"]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    line = next((ln for ln in p.stdout.splitlines() if ln.startswith("{")), None)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"mgpu_{world}.json"), "w") as fh:
        fh.write((line or "") + "\n")
    assert p.returncode == 0 and line is not None, p.stdout[-3000:] + p.stderr[-3000:]
    res = json.loads(line)
    assert res["ok"], res["checks"]
    assert res["checks"]["halo_path"] == "ipc"
