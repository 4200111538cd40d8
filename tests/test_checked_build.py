"""The checked build (libsemflow_b200_checked.so, device bounds checks; the pool
closes compute-sanitizer): it loads and exports the same ABI, runs the hot path
clean, and traps on a corrupted index instead of reading out of bounds.  The
trap test faults the GPU on purpose (a device trap is reported as Xid 13 on the
host), so it runs only when SEMFLOW_B200_TRAP_TEST=1 (its recorded run:
profiles/r2_checked_build_gpu_suite.log)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2207_07098_b200", "libsemflow_b200_checked.so")

pytestmark = pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build missing (build.py --checked)")

_PROG = r"""
import sys
sys.path.insert(0, {root!r})
import torch
from paper_2207_07098_b200 import _lib
assert _lib.LIB_PATH.endswith("_checked.so"), _lib.LIB_PATH
from paper_2207_07098_b200 import operators as ops
from paper_2207_07098_b200.basis import make_basis
from paper_2207_07098_b200.mesh import gen_box_mesh
from paper_2207_07098_b200.precond import HybridSchwarz
from paper_2207_07098_b200.space import build_space
dev = torch.device("cuda", 0)
sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (3, 3, 2)), make_basis(5), device=dev)
u = torch.randn(sp.shape, dtype=torch.float64, device=dev)
w = ops.make_global_op(sp, 1.0, 0.3)(u)
M = HybridSchwarz(sp)
z = M(sp.gs.avg(u))
torch.cuda.synchronize()
if {corrupt}:
    M.sub.view(-1)[7] = M.L + 5          # out of range of rw (L + 1 entries)
    z = M(sp.gs.avg(u))
    torch.cuda.synchronize()
print("clean", float(w.abs().max()), float(z.abs().max()))
"""


def _run(corrupt):
    env = dict(os.environ, SEMFLOW_B200_CHECKED="1")
    return subprocess.run([sys.executable, "-c", _PROG.format(root=ROOT, corrupt=corrupt)], env=env,
                          capture_output=True, text=True, timeout=600)


def test_checked_library_exports():
    import ctypes

    from paper_2207_07098_b200 import _lib

    lib = ctypes.CDLL(CHECKED)
    for name in _lib.EXPORTED:
        assert hasattr(lib, name), name


@pytest.mark.gpu
def test_checked_build_runs_clean():
    res = _run(False)
    assert res.returncode == 0 and "clean" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.skipif(os.environ.get("SEMFLOW_B200_TRAP_TEST", "0") != "1",
                    reason="deliberately faults the GPU (device trap, Xid 13): opt-in with SEMFLOW_B200_TRAP_TEST=1")
def test_checked_build_traps_bad_index():
    res = _run(True)
    assert res.returncode != 0
    assert "SF_CHECK failed" in res.stdout + res.stderr
