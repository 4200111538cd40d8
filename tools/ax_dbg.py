"""Debug helper: run one Ax variant through the bulk kernel at a given mesh size."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import poisson_space  # noqa: E402
from paper_2207_07098_b200 import _lib  # noqa: E402

ne = int(sys.argv[1])
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
sp, mask, f = poisson_space(ne, dev)
L = _lib.load()
_lib.call("sf_set_ax_kernel", kern)
u = torch.randn(sp.shape, dtype=torch.float64, device=dev)
w = torch.empty_like(u)
st = torch.cuda.current_stream().cuda_stream
_lib.call("sf_ax_helm_f64", sp.dmat.ctypes.data, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(), w.data_ptr(),
          sp.n_elements, 1.0, 0.0, 0, st)
torch.cuda.synchronize()
_lib.call("sf_set_ax_kernel", 1 - kern)
w2 = torch.empty_like(u)
_lib.call("sf_ax_helm_f64", sp.dmat.ctypes.data, 8, sp.geom.data_ptr(), sp.bm.data_ptr(), u.data_ptr(), w2.data_ptr(),
          sp.n_elements, 1.0, 0.0, 0, st)
torch.cuda.synchronize()
print("ne", ne, "equal", bool(torch.equal(w, w2)), float((w - w2).abs().max()))
