"""Per-device runtime state: reduction workspaces, scalar slots, arithmetic mode."""

import os

import torch

from . import _lib

#: production arithmetic (DFMA).  SEMFLOW_B200_EXACT=1 selects the non-contracted
#: reference-order arithmetic everywhere (bit-identical element kernels).
EXACT = os.environ.get("SEMFLOW_B200_EXACT", "0").strip().lower() in ("1", "true", "on")

_WORK = {}


class RedWork:
    """Reduction workspace for one (device, stream): partials + counter + scalar slots.

    Kernels on one stream execute in order, so one workspace per stream is
    enough.  ``slots`` is a device array of scalars the solvers use to pass
    values (rz, pap, h_ij ...) between kernels without host round-trips.
    """

    def __init__(self, device, nslots=256):
        lib = _lib.load()
        nd = lib.sf_red_workspace_doubles()
        self.device = device
        self.partials = torch.zeros(nd, dtype=torch.float64, device=device)
        self.counter = torch.zeros(4, dtype=torch.int32, device=device)
        self.slots = torch.zeros(nslots, dtype=torch.float64, device=device)
        self.pinned = torch.zeros(nslots, dtype=torch.float64, pin_memory=True)

    def args(self):
        return (_lib.ptr(self.partials), _lib.ptr(self.counter))

    def slot(self, i):
        """Device address of scalar slot i."""
        return self.slots.data_ptr() + 8 * i

    def read(self, i, n=1):
        """Blocking read of slots[i:i+n] to host floats."""
        self.pinned[:n].copy_(self.slots[i:i + n], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return [float(v) for v in self.pinned[:n].tolist()]


def workspace(device=None):
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    w = _WORK.get(key)
    if w is None:
        w = RedWork(dev)
        _WORK[key] = w
    return w
