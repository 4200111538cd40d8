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


class FieldWork:
    """Named field-sized scratch buffers of one space, allocated on first use and
    kept: the time step and the solvers take every temporary from here, so after
    the first step the device allocator sees only the fields a step returns (new
    state, solver iterates) and never has to map new memory inside a step (at
    64^3 each cudaMalloc of a GB-sized segment stalled the stream for ~57 ms).

    ``get(name, shape)`` returns the same tensor for the same (name, shape); the
    caller owns it until its next ``get`` with that name.  Names are unique per use
    site, so buffers of different call sites never alias."""

    def __init__(self, device):
        self.device = device
        self._bufs = {}

    def get(self, name, shape):
        key = (name, tuple(shape))
        t = self._bufs.get(key)
        if t is None:
            t = torch.empty(key[1], dtype=torch.float64, device=self.device)
            self._bufs[key] = t
        return t

    def like(self, name, t):
        return self.get(name, t.shape)

    def nbytes(self):
        return sum(t.numel() * 8 for t in self._bufs.values())


def field_work(space):
    """The FieldWork of a space (created on first use)."""
    w = getattr(space, "_field_work", None)
    if w is None:
        w = FieldWork(space.device)
        space._field_work = w
    return w
