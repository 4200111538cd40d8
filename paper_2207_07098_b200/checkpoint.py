"""Binary checkpoints and bitwise restart (reference output.py:69-128, runner.py:102-165).

The container is the reference's own format, so checkpoints written by either
implementation restart the other: 8-byte magic ``SEMFCKPT``, uint32 version 1,
uint64 header length, a JSON header ``{"arrays": [{"name", "shape"}...],
"meta": {...}}`` (sort_keys), then the float64 little-endian payloads in
header order.  Device fields are copied to the host only here.

``save_state`` / ``load_state`` carry exactly what the reference's runner
carries -- velocity and explicit-term histories, pressure, the projection
spaces (basis vectors, count, solve counter) and the last scheme order -- so a
restarted run reproduces the uninterrupted one bit for bit
(pkg/tests/test_runner.py:101-115).  On several ranks the element slices are
gathered, so the file is the same for any rank count.
"""

import json

import numpy as np
import torch

from . import dist as _dist
from . import operators
from .errors import CheckpointError, ConfigError
from .timestep import FlowState

MAGIC = b"SEMFCKPT"
VERSION = 1

#: per-step diagnostics CSV of the reference's runner (runner.py:27-28, 92-99)
DIAG_HEADER = ("step,time,cfl,p_iters,p_res,ux_iters,uy_iters,uz_iters,"
               "ux_res,uy_res,uz_res,div_norm,wall_time")


def _fmt(x):
    return f"{float(x):.17g}"


def diag_row(d):
    """One diagnostics.csv row for a StepDiagnostics, formatted as the reference
    writes it (17 significant digits), so runs can be diffed column by column."""
    vi, vr = d.v_iterations, d.v_residual
    return ",".join([str(d.step), _fmt(d.time), _fmt(d.cfl), str(d.p_iterations), _fmt(d.p_residual),
                     str(vi[0]), str(vi[1]), str(vi[2]), _fmt(vr[0]), _fmt(vr[1]), _fmt(vr[2]),
                     _fmt(d.div_norm), _fmt(d.wall_time)])


class Deferred:
    """A checkpoint payload produced while the file is written: ``chunks()`` yields
    host float64 arrays whose concatenation is the array of ``shape``.  Device
    fields are gathered and copied to the host one chunk at a time, so a
    checkpoint never holds more than one field on the device or the host."""

    def __init__(self, shape, chunks):
        self.shape = tuple(int(s) for s in shape)
        self.chunks = chunks


def _host(arr, name):
    a = arr.detach().cpu().numpy() if isinstance(arr, torch.Tensor) else np.asarray(arr)
    if a.dtype != np.float64:
        raise CheckpointError(f"checkpoint arrays must be float64, {name} is {a.dtype}")
    return np.ascontiguousarray(a, dtype="<f8")


def write_checkpoint(path, arrays, meta):
    """Named float64 arrays (or ``Deferred`` payloads) + JSON metadata -> checkpoint
    file (output.py:69-84).  Payloads are streamed to the file in header order."""
    specs = []
    for name, arr in arrays.items():
        if not isinstance(arr, Deferred) and not isinstance(arr, torch.Tensor):
            arr = np.asarray(arr)
        if not isinstance(arr, Deferred) and arr.dtype not in (np.float64, torch.float64):
            raise CheckpointError(f"checkpoint arrays must be float64, {name} is {arr.dtype}")
        specs.append({"name": name, "shape": list(arr.shape)})
    header = json.dumps({"arrays": specs, "meta": meta}, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(np.array(VERSION, dtype="<u4").tobytes())
        fh.write(np.array(len(header), dtype="<u8").tobytes())
        fh.write(header)
        for name, arr in arrays.items():
            if isinstance(arr, Deferred):
                want, got = int(np.prod(arr.shape)) if arr.shape else 1, 0
                for chunk in arr.chunks():
                    a = _host(chunk, name)
                    got += a.size
                    fh.write(a.tobytes())
                if got != want:
                    raise CheckpointError(f"{name}: produced {got} values for shape {arr.shape}")
            else:
                fh.write(_host(arr, name).tobytes())


def read_checkpoint(path):
    """Checkpoint file -> (arrays dict of numpy float64, meta dict) (output.py:87-128).
    Errors name the section and byte offset where the file went wrong."""
    with open(path, "rb") as fh:
        blob = memoryview(fh.read())
    cur = [0]

    def chunk(nbytes, section):
        at = cur[0]
        if at + nbytes > len(blob):
            raise CheckpointError(f"truncated checkpoint: wanted {nbytes} bytes, have {len(blob) - at}",
                                  offset=at, section=section)
        cur[0] = at + nbytes
        return blob[at:at + nbytes]

    magic = bytes(chunk(8, "magic"))
    if magic != MAGIC:
        raise CheckpointError(f"bad magic {magic!r}, expected {MAGIC!r}", offset=0, section="magic")
    version = int(np.frombuffer(chunk(4, "version"), dtype="<u4")[0])
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}, this build reads {VERSION}",
                              offset=8, section="version")
    hlen = int(np.frombuffer(chunk(8, "header_len"), dtype="<u8")[0])
    try:
        header = json.loads(bytes(chunk(hlen, "header")).decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise CheckpointError(f"corrupt JSON header: {exc}", offset=20, section="header") from exc
    arrays = {}
    for spec in header["arrays"]:
        shape = tuple(int(s) for s in spec["shape"])
        count = int(np.prod(shape)) if shape else 1
        arrays[spec["name"]] = np.frombuffer(chunk(8 * count, spec["name"]), dtype="<f8").reshape(shape).copy()
    if cur[0] != len(blob):
        raise CheckpointError(f"{len(blob) - cur[0]} trailing bytes after the last array",
                              offset=cur[0], section="trailer")
    return arrays, header["meta"]


def _starts(space):
    return _dist.element_ranges(space.mesh.n_elements, space.comm.world)


def _local(space, a):
    e0, e1 = space.e_range
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t[..., e0:e1, :, :, :].contiguous().to(space.device)


def _field(sp, t):
    """Deferred payload of one distributed field: the element slices are gathered to
    rank 0 (host numpy there, None elsewhere) when the writer reaches it."""
    shape = tuple(t.shape[:-4]) + (sp.mesh.n_elements,) + tuple(t.shape[-3:])
    return Deferred(shape, lambda: [sp.comm.gather_to_root(t, _starts(sp))])


def _basis(sp, vecs):
    """Deferred (count, P_global) payload of a projection basis, one vector at a time."""
    n = sp.mesh.n_elements * int(np.prod(sp.shape[1:]))
    return Deferred((len(vecs), n),
                    lambda: (sp.comm.gather_to_root(v, _starts(sp)) for v in vecs))


def save_state(path, stepper, state, case="semflow_b200"):
    """Write the runner's checkpoint for (stepper, state) (runner.py:102-126).
    Collective on several ranks: every field is gathered to rank 0 one at a time
    (never the whole state, never on every rank) and rank 0 streams it to the file."""
    sp = stepper.space
    arrays = {}
    for q, v in enumerate(state.vel_hist):
        arrays[f"vel_{q}"] = _field(sp, v)
    for q, nl in enumerate(state.nl_hist):
        arrays[f"nl_{q}"] = _field(sp, nl)
    arrays["prs"] = _field(sp, state.prs)
    proj_meta = {}
    for name, proj in stepper._proj.items():
        if proj.xs:
            arrays[f"proj_{name}_xs"] = _basis(sp, proj.xs)
            arrays[f"proj_{name}_axs"] = _basis(sp, proj.axs)
        proj_meta[name] = {"count": proj.count, "solves": proj._solves}
    meta = {"case": case, "time": state.time, "nsteps": state.nsteps, "primed": state.primed,
            "n_vel_hist": len(state.vel_hist), "n_nl_hist": len(state.nl_hist),
            "last_order": stepper._last_order, "projections": proj_meta,
            "forcing": stepper.forcing.get_state() if stepper.forcing is not None else None}
    if sp.comm.rank == 0:
        write_checkpoint(path, arrays, meta)
    else:   # the same gathers, in the writer's order
        for arr in arrays.values():
            for _ in arr.chunks():
                pass


def load_state(path, stepper):
    """Rebuild a FlowState and the stepper's side state from a checkpoint
    (runner.py:129-165); the device histories are this rank's element slice."""
    sp = stepper.space
    arrays, meta = read_checkpoint(path)
    E = sp.mesh.n_elements
    gshape = (3, E) + sp.shape[1:]
    try:
        vel_hist = [_local(sp, arrays[f"vel_{q}"].reshape(gshape)) for q in range(meta["n_vel_hist"])]
        nl_hist = [_local(sp, arrays[f"nl_{q}"].reshape(gshape)) for q in range(meta["n_nl_hist"])]
        prs = _local(sp, arrays["prs"].reshape(gshape[1:]))
    except (KeyError, ValueError) as exc:
        raise CheckpointError(f"checkpoint does not match this space: {exc}", section="arrays") from exc
    if meta.get("forcing") is not None:
        if stepper.forcing is None:
            raise ConfigError("checkpoint carries tripping state but the case has none")   # runner.py:158-159
        stepper.forcing.set_state(meta["forcing"])
    state = FlowState(time=float(meta["time"]), nsteps=int(meta["nsteps"]), vel_hist=vel_hist,
                      curl_hist=[operators.curl(sp, v) for v in vel_hist], nl_hist=nl_hist, prs=prs,
                      primed=bool(meta["primed"]))
    for name, pm in meta.get("projections", {}).items():
        proj = stepper._proj.get(name)
        if proj is None:
            continue
        proj.invalidate()
        proj._solves = int(pm["solves"])
        if pm["count"]:
            xs = arrays[f"proj_{name}_xs"]
            axs = arrays[f"proj_{name}_axs"]
            proj.xs = [_local(sp, xs[i].reshape(gshape[1:])) for i in range(xs.shape[0])]
            proj.axs = [_local(sp, axs[i].reshape(gshape[1:])) for i in range(axs.shape[0])]
    # the last scheme order keeps projection invalidation on the uninterrupted schedule
    stepper._last_order = meta.get("last_order")
    return state
