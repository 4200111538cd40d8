"""B200 kernel lane: drop-in for the reference plugin API ``semflow.kernels``.

Exports the seven callables of semflow/kernels/__init__.py:47-53 with the same
host-numpy signatures and ownership rules (fresh outputs; ``gs_scatter`` writes
``out`` in place and returns it), plus ``lane_name()`` and
``set_num_threads()``.  Each call copies its operands to the current CUDA device,
runs the sm_100a kernel from libsemflow_b200.so and copies the result back, so
it proves parity but not speed -- the device-resident API
(:mod:`paper_2207_07098_b200.space` / ``operators`` / ``krylov``) is the
performance boundary.

Arithmetic is the reference numba lane's, operation for operation and without
FMA contraction (``exact=1`` in the C ABI), so outputs are bit-identical to
``semflow.kernels._numba`` (tests/test_gpu_parity.py lane tests).  Install into
the reference with :func:`install`; tests/test_ref_hosted.py runs the
reference's own test suite with this lane installed.
"""

import numpy as np
import torch

from . import _lib

LANE = "b200"


def _dev():
    if not torch.cuda.is_available():
        raise _lib.LibraryError("the b200 lane needs a CUDA device (no CPU fallback)")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=_dev(), dtype=dtype)


def _apply(axis, a, u):
    a = np.asarray(a, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    e, n1, n2, n3 = u.shape
    m, n = a.shape
    if n != (n1, n2, n3)[axis]:
        raise ValueError(f"contraction size mismatch: a is {a.shape}, u is {u.shape}")
    shape = [e, n1, n2, n3]
    shape[1 + axis] = m
    ad, ud = _to_dev(a), _to_dev(u)
    out = torch.empty(shape, dtype=torch.float64, device=ud.device)
    _lib.call("sf_apply_axis3_f64", axis, _lib.ptr(ad), m, n1, n2, n3, _lib.ptr(ud), _lib.ptr(out), e, 1,
              _lib.stream_ptr())
    return out.cpu().numpy()


def apply_r(a, u):
    """out[e,p,j,k] = sum_i a[p,i] u[e,i,j,k]  (reference _numba.py:15-28)."""
    return _apply(0, a, u)


def apply_s(a, u):
    """out[e,i,p,k] = sum_j a[p,j] u[e,i,j,k]  (reference _numba.py:31-44)."""
    return _apply(1, a, u)


def apply_t(a, u):
    """out[e,i,j,p] = sum_k a[p,k] u[e,i,j,k]  (reference _numba.py:47-60)."""
    return _apply(2, a, u)


def grad_ref(d, u):
    """(du/dr, du/ds, du/dt)  (reference _numba.py:63-83)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    e, n = u.shape[0], u.shape[1]
    ud = _to_dev(u)
    outs = [torch.empty_like(ud) for _ in range(3)]
    _lib.call("sf_grad_ref_f64", d.ctypes.data, n, _lib.ptr(ud), *(_lib.ptr(o) for o in outs), e,
              1, _lib.stream_ptr())
    return tuple(o.cpu().numpy() for o in outs)


def ax_helmholtz_local(d, g, b, u, lam_visc, lam_mass):
    """w = lam_visc D^T G D u + lam_mass B u per element (reference _numba.py:86-131)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    e, n = u.shape[0], u.shape[1]
    ud, gd, bd = _to_dev(u), _to_dev(g), _to_dev(b)
    w = torch.empty_like(ud)
    _lib.call("sf_ax_helm_f64", d.ctypes.data, n, _lib.ptr(gd), _lib.ptr(bd), _lib.ptr(ud),
              _lib.ptr(w), e, float(lam_visc), float(lam_mass), 1, _lib.stream_ptr())
    return w.cpu().numpy()


def gs_gather(vals, perm, offsets):
    """Per-gid sequential sums in perm order (reference _numba.py:134-143)."""
    n_gid = int(np.asarray(offsets).shape[0]) - 1
    vd = _to_dev(np.asarray(vals, dtype=np.float64))
    pd = _to_dev(np.asarray(perm, dtype=np.int64), torch.int64)
    od = _to_dev(np.asarray(offsets, dtype=np.int64), torch.int64)
    sums = torch.empty(max(n_gid, 0), dtype=torch.float64, device=vd.device)
    _lib.call("sf_gs_gather_f64", _lib.ptr(vd), _lib.ptr(pd), _lib.ptr(od), n_gid, _lib.ptr(sums),
              _lib.stream_ptr())
    return sums.cpu().numpy()


def gs_scatter(sums, perm, offsets, out):
    """out[perm[o]] = sums[g], written in place into ``out`` (reference _numba.py:146-153)."""
    n_gid = int(np.asarray(offsets).shape[0]) - 1
    sd = _to_dev(np.asarray(sums, dtype=np.float64))
    pd = _to_dev(np.asarray(perm, dtype=np.int64), torch.int64)
    od = _to_dev(np.asarray(offsets, dtype=np.int64), torch.int64)
    outd = _to_dev(out)
    _lib.call("sf_gs_scatter_f64", _lib.ptr(sd), _lib.ptr(pd), _lib.ptr(od), n_gid,
              _lib.ptr(outd), _lib.stream_ptr())
    out[...] = outd.cpu().numpy()
    return out


def lane_name():
    return LANE


def set_num_threads(k):
    """Accepted for API compatibility; the GPU lane has no host thread pool."""
    int(k)


_EXPORTS = ("apply_r", "apply_s", "apply_t", "grad_ref", "ax_helmholtz_local", "gs_gather",
            "gs_scatter")


def install(kernels_module):
    """Swap this lane into a reference ``semflow.kernels`` module object.

    The reference resolves ``kernels.<fn>`` at call time (operators.py:18,47;
    space.py:47-48), so after this every reference operator runs on the B200.
    Returns the previous callables so the caller can restore them.
    """
    saved = {name: getattr(kernels_module, name) for name in _EXPORTS}
    if hasattr(kernels_module, "LANE"):
        saved["LANE"] = kernels_module.LANE
        kernels_module.LANE = LANE
    g = globals()
    for name in _EXPORTS:
        setattr(kernels_module, name, g[name])
    return saved


def uninstall(kernels_module, saved):
    for name, fn in saved.items():
        setattr(kernels_module, name, fn)
