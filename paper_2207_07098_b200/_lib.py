"""ctypes binding of libsemflow_b200.so (the C ABI in include/semflow_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``python -m
paper_2207_07098_b200.build``).  There is no fallback: if the shared object is
missing or no CUDA device is visible, every device entry point raises.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SEMFLOW_B200_CHECKED=1: the build with device bounds checks (build.py --checked)
LIB_PATH = os.path.join(_HERE, "libsemflow_b200_checked.so"
                        if os.environ.get("SEMFLOW_B200_CHECKED", "0") not in ("", "0") else "libsemflow_b200.so")

_lib = None

_vp = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "sf_version": [],
    "sf_last_error": [],
    "sf_red_workspace_doubles": [],
    "sf_set_ax_kernel": [_i],
    "sf_apply_axis_f64": [_i, _vp, _i, _i, _vp, _vp, _ll, _i, _vp],
    "sf_apply_axis3_f64": [_i, _vp, _i, _i, _i, _i, _vp, _vp, _ll, _i, _vp],
    "sf_grad_ref_f64": [_vp, _i, _vp, _vp, _vp, _vp, _ll, _i, _vp],
    "sf_ax_helm_f64": [_vp, _i, _vp, _vp, _vp, _vp, _ll, _d, _d, _i, _vp],
    "sf_gs_gather_f64": [_vp, _vp, _vp, _ll, _vp, _vp],
    "sf_gs_scatter_f64": [_vp, _vp, _vp, _ll, _vp, _vp],
    "sf_ax_masked_f64": [_vp, _i, _vp, _vp, _vp, _vp, _ll, _d, _d, _vp, _vp, _i, _vp],
    "sf_dssum_f64": [_vp, _vp, _vp, _i, _i, _vp, _vp, _i, _vp],
    "sf_dssum_cls_f64": [_vp, _vp, _i, _i, _i, _vp, _i, _i, _vp, _vp, _i, _vp],
    "sf_dssum_blk_f64": [_vp, _vp, _i, _i, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _i, _vp, _ll, _vp],
    "sf_ax_pre_f64": [_vp, _i, _vp, _vp, _vp, _vp, _vp, _ll, _d, _d, _vp, _vp, _i, _vp],
    "sf_ax_range_f64": [_vp, _i, _vp, _vp, _vp, _vp, _vp, _ll, _ll, _ll, _d, _d, _vp, _vp, _i, _vp],
    "sf_gather_f64": [_vp, _vp, _vp, _ll, _vp],
    "sf_rank_sum_f64": [_vp, _i, _i, _vp, _vp],
    "sf_glsc3_f64": [_i, _vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp],
    "sf_cg_init_f64": [_vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp],
    "sf_cg_update_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp],
    "sf_cg_direction_f64": [_vp, _vp, _vp, _vp, _vp, _ll, _vp],
    "sf_mgs_step_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _ll, _vp, _vp, _vp, _vp, _vp],
    "sf_gmres_gate_f64": [_vp, _i, _i, _i, _i, _vp],
    "sf_lincomb_f64": [_vp, _vp, _vp, _vp, _vp, _i, _ll, _vp],
    "sf_residual_f64": [_vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp],
    "sf_scale_div_f64": [_vp, _vp, _vp, _vp, _vp, _ll, _vp],
    "sf_deriv_f64": [_i, _vp, _i, _vp, _vp, _vp, _vp, _ll, _d, _i, _vp],
    "sf_cdtp_f64": [_vp, _i, _vp, _vp, _vp, _vp, _ll, _i, _vp],
    "sf_cfl_f64": [_vp, _vp, _vp, _i, _ll, _vp, _i, _vp],
    "sf_bdf_ext_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _ll, _vp],
    "sf_ipc_handle_bytes": [],
    "sf_peer_mailbox_doubles": [_i],
    "sf_dev_alloc_zero": [_ll, ctypes.POINTER(_vp)],
    "sf_dev_free": [_vp],
    "sf_ipc_get_handle": [_vp, ctypes.c_char_p],
    "sf_ipc_open_handle": [ctypes.c_char_p, ctypes.POINTER(_vp)],
    "sf_ipc_close_handle": [_vp],
    "sf_peer_allreduce_f64": [_vp, _i, _i, _vp, _vp, _vp, _i, _vp, _vp],
    "sf_mgs_step_peer_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _ll, _vp, _vp, _vp,
                             _vp, _i, _i, _vp, _vp, _vp, _vp],
    "sf_glsc3_peer_f64": [_vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp],
    "sf_halo_inbox_doubles": [_ll],
    "sf_halo_header_doubles": [],
    "sf_halo_put_f64": [_vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sf_halo_wait": [_vp, _i, _vp, _vp, _vp],
    "sf_trilinear_coords_f64": [_vp, _vp, _i, _ll, _vp, _vp],
    "sf_metrics_f64": [_vp, _vp, _i, _vp, _ll, _vp, _vp, _vp, _vp, _vp],
    "sf_dealias_advect_f64": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _ll, _d, _vp, _i, _vp],
    "sf_schwarz_gather_f64": [_vp, _vp, _vp],
    "sf_schwarz_restrict_f64": [_vp, _vp],
    "sf_schwarz_rank_sum_f64": [_vp, _vp, _i, _i, _vp],
    "sf_schwarz_coarse_f64": [_vp, _vp],
    "sf_schwarz_gather_rw_f64": [_vp, _vp],
    "sf_schwarz_finalize_f64": [_vp, _vp],
    "sf_schwarz_scatter_f64": [_vp, _vp, _vp],
    "sf_halo_unbank_f64": [_vp, _vp, _ll, _ll, _vp, _vp],
    "sf_schwarz_coarse_blocks": [],
}
_RESTYPES = {"sf_version": ctypes.c_char_p, "sf_last_error": ctypes.c_char_p}

EXPORTED = tuple(_SIGS)


class LibraryError(RuntimeError):
    """The CUDA extension is missing or a kernel call failed."""


def load(path=LIB_PATH):
    """Load (once) and return the ctypes handle; raises if the .so is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"{path} not found: build it with `python -m paper_2207_07098_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


#: number of library entry-point calls that launch kernels (bench.py's gpu_launches)
LAUNCHES = 0

#: algorithmic HBM bytes of the calls made while ACCOUNT is set, [ungated, gated
#: MGS passes] (traffic.py; bench.py's step roofline)
ACCOUNT = False
BYTES = [0, 0]


#: NVTX ranges around every entry point (SURVEY §5 tracing), named by the
#: SURVEY §2.2/§2.3 kernel/collective ids: "K2 dssum:sf_dssum_blk_f64".  Off by
#: default (no host cost); SEMFLOW_B200_NVTX=1 turns them on, e.g. for
#: ``ncu --nvtx --nvtx-include "K2 dssum/"`` or an nsys timeline.
NVTX = os.environ.get("SEMFLOW_B200_NVTX", "0") not in ("", "0")
NVTX_TAGS = {
    "sf_ax_helm_f64": "K1 ax", "sf_ax_masked_f64": "K1 ax", "sf_ax_pre_f64": "K1 ax",
    "sf_ax_range_f64": "K1 ax",
    "sf_dssum_f64": "K2 dssum", "sf_dssum_cls_f64": "K2 dssum", "sf_dssum_blk_f64": "K2 dssum",
    "sf_gs_gather_f64": "K2 dssum", "sf_gs_scatter_f64": "K2 dssum", "sf_gather_f64": "K2 dssum",
    "sf_grad_ref_f64": "K3 deriv", "sf_deriv_f64": "K3 deriv", "sf_cfl_f64": "K3 deriv",
    "sf_cdtp_f64": "K4 cdtp", "sf_dealias_advect_f64": "K4 cdtp", "sf_apply_axis_f64": "K4 cdtp", "sf_apply_axis3_f64": "K4 cdtp",
    "sf_glsc3_f64": "K5 glsc3", "sf_glsc3_peer_f64": "K5 glsc3",
    "sf_cg_init_f64": "K6 pcg", "sf_cg_update_f64": "K6 pcg", "sf_cg_direction_f64": "K6 pcg",
    "sf_mgs_step_f64": "K7 gmres", "sf_mgs_step_peer_f64": "K7 gmres", "sf_gmres_gate_f64": "K7 gmres",
    "sf_lincomb_f64": "K7 gmres", "sf_residual_f64": "K7 gmres", "sf_scale_div_f64": "K7 gmres",
    "sf_bdf_ext_f64": "K8 bdf_ext",
    "sf_halo_put_f64": "C1 halo", "sf_halo_wait": "C1 halo",
    "sf_peer_allreduce_f64": "C2 allreduce", "sf_rank_sum_f64": "C2 allreduce",
    "sf_schwarz_gather_f64": "K9 schwarz", "sf_schwarz_gather_rw_f64": "K9 schwarz",
    "sf_schwarz_restrict_f64": "K9 schwarz", "sf_schwarz_rank_sum_f64": "C2 allreduce",
    "sf_schwarz_coarse_f64": "K9 schwarz",
    "sf_schwarz_finalize_f64": "K9 schwarz", "sf_schwarz_scatter_f64": "K9 schwarz",
    "sf_halo_unbank_f64": "C1 halo",
}


def nvtx_push(label):
    if NVTX:
        torch.cuda.nvtx.range_push(label)


def nvtx_pop():
    if NVTX:
        torch.cuda.nvtx.range_pop()


def call(name, *args):
    """Invoke an entry point and raise LibraryError on a nonzero status."""
    global LAUNCHES
    lib = _lib if _lib is not None else load()
    LAUNCHES += 1
    if ACCOUNT:
        from . import traffic

        traffic.account(name, args, BYTES)
    if NVTX:
        torch.cuda.nvtx.range_push(f"{NVTX_TAGS.get(name, 'setup')}:{name}")
        try:
            st = getattr(lib, name)(*args)
        finally:
            torch.cuda.nvtx.range_pop()
    else:
        st = getattr(lib, name)(*args)
    if st != 0:
        msg = lib.sf_last_error().decode(errors="replace")
        raise LibraryError(f"{name} failed (status {st}): {msg}")


def ptr(t):
    """Raw device (or host) address of a tensor, or NULL for None."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(device=None):
    """cudaStream_t of torch's current stream on `device`."""
    return torch.cuda.current_stream(device).cuda_stream


def host_f64(a):
    """Keep-alive contiguous float64 host buffer + its address (for *_host args)."""
    import numpy as np

    buf = np.ascontiguousarray(a, dtype=np.float64)
    return buf, buf.ctypes.data


def require_cuda(t):
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise LibraryError("semflow_b200 device kernels need CUDA tensors (no CPU fallback)")
