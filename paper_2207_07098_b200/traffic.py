"""Algorithmic HBM bytes of each library call (the step-level roofline of
SURVEY §8(d): "Time step: GDOF/s plus the sum of per-kernel algorithmic bytes
over the step's measured call mix, divided by t_step").

The per-call figures follow the same convention as the per-kernel rooflines in
bench.py / DESIGN.md §4: every field a kernel must read or write once, 8 B per
f64 value; the 1-byte multiplicity of the weighted dots is counted, masks and
index widths are not ("masks, multiplicities and int64 widths are
not credited" -- the dssum's int32 perm index, 4 B per shared copy, is).  Library
calls not listed here (set-up kernels, the plugin-API entry points) add nothing
and are reported in UNMODELED.  The dssum is accounted by space.GatherScatter,
which knows its class sizes (GatherScatter.account_dssum).

Accounting is off unless _lib.ACCOUNT is set; bench.py turns it on for the timed
steps only.  GMRES passes skipped by the device-side reorthogonalisation gate
(sf_mgs_step_f64 with a gate) go to the second bucket; bench.py credits them
with the fraction of Arnoldi steps whose second sweep the host saw fire.
"""

UNMODELED = set()


def _n3(n):
    return int(n) ** 3


def _live(arr):
    """Non-NULL entries of a ctypes pointer array (host arrays of device pointers)."""
    return [p for p in arr if p]


def _mgs(a, gate_idx):
    w, vprev, _h, vnext, w2, _v2p, mult, want_norm, P = a[:9]
    b = 8 + (16 if vprev else 0) + (8 if vnext else 0) + (24 if (w2 and vprev) else 0)
    b += 1 if (mult and (vnext or want_norm)) else 0
    return int(P) * b, a[gate_idx] is not None


def _ax(E, n, lm, pre):
    return E * _n3(n) * (8 + 48 + 8 + (8 if lm != 0.0 else 0) + (8 if pre else 0))


def _deriv(a):
    op, _d, n, _in, c, _rx, _out, E = a[:8]
    fin = 8 if op == 0 else 24
    fout = 8 if op == 1 else 24
    return int(E) * _n3(n) * (fin + (24 if c else 0) + 72 + fout)


def _glsc3(a):
    K, pa, pb, mult, P = a[:5]
    ptrs = set(_live(pa)[:K]) | set(_live(pb)[:K])
    return int(P) * (8 * len(ptrs) + (1 if mult else 0))


def _bdf_ext(a):
    vhat, omega, vel, nl, crl, _adt, _b, order, P3 = a[:9]
    fields = (1 if vhat else 0) + (1 if omega else 0)
    fields += sum(len(_live(arr)[:order]) for arr in (vel, nl, crl))
    return int(P3) * 8 * fields


# name -> bytes(args); (bytes, gated) for the MGS passes
MODELS = {
    "sf_ax_helm_f64": lambda a: _ax(a[6], a[1], a[8], None),
    "sf_ax_masked_f64": lambda a: _ax(a[6], a[1], a[8], None),
    "sf_ax_pre_f64": lambda a: _ax(a[7], a[1], a[9], a[5]),
    "sf_ax_range_f64": lambda a: _ax(a[9] - a[8], a[1], a[11], a[5]),
    "sf_mgs_step_f64": lambda a: _mgs(a, 12),
    "sf_mgs_step_peer_f64": lambda a: _mgs(a, 17),
    "sf_glsc3_f64": _glsc3,
    "sf_glsc3_peer_f64": lambda a: int(a[3]) * (8 * len({a[0], a[1]}) + (1 if a[2] else 0)),
    "sf_cg_init_f64": lambda a: int(a[4]) * (16 + (8 if a[1] else 0) + (1 if a[3] else 0)),
    "sf_cg_update_f64": lambda a: int(a[8]) * (48 + (8 if a[4] else 0) + (1 if a[5] else 0)),
    "sf_cg_direction_f64": lambda a: int(a[5]) * (24 + (8 if a[2] else 0)),
    "sf_lincomb_f64": lambda a: int(a[6]) * (8 + (8 if a[1] else 0) + 8 * int(a[5]) + (8 if a[4] else 0)),
    "sf_residual_f64": lambda a: int(a[4]) * (24 + (1 if a[3] else 0)),
    "sf_scale_div_f64": lambda a: int(a[5]) * (16 + (16 if a[2] else 0)),
    "sf_deriv_f64": _deriv,
    "sf_cdtp_f64": lambda a: int(a[6]) * _n3(a[1]) * (24 + 72 + 8 + 8),
    "sf_cfl_f64": lambda a: int(a[4]) * _n3(a[3]) * (24 + 72),
    "sf_bdf_ext_f64": _bdf_ext,
    "sf_gather_f64": lambda a: int(a[3]) * (8 + 8 + 4),
    "sf_dssum_blk_f64": lambda a: 0,         # accounted by space.GatherScatter.account_dssum
    "sf_dssum_cls_f64": lambda a: 0,
    "sf_gmres_gate_f64": lambda a: 0,
    "sf_peer_allreduce_f64": lambda a: 0,
    "sf_rank_sum_f64": lambda a: 0,
    "sf_halo_put_f64": lambda a: 0,          # NVLink stores, not HBM traffic of this rank's step
    "sf_halo_wait": lambda a: 0,
}


def account(name, args, buckets):
    """Add the algorithmic bytes of one library call to buckets [ungated, gated]."""
    fn = MODELS.get(name)
    if fn is None:
        UNMODELED.add(name)
        return
    r = fn(args)
    if isinstance(r, tuple):
        buckets[1 if r[1] else 0] += r[0]
    else:
        buckets[0] += r


def dssum_bytes(n_local, n_halo, n_gid):
    """One dssum: each local shared copy read + written + its int32 index, each
    received halo copy read + its index, one CSR offset per shared gid (§8(d))."""
    return n_local * (8 + 8 + 4) + n_halo * (8 + 4) + n_gid * 4
