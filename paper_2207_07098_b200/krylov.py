"""Krylov solvers and projection on device (reference semflow/krylov.py).

Same signatures, stopping rules, breakdown semantics and loop order as the
reference (pcg krylov.py:36-75, gmres :78-160, ProjectionSpace :163-236).

When the operator is a :class:`~paper_2207_07098_b200.operators.GlobalOp`, the
preconditioner a :class:`~paper_2207_07098_b200.precond.BlockJacobi` (or None)
and ``dot`` the space's ``gs.dot`` (or None), the solvers run on fused sm_100a
kernels with all vector updates and inner products on the device (the host only
reads the scalars the reference's control flow branches on, once per
iteration).  Any other callables run through a generic torch path that follows
the reference line by line.
"""

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import SolverBreakdownError
from .operators import GlobalOp
from .precond import BlockJacobi, HybridSchwarz

#: Jacobi scaling formed inside the Ax kernel (SEMFLOW_B200_PRE_FUSED=0 materialises z)
_PRE_FUSED = os.environ.get("SEMFLOW_B200_PRE_FUSED", "1") != "0"


@dataclass
class SolveInfo:
    x: torch.Tensor
    iterations: int
    residual: float
    initial_residual: float
    converged: bool


def _default_dot(a, b):
    return float(torch.dot(a.reshape(-1), b.reshape(-1)))


def _ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


class _Fused:
    """Kernel-level helpers bound to one (space, weighting, preconditioner)."""

    def __init__(self, op, precond, dot):
        sp = op.space
        self.op = op
        self.sp = sp
        self.P = sp.n_points
        self.dev = sp.device
        gs = sp.gs
        # weighting: gs.dot -> 1/mult ; None -> plain dot (krylov.py:32-33)
        self.mult = _lib.ptr(gs.mult8) if dot is not None else None
        # a device preconditioner with its own kernels (hybrid Schwarz): z = M v is
        # formed explicitly and kept per Arnoldi step (flexible GMRES, krylov.py:104-105)
        self.pc = precond if isinstance(precond, HybridSchwarz) else None
        self.invdiag = precond.inv_diag if isinstance(precond, BlockJacobi) else None
        self.w = _device.workspace(self.dev)
        self.st = _lib.stream_ptr(self.dev)
        self.comm = sp.comm

    def dot(self, a, b, out):
        peer = self.comm.peer
        if peer is not None and self.mult is not None:
            # one kernel: local glsc3 + NVLink cross-rank sum in its last block
            _lib.call("sf_glsc3_peer_f64", _lib.ptr(a), _lib.ptr(b), self.mult, self.P, *self.w.args(),
                      _lib.ptr(out), *peer.fused_args(), self.st)
            return
        _lib.call("sf_glsc3_f64", 1, _ptrs([a]), _ptrs([b]), self.mult, self.P, *self.w.args(),
                  _lib.ptr(out), self.st)
        self.comm.sum_(out)

    def dots(self, pairs, out):
        for c in range(0, len(pairs), 4):
            chunk = pairs[c:c + 4]
            _lib.call("sf_glsc3_f64", len(chunk), _ptrs([a for a, _ in chunk]), _ptrs([b for _, b in chunk]),
                      self.mult, self.P, *self.w.args(), out.data_ptr() + 8 * c, self.st)
        self.comm.sum_(out[:len(pairs)])

    def mgs(self, out, *args, gate=None):
        """sf_mgs_step_f64 writing 2 partials to `out` (a 2-slot view), then allreduce
        -- fused into the same kernel over NVLink peer memory when available.
        ``gate``: device scalar; the pass is skipped when it is 0 (all ranks alike)."""
        peer = self.comm.peer
        if peer is not None:
            _lib.call("sf_mgs_step_peer_f64", *args, self.P, *self.w.args(), _lib.ptr(out),
                      *peer.fused_args(), gate, self.st)
            return
        _lib.call("sf_mgs_step_f64", *args, self.P, *self.w.args(), _lib.ptr(out), gate, self.st)
        if gate is None:
            self.comm.sum_(out)
        elif self.comm.world > 1:
            raise RuntimeError("gated MGS passes across ranks need the peer reducer")

    def read(self, t):
        return self.checked(t.to("cpu", non_blocking=False).tolist())

    def checked(self, vals):
        """Host values of a reduction; NaN across ranks may mean a peer timed out
        (the NVLink kernels then return NaN at once): raise instead of iterating."""
        if self.comm.peer is not None and any(v != v for v in vals):
            self.comm.check()
        return vals

    def precond_into(self, v, z):
        if self.pc is not None:
            return self.pc.apply_into(v, z)
        if self.invdiag is None:
            z.copy_(v)
        else:
            torch.mul(self.invdiag, v, out=z)
        return z

    def apply_precond(self, v, w, z):
        """w <- A M^-1 v (krylov.py:106-107, z = precond(v); w = apply_a(z)).  With
        Jacobi at n = 8 the product inv_diag * v is formed inside the Ax kernel as v
        is loaded (same bits, z never written); without a preconditioner A acts on
        v directly (the reference's copy is identical)."""
        if self.pc is not None:
            self.pc.apply_into(v, z)
            self.op.apply_into(z, w)
        elif self.invdiag is None:
            self.op.apply_into(v, w)
        elif self.sp.n == 8 and _PRE_FUSED:
            self.op.apply_into(v, w, pre=self.invdiag)
        else:
            self.precond_into(v, z)
            self.op.apply_into(z, w)
        return w


def _fusable(apply_a, precond, dot, device_pc=False):
    """The fused device path applies: our operator, our inner product, and a
    Jacobi preconditioner (or, with ``device_pc``, a hybrid Schwarz one) of the
    same space."""
    if not isinstance(apply_a, GlobalOp):
        return False
    if precond is not None:
        kinds = (BlockJacobi, HybridSchwarz) if device_pc else (BlockJacobi,)
        if not (isinstance(precond, kinds) and precond.space is apply_a.space):
            return False
    if dot is not None:
        owner = getattr(dot, "__self__", None)
        if owner is not apply_a.space.gs or getattr(dot, "__name__", "") != "dot":
            return False
    return apply_a.space.device.type == "cuda"


# =========================================================================== PCG

def pcg(apply_a, b, *, tol, max_iter, precond=None, dot=None, x0=None):
    """Preconditioned CG with absolute residual tolerance (krylov.py:36-75)."""
    if _fusable(apply_a, precond, dot):
        return _pcg_fused(apply_a, b, tol, max_iter, precond, dot, x0)
    return _pcg_generic(apply_a, b, tol, max_iter, precond, dot, x0)


def _pcg_generic(apply_a, b, tol, max_iter, precond, dot, x0):
    if dot is None:
        dot = _default_dot
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = b.clone() if x0 is None else b - apply_a(x)
    res0 = math.sqrt(dot(r, r))
    res = res0
    if res <= tol:
        return SolveInfo(x, 0, res, res0, True)
    z = precond(r) if precond is not None else r.clone()
    p = z.clone()
    rz = dot(r, z)
    it = 0
    converged = False
    for it in range(1, max_iter + 1):
        ap = apply_a(p)
        pap = dot(p, ap)
        if pap <= 0.0:
            raise SolverBreakdownError(
                f"non-positive curvature <p,Ap> = {pap:.3e} in conjugate gradients", iteration=it)
        alpha = rz / pap
        x += alpha * p
        r -= alpha * ap
        res = math.sqrt(dot(r, r))
        if res <= tol:
            converged = True
            break
        z = precond(r) if precond is not None else r.clone()
        rz_new = dot(r, z)
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return SolveInfo(x, it, res, res0, converged)


def _pcg_fused(op, b, tol, max_iter, precond, dot, x0):
    F = _Fused(op, precond, dot)
    P = F.P
    b = b.contiguous()
    ws = _device.field_work(op.space)      # work vectors kept across solves (no in-step cudaMalloc)
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = ws.like("kr_r", b)
    if x0 is None:
        r.copy_(b)
    else:
        torch.sub(b, op(x, out=ws.like("kr_ax", b)), out=r)
    # scalar slots: 0 rr, 1-2 rz (ping-pong), 3 pap, 4-5 update outputs (rr, rz_new)
    s = torch.zeros(8, dtype=torch.float64, device=F.dev)
    F.dot(r, r, s[0:1])
    res0 = math.sqrt(F.read(s[0:1])[0])
    res = res0
    if res <= tol:
        return SolveInfo(x, 0, res, res0, True)
    p = ws.like("kr_p", b)
    ap = ws.like("kr_ax", b)
    inv = _lib.ptr(F.invdiag)
    mult = F.mult
    wk = F.w.args()
    sp = lambda i: s.data_ptr() + 8 * i
    _lib.call("sf_cg_init_f64", _lib.ptr(r), inv, _lib.ptr(p), mult, P, *wk, sp(1), F.st)
    F.comm.sum_(s[1:2])
    rz_slot = 1
    it = 0
    converged = False
    for it in range(1, max_iter + 1):
        op.apply_into(p, ap)
        F.dot(p, ap, s[3:4])
        _lib.call("sf_cg_update_f64", _lib.ptr(x), _lib.ptr(r), _lib.ptr(p), _lib.ptr(ap), inv, mult,
                  sp(rz_slot), sp(3), P, *wk, sp(4), F.st)
        F.comm.sum_(s[4:6])
        pap, rr = F.read(s[3:5])
        if pap <= 0.0:
            raise SolverBreakdownError(
                f"non-positive curvature <p,Ap> = {pap:.3e} in conjugate gradients", iteration=it)
        res = math.sqrt(rr)
        if res <= tol:
            converged = True
            break
        new_slot = 2 if rz_slot == 1 else 1
        # rz_new lives in slot 5; copy it into the free ping-pong slot for the next round
        s[new_slot:new_slot + 1].copy_(s[5:6])
        _lib.call("sf_cg_direction_f64", _lib.ptr(p), _lib.ptr(r), inv, sp(new_slot), sp(rz_slot), P, F.st)
        rz_slot = new_slot
    return SolveInfo(x, it, res, res0, converged)


# =========================================================================== GMRES

def gmres(apply_a, b, *, tol, max_iter, restart=10, precond=None, dot=None, x0=None):
    """Flexible right-preconditioned restarted GMRES (krylov.py:78-160)."""
    if _fusable(apply_a, precond, dot, device_pc=True):
        return _gmres_fused(apply_a, b, tol, max_iter, restart, precond, dot, x0)
    return _gmres_generic(apply_a, b, tol, max_iter, restart, precond, dot, x0)


def _givens_column(hcol, j, cs, sn, g, total):
    """Apply the stored rotations to column j and form the new one (krylov.py:124-142)."""
    for i in range(j):
        tmp = cs[i] * hcol[i] + sn[i] * hcol[i + 1]
        hcol[i + 1] = -sn[i] * hcol[i] + cs[i] * hcol[i + 1]
        hcol[i] = tmp
    denom = np.hypot(hcol[j], hcol[j + 1])
    if denom == 0.0:
        raise SolverBreakdownError(
            "zero Hessenberg column in GMRES (operator annihilated the search direction)",
            iteration=total + 1)
    cs[j] = hcol[j] / denom
    sn[j] = hcol[j + 1] / denom
    hcol[j] = denom
    hcol[j + 1] = 0.0
    g[j + 1] = -sn[j] * g[j]
    g[j] = cs[j] * g[j]


def _back_substitute(h, g, j_end):
    y = np.zeros(j_end)
    for i in range(j_end - 1, -1, -1):
        y[i] = (g[i] - h[i, i + 1:j_end] @ y[i + 1:j_end]) / h[i, i]
    return y


def _gmres_generic(apply_a, b, tol, max_iter, restart, precond, dot, x0):
    if dot is None:
        dot = _default_dot
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = b.clone() if x0 is None else b - apply_a(x)
    beta = math.sqrt(dot(r, r))
    res0 = beta
    if beta <= tol:
        return SolveInfo(x, 0, beta, res0, True)
    total = 0
    converged = False
    while total < max_iter and not converged:
        m = min(restart, max_iter - total)
        vs = [r / beta]
        zs = []
        h = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        j_end = 0
        for j in range(m):
            z = precond(vs[j]) if precond is not None else vs[j].clone()
            zs.append(z)
            w = apply_a(z)
            norm_before = math.sqrt(dot(w, w))
            hcol = np.zeros(j + 2)
            for i in range(j + 1):
                hij = dot(w, vs[i])
                w -= hij * vs[i]
                hcol[i] = hij
            norm_after = math.sqrt(dot(w, w))
            if norm_after < 0.7071 * norm_before:
                for i in range(j + 1):
                    c = dot(w, vs[i])
                    w -= c * vs[i]
                    hcol[i] += c
                norm_after = math.sqrt(dot(w, w))
            hcol[j + 1] = norm_after
            _givens_column(hcol, j, cs, sn, g, total)
            h[: j + 2, j] = hcol
            total += 1
            j_end = j + 1
            happy = norm_after <= 1e-14 * max(norm_before, 1.0)
            if abs(g[j + 1]) <= tol or happy or total >= max_iter:
                break
            vs.append(w / norm_after)
        y = _back_substitute(h, g, j_end)
        for i in range(j_end):
            x += float(y[i]) * zs[i]
        r = b - apply_a(x)
        beta = math.sqrt(dot(r, r))
        if beta <= tol:
            converged = True
    return SolveInfo(x, total, beta, res0, converged)


#: [Arnoldi steps whose second Gram-Schmidt sweep fired, steps] of the look-ahead
#: GMRES (its second sweep is gated on the device; bench.py's step accounting)
GATE_STATS = [0, 0]


def _pipelinable(F, b):
    """The pipelined GMRES needs the gated (vectorised) MGS kernels and, across
    ranks, the fused peer reduction.  It pays off where the host round trip per
    Arnoldi step is exposed -- multi-GPU (64^3 on 4 B200: 494 -> 461 ms/step)
    and large single-GPU meshes (64^3 on 1 B200: 1004 -> 959 ms/step); below
    ~4 M points per rank the look-ahead's discarded step costs more than it
    hides.  SEMFLOW_B200_GMRES_PIPELINE=0/1 forces it off/on."""
    env = os.environ.get("SEMFLOW_B200_GMRES_PIPELINE", "auto")
    want = (F.comm.world > 1 or F.P >= 1 << 22) if env == "auto" else env != "0"
    return (want and F.mult is not None and F.P % 2 == 0 and b.data_ptr() % 16 == 0
            and (F.comm.world == 1 or F.comm.peer is not None))


class _GraphBuffers:
    """Fixed buffers and the per-step CUDA graphs of the look-ahead GMRES for one
    (operator, preconditioner, restart, size) -- kept on the operator."""

    @property
    def z(self):
        """Scratch preconditioned vector, allocated on first use (the Jacobi
        pre-scaled Ax never writes it)."""
        z = getattr(self, "_z", None)
        if z is None:
            z = self._z = torch.empty(self._shape, dtype=torch.float64, device=self._dev)
        return z

    def __init__(self, b, restart, S, key, flexible=False):
        self.key = key
        self.V = torch.empty((restart + 1,) + tuple(b.shape), dtype=torch.float64, device=b.device)
        # flexible GMRES keeps every preconditioned direction z_j (krylov.py:104-105)
        self.Z = torch.empty((restart,) + tuple(b.shape), dtype=torch.float64, device=b.device) \
            if flexible else None
        self.blk = torch.zeros((restart, S), dtype=torch.float64, device=b.device)
        self.host = torch.zeros((restart, S), dtype=torch.float64, pin_memory=True)
        self._shape = tuple(b.shape)
        self._dev = b.device
        self.graphs = {}
        self.counts = {}          # library launches recorded in each captured step
        self.bytes = {}           # and their algorithmic bytes (traffic.py)
        self.pool = torch.cuda.graph_pool_handle()


def _graph_buffers(F, op, b, restart, S):
    """Graph replay of the Arnoldi steps unless SEMFLOW_B200_GRAPHS=0.  Across ranks
    the captured NVLink reductions and halo exchanges take their call numbers and
    mailbox banks from device counters (peer.cuh, halo.cu), so a replay is the
    same launch sequence as an eager step.  The opt-in fused Ax+dssum launch
    (axdss.cu) takes a host-side epoch and is never captured.  A hybrid Schwarz
    preconditioner is captured with the step (its launches take fixed buffers)."""
    if os.environ.get("SEMFLOW_B200_GRAPHS", "1") == "0" or getattr(op, "fused", False):
        return None
    if F.comm.world > 1 and F.comm.peer is None:
        return None
    # every device address a captured step reads: the graphs stay valid only while
    # these are the same tensors (the buffers below are held alive by the cache)
    key = (restart, tuple(b.shape), F.invdiag.data_ptr() if F.invdiag is not None else None, F.mult,
           F.w.args()[0], _lib.stream_ptr(F.dev), id(F.pc) if F.pc is not None else None)
    gb = getattr(op, "_gmres_graphs", None)
    if gb is None or gb.key != key:
        gb = _GraphBuffers(b, restart, S, key, flexible=F.pc is not None)
        gb.refs = (F.invdiag, F.pc)
        op._gmres_graphs = gb
    return gb


def _gmres_pipelined(F, op, b, tol, max_iter, restart):
    """GMRES with one Arnoldi step of look-ahead (same arithmetic as _gmres_fused).

    Every Arnoldi step is enqueued without a host round trip: both Gram-Schmidt
    sweeps, the reorthogonalisation test (sf_gmres_gate_f64: the same IEEE
    comparison the host makes, evaluated on the device) and the normalisation of
    the next basis vector.  Step j's scalars are copied to pinned memory behind
    an event; while the host runs the Givens rotations and the convergence test
    of step j, step j+1 is already executing.  When step j converges, the
    speculatively computed step j+1 is discarded (nothing it wrote is used), so
    the iterate, the iteration count and the residual are those of the
    reference loop (krylov.py:95-160).  Look-ahead is skipped while the residual
    estimate is within 10x of the tolerance.
    """
    P = F.P
    dev = F.dev
    mult = F.mult
    wk = F.w.args()
    ws = _device.field_work(op.space)
    x = torch.zeros_like(b)
    r = ws.like("kr_r", b).copy_(b)
    s0 = torch.zeros(4, dtype=torch.float64, device=dev)
    F.dot(r, r, s0[0:1])
    beta = math.sqrt(F.read(s0[0:1])[0])
    res0 = beta
    if beta <= tol:
        return SolveInfo(x, 0, beta, res0, True)
    o2 = 2 * (restart + 2)           # second sweep within an iteration block
    o3 = 4 * (restart + 2)           # [o3] reorth flag, [o3+1] final norm
    S = o3 + 4
    total = 0
    converged = False
    gb = _graph_buffers(F, op, b, restart, S)
    if gb is not None:
        # the scratch z only where apply_precond writes it (not with the
        # Jacobi-prescaled Ax, nor with no preconditioner, nor with Schwarz's Z)
        need_z = F.pc is None and F.invdiag is not None and not (F.sp.n == 8 and _PRE_FUSED)
        blk, host, z, Vbuf, Z = gb.blk, gb.host, (gb.z if need_z else None), gb.V, gb.Z
    else:
        blk = torch.zeros((restart, S), dtype=torch.float64, device=dev)
        host = torch.zeros((restart, S), dtype=torch.float64, pin_memory=True)
        z = torch.empty_like(b)
        Vbuf = None
        Z = torch.empty((restart,) + tuple(b.shape), dtype=torch.float64, device=dev) \
            if F.pc is not None else None

    def launch(j, V):
        if gb is not None:
            # the whole Arnoldi step replayed from a CUDA graph captured once per
            # operator (fixed buffers; ~10 us of host time instead of ~30 launches)
            g = gb.graphs.get(j)
            if g is None:
                g = torch.cuda.CUDAGraph()
                st_saved = F.st
                n0, b0 = _lib.LAUNCHES, list(_lib.BYTES)
                acc, _lib.ACCOUNT = _lib.ACCOUNT, True
                with torch.cuda.graph(g, pool=gb.pool):
                    F.st = _lib.stream_ptr(dev)
                    body(j, V)
                F.st = st_saved
                _lib.ACCOUNT = acc
                # captured, not launched: launches and bytes are counted per replay
                gb.counts[j] = _lib.LAUNCHES - n0
                gb.bytes[j] = [a - c for a, c in zip(_lib.BYTES, b0)]
                _lib.LAUNCHES, _lib.BYTES[:] = n0, b0
                gb.graphs[j] = g
            g.replay()
            _lib.LAUNCHES += gb.counts[j]
            if _lib.ACCOUNT:
                _lib.BYTES[0] += gb.bytes[j][0]
                _lib.BYTES[1] += gb.bytes[j][1]
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dev))
            V.append(Vbuf[j + 1])
            return ev
        ev = body(j, V)
        return ev

    def body(j, V):
        bl = blk[j]
        bp = lambda i: bl.data_ptr() + 8 * i
        w = torch.empty_like(b) if Vbuf is None else Vbuf[j + 1]
        F.apply_precond(V[j], w, z if Z is None else Z[j])
        F.mgs(bl[0:2], _lib.ptr(w), None, None, _lib.ptr(V[0]), None, None, mult, 1)
        for i in range(1, j + 1):
            F.mgs(bl[2 * i:2 * i + 2], _lib.ptr(w), _lib.ptr(V[i - 1]), bp(2 * (i - 1)), _lib.ptr(V[i]),
                  None, None, mult, 0)
        # the first sweep's last pass also dots the updated w with v_0: the second
        # sweep's first coefficient (bit-identical to a separate pass, which
        # would re-read w), moved into place by the gate kernel (phase 2)
        F.mgs(bl[2 * (j + 1):2 * (j + 2)], _lib.ptr(w), _lib.ptr(V[j]), bp(2 * j), _lib.ptr(V[0]), None, None,
              mult, 1)
        _lib.call("sf_gmres_gate_f64", bl.data_ptr(), j, o2, o3, 2, F.st)
        g8 = bp(o3)
        for i in range(1, j + 1):
            F.mgs(bl[o2 + 2 * i:o2 + 2 * i + 2], _lib.ptr(w), _lib.ptr(V[i - 1]), bp(o2 + 2 * (i - 1)),
                  _lib.ptr(V[i]), None, None, mult, 0, gate=g8)
        F.mgs(bl[o2 + 2 * (j + 1):o2 + 2 * (j + 2)], _lib.ptr(w), _lib.ptr(V[j]), bp(o2 + 2 * j), None, None,
              None, mult, 1, gate=g8)
        _lib.call("sf_gmres_gate_f64", bl.data_ptr(), j, o2, o3, 1, F.st)
        host[j].copy_(bl, non_blocking=True)
        if Vbuf is not None:          # graph capture: the caller records the event
            _lib.call("sf_scale_div_f64", _lib.ptr(w), _lib.ptr(w), None, None, bp(o3 + 1), P, F.st)
            return None
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        # speculative next basis vector v_{j+1} = w / norm_after (krylov.py:149)
        _lib.call("sf_scale_div_f64", _lib.ptr(w), _lib.ptr(w), None, None, bp(o3 + 1), P, F.st)
        V.append(w)
        return ev

    while total < max_iter and not converged:
        m = min(restart, max_iter - total)
        v0 = torch.empty_like(b) if Vbuf is None else Vbuf[0]
        s0[1:2].fill_(beta)
        _lib.call("sf_scale_div_f64", _lib.ptr(v0), _lib.ptr(r), None, None, s0.data_ptr() + 8, P, F.st)
        V = [v0]
        h = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        j_end = 0
        evs = {0: launch(0, V)}
        for j in range(m):
            if j + 1 < m and j + 1 not in evs and abs(g[j]) > 10.0 * tol:
                evs[j + 1] = launch(j + 1, V)
            evs[j].synchronize()
            vals = F.checked(host[j].tolist())
            norm_before = math.sqrt(vals[1])
            hcol = np.zeros(j + 2)
            for i in range(j + 1):
                hcol[i] = vals[2 * i]
            norm_after = math.sqrt(vals[2 * (j + 1) + 1])
            GATE_STATS[1] += 1
            if norm_after < 0.7071 * norm_before:
                GATE_STATS[0] += 1
                for i in range(j + 1):
                    hcol[i] += vals[o2 + 2 * i]
                norm_after = math.sqrt(vals[o2 + 2 * (j + 1) + 1])
            hcol[j + 1] = norm_after
            _givens_column(hcol, j, cs, sn, g, total)
            h[: j + 2, j] = hcol
            total += 1
            j_end = j + 1
            happy = norm_after <= 1e-14 * max(norm_before, 1.0)
            if abs(g[j + 1]) <= tol or happy or total >= max_iter:
                break
            if j + 1 < m and j + 1 not in evs:
                evs[j + 1] = launch(j + 1, V)
        y = _back_substitute(h, g, j_end)
        if Z is None:
            _lincomb(x, x, V[:j_end], y, F.invdiag, P, dev, F.st)
        else:                              # x += sum_i y_i z_i (krylov.py:153-154)
            _lincomb(x, x, [Z[i] for i in range(j_end)], y, None, P, dev, F.st)
        ax = op(x, out=ws.like("kr_ax", b))
        _lib.call("sf_residual_f64", _lib.ptr(r), _lib.ptr(b), _lib.ptr(ax), mult, P, *wk, _lib.ptr(s0[0:1]), F.st)
        F.comm.sum_(s0[0:1])
        beta = math.sqrt(F.read(s0[0:1])[0])
        if beta <= tol:
            converged = True
    return SolveInfo(x, total, beta, res0, converged)


def _gmres_fused(op, b, tol, max_iter, restart, precond, dot, x0):
    F = _Fused(op, precond, dot)
    if x0 is None and _pipelinable(F, b.contiguous()):
        return _gmres_pipelined(F, op, b.contiguous(), tol, max_iter, restart)
    P = F.P
    dev = F.dev
    b = b.contiguous()
    ws = _device.field_work(op.space)
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = ws.like("kr_r", b)
    if x0 is None:
        r.copy_(b)
    else:
        torch.sub(b, op(x, out=ws.like("kr_ax", b)), out=r)
    # Krylov basis kept across solves: restart + 1 fields
    Vblk = ws.get("gm_V", (restart + 1,) + tuple(b.shape))
    mult = F.mult
    wk = F.w.args()
    inv = _lib.ptr(F.invdiag)
    s0 = torch.zeros(4, dtype=torch.float64, device=dev)
    F.dot(r, r, s0[0:1])
    beta = math.sqrt(F.read(s0[0:1])[0])
    res0 = beta
    if beta <= tol:
        return SolveInfo(x, 0, beta, res0, True)
    # per-cycle device scalars: [2*i] = h_i (first pass), [2*i+1] = <w,w> ; second
    # pass at offset 2*(restart+2); slot `sc` holds the divisor for scale_div
    nh = 2 * (restart + 2)
    hs = torch.zeros(2 * nh + 4, dtype=torch.float64, device=dev)
    sc = 2 * nh
    hp = lambda i: hs.data_ptr() + 8 * i
    z = ws.like("kr_p", b)
    Zblk = ws.get("gm_Z", (restart,) + tuple(b.shape)) if F.pc is not None else None
    total = 0
    converged = False
    while total < max_iter and not converged:
        m = min(restart, max_iter - total)
        v0 = Vblk[0]
        hs[sc:sc + 1].fill_(beta)
        _lib.call("sf_scale_div_f64", _lib.ptr(v0), _lib.ptr(r), None, None, hp(sc), P, F.st)
        vs = [v0]
        h = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        j_end = 0
        for j in range(m):
            w = Vblk[j + 1]
            F.apply_precond(vs[j], w, z if Zblk is None else Zblk[j])
            # MGS sweep: pass 0 = (<w,v0>, <w,w>), pass i = (w -= h_{i-1} v_{i-1}; <w,v_i>),
            # last = (w -= h_j v_j; <w,w>)
            F.mgs(hs[0:2], _lib.ptr(w), None, None, _lib.ptr(vs[0]), None, None, mult, 1)
            for i in range(1, j + 1):
                F.mgs(hs[2 * i:2 * i + 2], _lib.ptr(w), _lib.ptr(vs[i - 1]), hp(2 * (i - 1)),
                      _lib.ptr(vs[i]), None, None, mult, 0)
            F.mgs(hs[2 * (j + 1):2 * (j + 2)], _lib.ptr(w), _lib.ptr(vs[j]), hp(2 * j), None, None, None,
                  mult, 1)
            vals = F.read(hs[: 2 * (j + 2)])
            norm_before = math.sqrt(vals[1])
            hcol = np.zeros(j + 2)
            for i in range(j + 1):
                hcol[i] = vals[2 * i]
            norm_after = math.sqrt(vals[2 * (j + 1) + 1])
            if norm_after < 0.7071 * norm_before:
                o = nh
                F.mgs(hs[o:o + 2], _lib.ptr(w), None, None, _lib.ptr(vs[0]), None, None, mult, 0)
                for i in range(1, j + 1):
                    F.mgs(hs[o + 2 * i:o + 2 * i + 2], _lib.ptr(w), _lib.ptr(vs[i - 1]), hp(o + 2 * (i - 1)),
                          _lib.ptr(vs[i]), None, None, mult, 0)
                F.mgs(hs[o + 2 * (j + 1):o + 2 * (j + 2)], _lib.ptr(w), _lib.ptr(vs[j]), hp(o + 2 * j), None,
                      None, None, mult, 1)
                v2 = F.read(hs[o: o + 2 * (j + 2)])
                for i in range(j + 1):
                    hcol[i] += v2[2 * i]
                norm_after = math.sqrt(v2[2 * (j + 1) + 1])
            hcol[j + 1] = norm_after
            _givens_column(hcol, j, cs, sn, g, total)
            h[: j + 2, j] = hcol
            total += 1
            j_end = j + 1
            happy = norm_after <= 1e-14 * max(norm_before, 1.0)
            if abs(g[j + 1]) <= tol or happy or total >= max_iter:
                break
            hs[sc:sc + 1].fill_(norm_after)
            _lib.call("sf_scale_div_f64", _lib.ptr(w), _lib.ptr(w), None, None, hp(sc), P, F.st)
            vs.append(w)
        y = _back_substitute(h, g, j_end)
        if Zblk is None:
            _lincomb(x, x, vs[:j_end], y, F.invdiag, P, dev, F.st)
        else:
            _lincomb(x, x, [Zblk[i] for i in range(j_end)], y, None, P, dev, F.st)
        ax = op(x, out=ws.like("kr_ax", b))
        _lib.call("sf_residual_f64", _lib.ptr(r), _lib.ptr(b), _lib.ptr(ax), mult, P, *wk, _lib.ptr(s0[0:1]), F.st)
        F.comm.sum_(s0[0:1])
        beta = math.sqrt(F.read(s0[0:1])[0])
        if beta <= tol:
            converged = True
    return SolveInfo(x, total, beta, res0, converged)


def _lincomb(x, x0, vecs, coef, invdiag, P, dev, st):
    """x = x0 + sum_i coef[i] M vecs[i] (coef host array or device tensor)."""
    nv = len(vecs)
    if nv == 0:
        if x0 is not None and x0.data_ptr() != x.data_ptr():
            x.copy_(x0)
        elif x0 is None:
            x.zero_()
        return x
    ptrs = torch.tensor([v.data_ptr() for v in vecs], dtype=torch.int64, device=dev)
    if isinstance(coef, torch.Tensor):
        cd = coef.to(device=dev, dtype=torch.float64).contiguous()
    else:
        cd = torch.tensor(np.asarray(coef, dtype=np.float64), device=dev)
    _lib.call("sf_lincomb_f64", _lib.ptr(x), _lib.ptr(x0), _lib.ptr(ptrs), _lib.ptr(cd), _lib.ptr(invdiag),
              nv, P, st)
    return x


# =========================================================================== projection

class ProjectionSpace:
    """A-orthonormal basis of previous solutions (krylov.py:163-236)."""

    def __init__(self, dot=None, capacity=20, reset_every=20):
        self.dot = dot if dot is not None else _default_dot
        self.capacity = int(capacity)
        self.reset_every = int(reset_every)
        self.xs = []
        self.axs = []
        self._solves = 0
        self._slots = []

    def reserve(self, like, pairs):
        """Preallocate `pairs` (x, Ax) basis slots shaped like `like`; `absorb` fills
        them before growing the device heap.  Neko allocates its projection basis at
        init; growing it inside the time loop costs one multi-GB cudaMalloc per new
        vector (tens of ms of host time each at 64^3, with the device idle)."""
        for _ in range(int(pairs)):
            self._slots.append((torch.empty_like(like), torch.empty_like(like)))

    def _slot(self, like):
        while self._slots:
            x, ax = self._slots.pop()
            if x.shape == like.shape and x.dtype == like.dtype and x.device == like.device:
                return x, ax
        return torch.empty_like(like), torch.empty_like(like)

    @property
    def count(self):
        return len(self.xs)

    def invalidate(self):
        self.xs = []
        self.axs = []
        self._solves = 0

    def _fused(self, apply_a):
        if not isinstance(apply_a, GlobalOp):
            return None
        gs = apply_a.space.gs
        owner = getattr(self.dot, "__self__", None)
        if owner is not gs:
            return None
        return _Fused(apply_a, None, self.dot)

    def prepare(self, rhs, apply_a):
        self._solves += 1
        if self._solves > self.reset_every:
            self.xs = []
            self.axs = []
            self._solves = 1
        F = self._fused(apply_a)
        if not self.xs:
            if F is None:
                return torch.zeros_like(rhs), rhs.clone()
            # the right-hand side handed to the solver lives in the space's work
            # buffers (valid until the next prepare); x0 is returned fresh
            return torch.zeros_like(rhs), _device.field_work(F.sp).like("proj_b", rhs).copy_(rhs)
        if F is None:
            x0 = torch.zeros_like(rhs)
            for xi in self.xs:
                x0 += self.dot(xi, rhs) * xi
            return x0, rhs - apply_a(x0)
        k = len(self.xs)
        coef = torch.zeros(k, dtype=torch.float64, device=F.dev)
        F.dots([(xi, rhs) for xi in self.xs], coef)
        x0 = torch.empty_like(rhs)
        _lincomb(x0, None, self.xs, coef, None, F.P, F.dev, F.st)
        ws = _device.field_work(F.sp)
        return x0, torch.sub(rhs, apply_a(x0, out=ws.like("proj_ad", rhs)), out=ws.like("proj_b", rhs))

    def absorb(self, dx, apply_a):
        if len(self.xs) >= self.capacity:
            self.xs = []
            self.axs = []
        F = self._fused(apply_a)
        if F is None:
            d = dx.clone()
            ad = apply_a(d)
        else:
            ws = _device.field_work(F.sp)
            d = ws.like("proj_d", dx).copy_(dx)
            ad = apply_a(d, out=ws.like("proj_ad", dx))
        if F is None:
            a0 = self.dot(d, ad)
            if a0 <= 0.0:
                return
            for xi, axi in zip(self.xs, self.axs):
                c = self.dot(xi, ad)
                d -= c * xi
                ad -= c * axi
            nrm2 = self.dot(d, ad)
            if nrm2 <= 1e-14 * a0:
                return
            nrm = math.sqrt(nrm2)
            self.xs.append(d / nrm)
            self.axs.append(ad / nrm)
            return
        k = len(self.xs)
        s = torch.zeros(2 * k + 8, dtype=torch.float64, device=F.dev)
        sp = lambda i: s.data_ptr() + 8 * i
        F.dot(d, ad, s[0:1])
        a0 = F.read(s[0:1])[0]
        if a0 <= 0.0:
            return
        wk = F.w.args()
        # c_i = <ad, x_i> after the updates of 0..i-1 (slot 2 + 2 i)
        for i in range(k):
            vprev = self.axs[i - 1] if i else None
            v2prev = self.xs[i - 1] if i else None
            F.mgs(s[2 + 2 * i:4 + 2 * i], _lib.ptr(ad), _lib.ptr(vprev), sp(2 + 2 * (i - 1)) if i else None,
                  _lib.ptr(self.xs[i]), _lib.ptr(d) if i else None, _lib.ptr(v2prev), F.mult, 0)
        if k:
            _lib.call("sf_mgs_step_f64", _lib.ptr(ad), _lib.ptr(self.axs[k - 1]), sp(2 + 2 * (k - 1)), None,
                      _lib.ptr(d), _lib.ptr(self.xs[k - 1]), F.mult, 0, F.P, *wk, sp(2 + 2 * k), None, F.st)
        F.dot(d, ad, s[1:2])
        nrm2 = F.read(s[1:2])[0]
        if nrm2 <= 1e-14 * a0:
            return
        nrm = math.sqrt(nrm2)
        s[0:1].fill_(nrm)
        xn, axn = self._slot(d)
        _lib.call("sf_scale_div_f64", _lib.ptr(xn), _lib.ptr(d), _lib.ptr(axn), _lib.ptr(ad), sp(0), F.P, F.st)
        self.xs.append(xn)
        self.axs.append(axn)
