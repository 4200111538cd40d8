"""Device matrix-free operators (reference semflow/operators.py).

Every function takes a :class:`~paper_2207_07098_b200.space.FunctionSpace` and
torch CUDA tensors and mirrors the reference signature of the same name.  The
assembled operator returned by :func:`make_global_op` is the hot path: one
sm_100a Ax_helm launch (mask applied on load, output select fused) followed by
one in-place dssum over the shared gids.
"""

import os

import numpy as np
import torch

from . import _device, _lib
from .space import pack_bits

OP_GRAD, OP_DIV, OP_CURL, OP_ADVECT = 0, 1, 2, 3


def _ex():
    return 1 if _device.EXACT else 0


#: multi-GPU operator: compute halo elements, post the exchange, then the interior
_OVERLAP = os.environ.get("SEMFLOW_B200_OVERLAP", "1") != "0"


def _ax_local(space, u, lam_visc, lam_mass, out=None):
    _lib.require_cuda(u)
    u = u.contiguous()
    w = torch.empty_like(u) if out is None else out
    E = u.shape[0]
    _lib.call("sf_ax_helm_f64", space.dmat.ctypes.data, space.n, _lib.ptr(space.geom), _lib.ptr(space.bm),
              _lib.ptr(u), _lib.ptr(w), E, float(lam_visc), float(lam_mass), _ex(),
              _lib.stream_ptr(space.device))
    return w


def laplace_local(space, u, out=None):
    """Element-local D^T G D u (operators.py:16-18)."""
    return _ax_local(space, u, 1.0, 0.0, out)


def helmholtz_local(space, u, lam_visc, lam_mass, out=None):
    """Element-local lam_visc D^T G D u + lam_mass B u (operators.py:21-29)."""
    if lam_visc <= 0.0:
        raise ValueError(f"lam_visc must be positive, got {lam_visc}")
    if lam_mass < 0.0:
        raise ValueError(f"lam_mass must be non-negative, got {lam_mass}")
    return _ax_local(space, u, float(lam_visc), float(lam_mass), out)


class GlobalOp:
    """u -> mask*gs.add(ax(mask*u)) + (1-mask)*u  (operators.py:32-56).

    Callable like the reference closure.  ``mask`` must be a 0/1 field (as built
    by BoundarySet); it is stored as per-element bitmasks, and the masked copies
    of shared gids are flagged in a private copy of the shared perm.

    Whether the operator is masked is decided over all ranks (collective on a
    multi-rank space): a rank whose slab holds no masked point still runs the
    masked kernel, so every rank -- and a single-GPU run -- computes each element
    with the same kernel variant (the masked and unmasked variants may round
    differently in the last bit: FMA contraction is the compiler's per variant).
    """

    def __init__(self, space, lam_visc, lam_mass, mask=None):
        self.space = space
        self.lam_visc = float(lam_visc)
        self.lam_mass = float(lam_mass)
        gs = space.gs
        E, n = space.n_elements, space.n
        self.masked = False
        if mask is not None:
            m = torch.as_tensor(mask, dtype=torch.float64, device=space.device).reshape(E, n ** 3)
            if not bool(((m == 0.0) | (m == 1.0)).all()):
                raise ValueError("make_global_op: mask must contain only 0.0 and 1.0")
            keep = m != 0.0
            if space.comm.any(not bool(keep.all())):
                self.masked = True
                self.inmask = pack_bits(keep)
                self.outsel = pack_bits(keep) | gs.shared_bits
                self.sh_perm = gs.masked_perm(keep.reshape(-1))
            # the float mask is not kept: the kernels read the bit-packed words
            self.mask = mask
        else:
            self.mask = None
        self.launches = 0

    def apply_into(self, u, w, pre=None):
        """w <- A u (w must not alias u).  With ``pre`` (n = 8): w <- A (pre * u),
        the product formed as u is loaded -- the Jacobi-preconditioned Krylov
        vector is never written (krylov.py:106-107)."""
        sp = self.space
        gs = sp.gs
        st = _lib.stream_ptr(sp.device)
        E = sp.n_elements
        split = gs.interior_range() if (sp.n == 8 and _OVERLAP) else None
        if split is not None:
            # halo elements first, post the NVLink exchange, interior while it
            # travels, then the wait and the dssum
            lo, hi = split
            args = (_lib.ptr(self.inmask) if self.masked else None, _lib.ptr(self.outsel) if self.masked else None,
                    _ex(), st)

            def rng(e0, e1):
                _lib.call("sf_ax_range_f64", sp.dmat.ctypes.data, sp.n, _lib.ptr(sp.geom), _lib.ptr(sp.bm),
                          _lib.ptr(u), _lib.ptr(pre), _lib.ptr(w), E, e0, e1, self.lam_visc, self.lam_mass, *args)

            rng(0, lo)
            rng(hi, E)
            gs.halo_put(w)
            rng(lo, hi)
            recv = gs.halo_wait()
            if self.masked:
                gs.dssum_into(w, 2, u=u, perm=self.sh_perm, pre=pre, recv=recv)
            else:
                gs.dssum_into(w, 0, recv=recv)
            self.launches += 5
            return w
        if pre is not None:
            if sp.n != 8:
                return self.apply_into(pre * u, w)
            _lib.call("sf_ax_pre_f64", sp.dmat.ctypes.data, sp.n, _lib.ptr(sp.geom), _lib.ptr(sp.bm),
                      _lib.ptr(u), _lib.ptr(pre), _lib.ptr(w), E, self.lam_visc, self.lam_mass,
                      _lib.ptr(self.inmask) if self.masked else None,
                      _lib.ptr(self.outsel) if self.masked else None, _ex(), st)
            if self.masked:
                gs.dssum_into(w, 2, u=u, perm=self.sh_perm, pre=pre)
            else:
                gs.dssum_into(w, 0)
            self.launches += 2
            return w
        if self.masked:
            _lib.call("sf_ax_masked_f64", sp.dmat.ctypes.data, sp.n, _lib.ptr(sp.geom), _lib.ptr(sp.bm),
                      _lib.ptr(u), _lib.ptr(w), E, self.lam_visc, self.lam_mass, _lib.ptr(self.inmask),
                      _lib.ptr(self.outsel), _ex(), st)
            gs.dssum_into(w, 2, u=u, perm=self.sh_perm)
        else:
            _lib.call("sf_ax_helm_f64", sp.dmat.ctypes.data, sp.n, _lib.ptr(sp.geom), _lib.ptr(sp.bm),
                      _lib.ptr(u), _lib.ptr(w), E, self.lam_visc, self.lam_mass, _ex(), st)
            gs.dssum_into(w, 0)
        self.launches += 2
        return w

    def __call__(self, u, out=None):
        _lib.require_cuda(u)
        u = u.contiguous()
        return self.apply_into(u, torch.empty_like(u) if out is None else out)


def make_global_op(space, lam_visc, lam_mass, mask=None):
    return GlobalOp(space, lam_visc, lam_mass, mask)


def _deriv(space, op, inp, c=None, sign=1.0, out_comps=3, out=None):
    E, n = space.n_elements, space.n
    if out is None:
        out = torch.empty((out_comps,) + space.shape if out_comps > 1 else space.shape,
                          dtype=torch.float64, device=space.device)
    _lib.call("sf_deriv_f64", op, space.dmat.ctypes.data, n, _lib.ptr(inp.contiguous()),
              _lib.ptr(c.contiguous()) if c is not None else None, _lib.ptr(space.rx), _lib.ptr(out),
              E, float(sign), _ex(), _lib.stream_ptr(space.device))
    return out


def grad(space, u, out=None):
    """Physical gradient (3, E, n, n, n) (operators.py:59-66)."""
    return _deriv(space, OP_GRAD, u, out=out)


def div(space, v, out=None):
    """Pointwise divergence (operators.py:69-76)."""
    return _deriv(space, OP_DIV, v, out_comps=1, out=out)


def curl(space, v, out=None):
    """Pointwise curl (operators.py:79-88)."""
    return _deriv(space, OP_CURL, v, out=out)


def advect_vec(space, c, v, dealias=None, sign=1.0):
    """(c . grad) v_l for l = 0, 1, 2 (operators.py:108-126): collocation, or
    over-integrated on the Gauss-Legendre grid with a :class:`Dealias`."""
    if dealias is not None:
        return dealias.advect_vec(c, v, sign=sign)
    return _deriv(space, OP_ADVECT, v, c=c, sign=sign)


def advect(space, c, u, dealias=None):
    """(c . grad) u for a scalar u (operators.py:108-116)."""
    if dealias is not None:
        return dealias.advect(c, u)
    g = grad(space, u)
    return c[0] * g[0] + c[1] * g[1] + c[2] * g[2]


class Dealias:
    """Over-integration of the convective term on ceil(3 n / 2) Gauss-Legendre
    points per direction (operators.py:129-158): c and grad u are interpolated
    to the fine grid, multiplied there, weighted by the fine quadrature and
    Jacobian and L2-projected back, then divided by the GLL mass."""

    def __init__(self, space):
        from .basis import gauss_legendre, interp_matrix

        self.space = space
        n = space.n
        self.m = int(np.ceil(1.5 * n))
        pts, wts = gauss_legendre(self.m)
        self.interp = np.ascontiguousarray(interp_matrix(space.basis, pts))
        self.interp_t = np.ascontiguousarray(self.interp.T)
        dev = space.device
        self._J = torch.from_numpy(self.interp).to(dev)
        self._Jt = torch.from_numpy(self.interp_t).to(dev)
        w3 = wts[:, None, None] * wts[None, :, None] * wts[None, None, :]
        self.wjac_f = torch.from_numpy(np.ascontiguousarray(w3)).to(dev)[None] * self._to_fine(space.jac)

    def _chain(self, mat, u):
        """apply_t(A, apply_s(A, apply_r(A, u))) (operators.py:141-147)."""
        m = mat.shape[0]
        out = u.contiguous()
        for axis in (0, 1, 2):
            shape = list(out.shape)
            shape[1 + axis] = m
            nxt = torch.empty(shape, dtype=torch.float64, device=out.device)
            _lib.call("sf_apply_axis3_f64", axis, _lib.ptr(mat), m, out.shape[1], out.shape[2], out.shape[3],
                      _lib.ptr(out), _lib.ptr(nxt), out.shape[0], _ex(), _lib.stream_ptr(out.device))
            out = nxt
        return out

    def _to_fine(self, u):
        return self._chain(self._J, u)

    def _project_back(self, f):
        return self._chain(self._Jt, f)

    def _advect_fine(self, cf, u):
        g = grad(self.space, u)
        fine = cf[0] * self._to_fine(g[0])
        fine += cf[1] * self._to_fine(g[1])
        fine += cf[2] * self._to_fine(g[2])
        weak = self._project_back(self.wjac_f * fine)
        return weak / self.space.bm

    def advect(self, c, u):
        return self._advect_fine([self._to_fine(c[l]) for l in range(3)], u)

    def advect_vec(self, c, v, sign=1.0, out=None):
        """sign * (c . grad) v_l for l = 0, 1, 2, over-integrated.  lx = 4, 6, 8: one
        fused launch per call (csrc/dealias.cu: every fine-grid field lives in
        shared memory); other orders: the contraction chain."""
        sp = self.space
        if (sp.n, self.m) in ((8, 12), (6, 9), (4, 6)):
            out = torch.empty((3,) + sp.shape, dtype=torch.float64, device=sp.device) if out is None else out
            _lib.call("sf_dealias_advect_f64", sp.dmat.ctypes.data, self.interp.ctypes.data, sp.n, self.m,
                      _lib.ptr(c.contiguous()), _lib.ptr(v.contiguous()), _lib.ptr(sp.rx), _lib.ptr(self.wjac_f),
                      _lib.ptr(sp.bm), sp.n_elements, float(sign), _lib.ptr(out), _ex(), _lib.stream_ptr(sp.device))
            return out
        cf = [self._to_fine(c[l]) for l in range(3)]     # the advecting field, once
        res = torch.stack([self._advect_fine(cf, v[l]) for l in range(3)])
        return res if sign == 1.0 else res * sign


def weak_grad_dot(space, w, out=None):
    """r_i = (grad phi_i, w) -- Nek cdtp (operators.py:91-105)."""
    if out is None:
        out = torch.empty(space.shape, dtype=torch.float64, device=space.device)
    _lib.call("sf_cdtp_f64", space.dmat.ctypes.data, space.n, _lib.ptr(w.contiguous()), _lib.ptr(space.rx),
              _lib.ptr(space.bm), _lib.ptr(out), space.n_elements, _ex(), _lib.stream_ptr(space.device))
    return out


def _dxi(points):
    xi = np.asarray(points, dtype=np.float64)
    gaps = np.diff(xi)
    dxi = np.empty_like(xi)
    dxi[0] = gaps[0]
    dxi[-1] = gaps[-1]
    if xi.size > 2:
        dxi[1:-1] = np.minimum(gaps[:-1], gaps[1:])
    return np.ascontiguousarray(dxi)


def cfl_max_async(space, v, out_bits):
    """out_bits (uint64 as int64 tensor) <- bits of max_p sum_s |rx_s . v| / dxi_s."""
    dxi = _dxi(space.basis.points)
    _lib.call("sf_cfl_f64", _lib.ptr(v.contiguous()), _lib.ptr(space.rx), dxi.ctypes.data, space.n,
              space.n_elements, _lib.ptr(out_bits), _ex(), _lib.stream_ptr(space.device))
    return out_bits


def cfl(space, v, dt):
    """CFL number (operators.py:161-182)."""
    bits = torch.zeros(1, dtype=torch.int64, device=space.device)
    cfl_max_async(space, v, bits)
    space.comm.max_(bits)          # non-negative doubles order like their bit patterns
    val = bits.cpu().view(torch.float64).item()
    return float(dt) * float(val)
