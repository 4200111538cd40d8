"""GLL basis (setup only): nodes, weights and the differentiation matrix.

Restates the reference's algorithm (basis.py) so a device space can be built
without the reference installed; the arithmetic is kept operation-for-operation
so the arrays are bit-identical to ``semflow.basis.make_basis`` (pinned by
tests/test_setup_parity.py against tests/golden):

* nodes: Newton on P_N' seeded with Chebyshev-Gauss-Lobatto points, then exact
  antisymmetrisation (reference basis.py:43-65),
* weights 2 / (N (N+1) P_N(x)^2) (basis.py:113),
* D by barycentric weights with the negated-row-sum diagonal (basis.py:120-139).
"""

from dataclasses import dataclass

import numpy as np


def _legendre(n, x):
    """P_n(x) and P_n'(x) by the three-term recurrence (reference basis.py:17-40)."""
    x = np.asarray(x, dtype=np.float64)
    if n == 0:
        return np.ones_like(x), np.zeros_like(x)
    pm, p = np.ones_like(x), x.copy()
    for k in range(2, n + 1):
        pm, p = p, ((2 * k - 1) * x * p - (k - 1) * pm) / k
    edge = np.abs(x) == 1.0
    safe = np.where(edge, 1.0, 1.0 - x * x)
    dp = np.where(edge, 0.5 * n * (n + 1) * np.sign(x) ** (n + 1), n * (pm - x * p) / safe)
    return p, dp


def _nodes(n):
    if n == 1:
        return np.array([-1.0, 1.0])
    x = -np.cos(np.pi * np.arange(1, n) / n)
    for _ in range(100):
        p, dp = _legendre(n, x)
        step = dp / ((2.0 * x * dp - n * (n + 1) * p) / (1.0 - x * x))
        x = x - step
        if np.max(np.abs(step)) < 1e-14:
            break
    else:
        raise RuntimeError(f"GLL Newton iteration failed to converge at order {n}")
    pts = np.concatenate(([-1.0], x, [1.0]))
    return 0.5 * (pts - pts[::-1])


def _bary(pts):
    diff = pts[:, None] - pts[None, :]
    np.fill_diagonal(diff, 1.0)
    return 1.0 / np.prod(diff, axis=1)


def _dmat(pts):
    w = _bary(pts)
    dx = pts[:, None] - pts[None, :]
    np.fill_diagonal(dx, 1.0)
    d = (w[None, :] / w[:, None]) / dx
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, -np.sum(d, axis=1))
    return d


@dataclass(frozen=True)
class Basis1D:
    """Same fields as the reference ``Basis1D`` (basis.py:68-93)."""

    order: int
    points: np.ndarray
    weights: np.ndarray
    dmat: np.ndarray

    @property
    def n(self):
        return self.order + 1


def make_basis(order):
    if not isinstance(order, (int, np.integer)) or order < 1:
        raise ValueError(f"polynomial order must be an integer >= 1, got {order!r}")
    n = int(order)
    pts = _nodes(n)
    p, _ = _legendre(n, pts)
    wts = 2.0 / (n * (n + 1) * p * p)
    d = _dmat(pts)
    for a in (pts, wts, d):
        a.setflags(write=False)
    return Basis1D(order=n, points=pts, weights=wts, dmat=d)


def interp_matrix(basis, targets):
    """J[k, j] = l_j(targets[k]), barycentric form; rows of targets that hit a
    node (|diff| < 1e-14) are exact unit vectors (basis.py:142-174)."""
    t = np.atleast_1d(np.asarray(targets, dtype=np.float64))
    if t.ndim != 1:
        raise ValueError("target points must be one-dimensional")
    outside = (t < -1.0 - 1e-12) | (t > 1.0 + 1e-12)
    if np.any(outside):
        raise ValueError(f"interpolation target {t[outside][0]} lies outside [-1, 1]")
    pts = basis.points
    lam = _bary(pts)
    dist = t[:, None] - pts[None, :]
    hit_r, hit_c = np.nonzero(np.abs(dist) < 1e-14)
    J = np.zeros((t.size, pts.size))
    free = np.ones(t.size, dtype=bool)
    free[hit_r] = False
    if np.any(free):
        q = lam[None, :] / dist[free]
        J[free] = q / np.sum(q, axis=1, keepdims=True)
    J[hit_r, hit_c] = 1.0
    return J


def gauss_legendre(m):
    """m-point Gauss-Legendre rule on [-1, 1] (basis.py:177-181, numpy's leggauss)."""
    if m < 1:
        raise ValueError(f"Gauss-Legendre rule needs at least 1 point, got {m}")
    return np.polynomial.legendre.leggauss(m)
