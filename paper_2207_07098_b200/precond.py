"""Block-Jacobi preconditioner on device (reference precond.py:27-59).

The hybrid Schwarz preconditioner (precond.py:94-250) is not on the device path
(SURVEY.md section 8f, rank 1).
"""

import torch

from .errors import SolverBreakdownError


def assembled_diagonal(space, lam_visc, lam_mass):
    """Analytic diagonal of lam_visc D^T G D + lam_mass B, assembled (precond.py:27-40).

    The three einsum terms are accumulated over m in ascending order starting
    from 0.0 -- the order numpy's einsum uses -- so the result is bit-identical
    to the reference.
    """
    d = torch.tensor(space.dmat, dtype=torch.float64, device=space.device)
    g = space.geom
    n = space.n
    d2 = d * d
    dd = torch.diagonal(d).contiguous()
    diag = torch.zeros(space.shape, dtype=torch.float64, device=space.device)
    for m in range(n):        # einsum("mi,emjk->eijk", d2, g0)
        diag = diag + d2[m].view(1, n, 1, 1) * g[0][:, m:m + 1, :, :]
    t = torch.zeros_like(diag)
    for m in range(n):        # einsum("mj,eimk->eijk", d2, g3)
        t = t + d2[m].view(1, 1, n, 1) * g[3][:, :, m:m + 1, :]
    diag = diag + t
    t = torch.zeros_like(diag)
    for m in range(n):        # einsum("mk,eijm->eijk", d2, g5)
        t = t + d2[m].view(1, 1, 1, n) * g[5][:, :, :, m:m + 1]
    diag = diag + t
    di = dd.view(1, n, 1, 1)
    dj = dd.view(1, 1, n, 1)
    dk = dd.view(1, 1, 1, n)
    diag = diag + ((2.0 * g[1]) * di) * dj
    diag = diag + ((2.0 * g[2]) * di) * dk
    diag = diag + ((2.0 * g[4]) * dj) * dk
    diag = lam_visc * diag + lam_mass * space.bm
    return space.gs.add(diag)


class BlockJacobi:
    """Inverse assembled diagonal; masked rows are identity (precond.py:43-59)."""

    def __init__(self, space, lam_visc, lam_mass, mask=None):
        diag = assembled_diagonal(space, float(lam_visc), float(lam_mass))
        if mask is not None:
            m = torch.as_tensor(mask, dtype=torch.float64, device=space.device).view(space.shape)
            diag = torch.where(m == 0.0, torch.ones_like(diag), diag)
        if not bool((diag > 0.0).all()):
            flat = diag.reshape(-1)
            bad = int(torch.argmin(flat))
            raise SolverBreakdownError(
                f"non-positive operator diagonal {float(flat[bad]):.3e} at flat point {bad}")
        self.inv_diag = (1.0 / diag).contiguous()
        self.space = space

    def __call__(self, r):
        return self.inv_diag * r
