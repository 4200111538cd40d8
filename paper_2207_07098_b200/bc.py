"""Boundary conditions on device (reference semflow/bc.py).

Masks and per-step boundary terms for every reference kind: ``noslip``,
``velocity``, ``inflow``, ``rotor``, ``function``, ``taylor_green``
(Dirichlet), ``symmetry`` and ``outflow`` (bc.py:33-270).  Dirichlet evaluators are called with host numpy
coordinates of the constrained points -- the same call the reference makes
(bc.py:218-229), so user functions written for the reference work unchanged --
and only those boundary values cross to the device.

Surface terms (``pressure_surface_rhs``, ``surface_flux_rhs``) reproduce the
reference's ``np.add.at`` accumulation order: contributions are added group by
group (tag order), and inside a group in facet-point order, one "round" per
repeated target so every local point sums its contributions sequentially.
"""

import numpy as np
import torch

from .errors import ConfigError

DIRICHLET_KINDS = ("noslip", "velocity", "inflow", "rotor", "function", "taylor_green")


def _const_fn(value):
    v = np.asarray(value, dtype=np.float64)
    if v.shape != (3,):
        raise ConfigError(f"constant velocity must have 3 components, got {v.shape}")

    def fn(x, y, z, t):
        return np.broadcast_to(v.reshape((3,) + (1,) * np.ndim(x)), (3,) + np.shape(x)).copy()

    return fn


def power_law_profile(y, u_cl, h, exponent=1.0 / 7.0):
    """Streamwise inflow speed u_cl (y/h)^exponent with y clamped into [0, h]
    (bc.py:36-45; the out-of-range warning is not reproduced)."""
    yc = np.minimum(np.maximum(np.asarray(y, dtype=np.float64), 0.0), h)
    return u_cl * (yc / h) ** exponent


def spin_ramp(y, u_spin, delta):
    """Rotor surface speed vs. height (bc.py:48-66): 0 for y <= 0, u_spin for
    y >= delta, u_spin / (1 + exp(1/(q-1) + 1/q)) with q = y/delta between
    (exponent argument clipped to +-700)."""
    q = np.asarray(y, dtype=np.float64) / delta
    out = np.where(q >= 1.0, u_spin, 0.0)
    inner = (q > 0.0) & (q < 1.0)
    qi = q[inner]
    out[inner] = u_spin / (1.0 + np.exp(np.clip(1.0 / (qi - 1.0) + 1.0 / qi, -700.0, 700.0)))
    return out


def spinning_wall(x, y, z, u_spin, delta, center=(0.0, 0.0)):
    """Azimuthal velocity of a cylinder about the y axis (bc.py:69-87):
    (s dz / rho, 0, -s dx / rho), zero on the axis itself."""
    dx = np.asarray(x, dtype=np.float64) - center[0]
    dz = np.asarray(z, dtype=np.float64) - center[1]
    rho = np.hypot(dx, dz)
    s = spin_ramp(y, u_spin, delta)
    fac = np.where(rho > 0.0, s / np.where(rho > 0.0, rho, 1.0), 0.0)
    out = np.zeros((3,) + np.broadcast(dx, np.asarray(y), dz).shape)
    out[0] = fac * dz
    out[2] = -fac * dx
    return out


def decaying_vortex(x, y, z, t, nu):
    """Planar Taylor-Green velocity (analytic.py:11-17)."""
    amp = np.exp(-2.0 * nu * t)
    out = np.zeros((3,) + np.broadcast(np.asarray(x), np.asarray(y)).shape)
    out[0] = np.sin(x) * np.cos(y) * amp
    out[1] = -np.cos(x) * np.sin(y) * amp
    return out


def make_evaluator(kind, params):
    """Host evaluator g(x, y, z, t) -> (3, ...) for a Dirichlet kind (bc.py:142-157)."""
    if kind == "noslip":
        return _const_fn((0.0, 0.0, 0.0))
    if kind == "velocity":
        return _const_fn(params["value"])
    if kind == "function":
        return params["fn"]
    if kind == "inflow":
        u_cl, h = float(params["u_cl"]), float(params["h"])
        ex = float(params.get("exponent", 1.0 / 7.0))
        if h <= 0.0:
            raise ConfigError(f"inflow height h must be positive, got {h}")

        def inflow(x, y, z, t):
            out = np.zeros((3,) + np.shape(x))
            out[0] = power_law_profile(y, u_cl, h, ex)
            return out
        return inflow
    if kind == "rotor":
        u_spin = float(params["u_spin"]) if "u_spin" in params else \
            float(params["u_cl"]) * float(params.get("alpha", 3.0))
        delta = float(params["delta"])
        if delta <= 0.0:
            raise ConfigError(f"rotor smoothing distance delta must be positive, got {delta}")
        center = tuple(float(c) for c in params.get("center", (0.0, 0.0)))
        return lambda x, y, z, t: spinning_wall(x, y, z, u_spin, delta, center)
    if kind == "taylor_green":
        nu = float(params["nu"])
        return lambda x, y, z, t: decaying_vortex(x, y, z, t, nu)
    raise ConfigError(f"unknown Dirichlet kind {kind!r}")


class _Scatter:
    """Ordered scatter-add of per-facet-point values into a local field."""

    def __init__(self, targets):
        # targets: (K,) int64 device tensor of local point indices in reference order
        self.targets = targets
        order = torch.sort(targets, stable=True).indices
        st = targets[order]
        first = torch.ones_like(st, dtype=torch.bool)
        if st.numel() > 1:
            first[1:] = st[1:] != st[:-1]
        grp_start = torch.cummax(torch.where(first, torch.arange(st.numel(), device=st.device),
                                             torch.zeros_like(st)), 0).values
        occ_sorted = torch.arange(st.numel(), device=st.device) - grp_start
        occ = torch.empty_like(occ_sorted)
        occ[order] = occ_sorted
        nround = int(occ.max()) + 1 if occ.numel() else 0
        self.rounds = [torch.nonzero(occ == r).view(-1) for r in range(nround)]

    def add_into(self, out_flat, vals):
        for sel in self.rounds:
            out_flat.index_add_(0, self.targets[sel], vals[sel])


class BoundarySet:
    """Compiled boundary conditions for one device FunctionSpace (bc.py:159-203)."""

    def __init__(self, space, specs):
        self.space = space
        dev = space.device
        # 0/1 masks as uint8 (the reference's are float64 0.0/1.0, bc.py:164-201):
        # the same values in every product (x * 1 = x, x * 0 = +-0), 1 byte per point
        self.vel_mask = torch.ones((3,) + space.shape, dtype=torch.uint8, device=dev)
        self.prs_mask = torch.ones(space.shape, dtype=torch.uint8, device=dev)
        self.dirichlet = []   # (tag, facet indices (host), evaluator, flat points (device), host coords)
        self.symmetry = []    # (facet indices, axis, flat points)
        seen = set()
        coords_h = None
        ftag = np.asarray(space.facet_tag)
        for tag, spec in sorted(specs.items()):
            if tag not in space.mesh.tag_names:
                raise ConfigError(f"boundary condition references unknown tag {tag!r}; "
                                  f"mesh has {space.mesh.tag_names}")
            kind = spec["kind"]
            params = {k: v for k, v in spec.items() if k != "kind"}
            tix = space.mesh.tag_names.index(tag)
            idx = np.nonzero(ftag == tix)[0]
            if not np.any(np.asarray(space.mesh.facet_tag) == tix):
                raise ConfigError(f"tag {tag!r} has no facets on this mesh")
            seen.add(tag)
            if idx.size == 0:
                continue      # the tag's facets live on other ranks' elements
            it = torch.from_numpy(idx).to(dev)
            flat = space.facet_flat[it].reshape(-1)
            if kind in DIRICHLET_KINDS:
                fn = make_evaluator(kind, params)
                if coords_h is None:
                    coords_h = space.coords.reshape(3, -1)
                xs = coords_h[:, flat].cpu().numpy()
                self.dirichlet.append((tag, it, fn, flat, xs))
            elif kind == "symmetry":
                self.symmetry.append((it, self._symmetry_axis(tag, it), flat))
            elif kind == "outflow":
                self.prs_mask.view(-1)[flat] = 0
            else:
                raise ConfigError(f"boundary kind {kind!r} for tag {tag!r} is not supported on the device path")
        missing = set(space.mesh.tag_names) - seen
        if missing:
            raise ConfigError(f"no boundary condition given for tags {sorted(missing)}")
        for _, axis, flat in self.symmetry:
            self.vel_mask[axis].view(-1)[flat] = 0
        for _, _, _, flat, _ in self.dirichlet:
            for l in range(3):
                self.vel_mask[l].view(-1)[flat] = 0
        self.has_pressure_dirichlet = space.comm.any(bool((self.prs_mask == 0).any()))
        self.has_dirichlet = bool(self.dirichlet)
        self._neumann = [it for _, it, _, _, _ in self.dirichlet] + [it for it, _, _ in self.symmetry]
        self._neu_scatter = [_Scatter(space.facet_flat[it].reshape(-1)) for it in self._neumann]
        self._dir_scatter = [_Scatter(flat) for _, _, _, flat, _ in self.dirichlet]

    def _symmetry_axis(self, tag, it):
        nrm = self.space.facet_normal[it].abs()          # (k, n, n, 3)
        axis = int(torch.argmax(nrm.reshape(-1, 3).mean(dim=0)))
        comp = nrm[..., axis]
        others = torch.cat([nrm[..., a:a + 1] for a in range(3) if a != axis], dim=-1)
        if bool((comp < 1.0 - 1e-8).any()) or bool((others > 1e-8).any()):
            raise ConfigError(f"symmetry tag {tag!r} lies on a non-axis-aligned surface; "
                              "only coordinate-plane symmetry is supported")
        return axis

    def _values(self, fn, xs, t):
        """Boundary values at time t, evaluated on the host coordinates as the
        reference does (its evaluators are host numpy callables); the last time's
        upload is reused -- a step asks for the same t up to three times."""
        cache = self.__dict__.setdefault("_vcache", {})
        key = (id(fn), float(t))
        hit = cache.get(id(fn))
        if hit is not None and hit[0] == key:
            return hit[1]
        g = np.asarray(fn(xs[0], xs[1], xs[2], t), dtype=np.float64)
        val = torch.from_numpy(np.ascontiguousarray(g.reshape(3, -1))).to(self.space.device)
        cache[id(fn)] = (key, val)
        return val

    def apply_dirichlet(self, vel, t):
        """Overwrite constrained velocity points with boundary values (bc.py:218-229)."""
        flat = vel.view(3, -1)
        for _, axis, pts in self.symmetry:
            flat[axis][pts] = 0.0
        for _, _, fn, pts, xs in self.dirichlet:
            g = self._values(fn, xs, t)
            for l in range(3):
                flat[l][pts] = g[l]
        return vel

    def dirichlet_field(self, t, out=None):
        if out is None:
            g = torch.zeros((3,) + self.space.shape, dtype=torch.float64, device=self.space.device)
        else:
            g = out.zero_()
        self.apply_dirichlet(g, t)
        return g

    def pressure_surface_rhs(self, t, out=None):
        """sum over Dirichlet facets of phi_i (g . n) dA (bc.py:237-253)."""
        sp = self.space
        out = torch.zeros(sp.n_points, dtype=torch.float64, device=sp.device) if out is None \
            else out.view(-1).zero_()
        for (_, it, fn, pts, xs), sc in zip(self.dirichlet, self._dir_scatter):
            g = self._values(fn, xs, t).view(3, *sp.facet_flat[it].shape)
            nrm = sp.facet_normal[it].permute(3, 0, 1, 2)
            gn = (g[0] * nrm[0] + g[1] * nrm[1] + g[2] * nrm[2]) * sp.facet_warea[it]
            sc.add_into(out, gn.reshape(-1))
        return out.view(sp.shape)

    def surface_flux_rhs(self, field, out=None):
        """sum over velocity-BC facets of phi_i (F . n) dA (bc.py:255-270)."""
        sp = self.space
        out = torch.zeros(sp.n_points, dtype=torch.float64, device=sp.device) if out is None \
            else out.view(-1).zero_()
        flat = field.reshape(3, -1)
        for it, sc in zip(self._neumann, self._neu_scatter):
            pts = sp.facet_flat[it]
            f = flat[:, pts.reshape(-1)].view(3, *pts.shape)
            nrm = sp.facet_normal[it].permute(3, 0, 1, 2)
            fn = (f[0] * nrm[0] + f[1] * nrm[1] + f[2] * nrm[2]) * sp.facet_warea[it]
            sc.add_into(out, fn.reshape(-1))
        return out.view(sp.shape)
