"""Generate the golden fixtures from the REFERENCE implementation (run here only).

    NUMBA_CACHE_DIR=/tmp/numba_cache SEMFLOW_NUMBA=1 \
        python tests/golden/make_golden.py [--skip-big]

Imports `semflow` from /root/reference/pkg/src (read-only, never shipped) and
records, with the numba lane:

* kernels.npz    -- lane kernel inputs/outputs (sample_fields of
                    pkg/tests/test_kernels.py plus an lx=8 case), gather/scatter;
* basis.npz      -- GLL points/weights/D for orders 1..10;
* spaces.npz     -- meshes (as arrays) and sha256 of coords/rx/jac/bm/geom/gid/
                    perm/offsets for box, perturbed-box and cylinder meshes, full
                    arrays for the small ones;
* operators.npz  -- Ax / global op / gs.add / avg / dot / grad / div / curl /
                    advect / weak_grad_dot / cfl / BlockJacobi on a perturbed box;
* solvers.json   -- PCG / GMRES iteration counts and residuals, per-step TGV
                    and channel diagnostics (iteration counts, residuals, CFL,
                    divergence, kinetic energy, enstrophy).
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("SEMFLOW_NUMBA", "1")

from semflow import kernels  # noqa: E402
from semflow import operators as ops  # noqa: E402
from semflow.basis import make_basis  # noqa: E402
from semflow.bc import BoundarySet  # noqa: E402
from semflow.diagnostics import kinetic_energy  # noqa: E402
from semflow.krylov import ProjectionSpace, gmres, pcg  # noqa: E402
from semflow.mesh import gen_box_mesh, gen_cylinder_box_mesh  # noqa: E402
from semflow.precond import BlockJacobi  # noqa: E402
from semflow.space import build_space  # noqa: E402
from semflow.timestep import SolverOptions, Stepper  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
assert kernels.lane_name() == "numba"


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def sample_fields(e, n, seed):
    """Same recipe as pkg/tests/test_kernels.py:25-35."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((e, n, n, n))
    a = rng.standard_normal((n, n))
    g = rng.standard_normal((6, e, n, n, n))
    g[0] += 3.0
    g[3] += 3.0
    g[5] += 3.0
    b = rng.uniform(0.5, 2.0, (e, n, n, n))
    return a, g, b, u


def gen_kernels():
    out = {}
    for tag, (e, n, seed) in {"n5": (3, 5, 7), "n6": (4, 6, 11), "n8": (6, 8, 3)}.items():
        a, g, b, u = sample_fields(e, n, seed)
        out[f"{tag}_a"], out[f"{tag}_g"], out[f"{tag}_b"], out[f"{tag}_u"] = a, g, b, u
        for ax, fn in enumerate((kernels.apply_r, kernels.apply_s, kernels.apply_t)):
            out[f"{tag}_apply{ax}"] = fn(a, u)
        rect = np.random.default_rng(seed + 1).standard_normal((n + 3, n))
        out[f"{tag}_rect"] = rect
        for ax, fn in enumerate((kernels.apply_r, kernels.apply_s, kernels.apply_t)):
            out[f"{tag}_rect{ax}"] = fn(rect, u)
        ur, us, ut = kernels.grad_ref(a, u)
        out[f"{tag}_ur"], out[f"{tag}_us"], out[f"{tag}_ut"] = ur, us, ut
        for k, (lv, lm) in enumerate(((1.0, 0.0), (0.7, 2.5), (1.0, 0.3))):
            out[f"{tag}_ax{k}"] = kernels.ax_helmholtz_local(a, g, b, u, lv, lm)
    # gather/scatter case (pkg/tests/test_kernels.py:98-108)
    rng = np.random.default_rng(5)
    nloc, ngid = 40, 12
    gid = rng.integers(0, ngid, nloc)
    gid[:ngid] = np.arange(ngid)
    perm = np.argsort(gid, kind="stable").astype(np.int64)
    counts = np.bincount(gid, minlength=ngid)
    offsets = np.zeros(ngid + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    vals = rng.standard_normal(nloc)
    out["gs_gid"], out["gs_perm"], out["gs_off"], out["gs_vals"] = gid, perm, offsets, vals
    out["gs_sums"] = kernels.gs_gather(vals, perm, offsets)
    out["gs_scat"] = kernels.gs_scatter(out["gs_sums"], perm, offsets, np.zeros(nloc))
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def gen_basis():
    out = {}
    for order in range(1, 11):
        b = make_basis(order)
        out[f"p{order}"], out[f"w{order}"], out[f"d{order}"] = b.points, b.weights, b.dmat
    np.savez_compressed(os.path.join(OUT, "basis.npz"), **out)


def perturbed_box(counts, seed, amp=0.08, extent=(0.0, 1.5, 0.0, 1.0, 0.0, 1.2)):
    m = gen_box_mesh(extent, counts)
    rng = np.random.default_rng(seed)
    v = m.vertices.copy()
    lo = np.array([extent[0], extent[2], extent[4]])
    hi = np.array([extent[1], extent[3], extent[5]])
    interior = np.all((v > lo + 1e-9) & (v < hi - 1e-9), axis=1)
    h = (hi - lo) / np.array(counts)
    v[interior] += amp * h * rng.uniform(-1, 1, (int(interior.sum()), 3))
    m.vertices = v
    return m


def mesh_arrays(prefix, m, out):
    out[f"{prefix}_vertices"] = m.vertices
    out[f"{prefix}_elements"] = m.elements
    out[f"{prefix}_facet_elem"] = m.facet_elem
    out[f"{prefix}_facet_face"] = m.facet_face
    out[f"{prefix}_facet_tag"] = m.facet_tag
    out[f"{prefix}_curved_elem"] = m.curved_elem
    out[f"{prefix}_curved_coords"] = m.curved_coords
    out[f"{prefix}_geom_order"] = np.array(-1 if m.geom_order is None else m.geom_order)
    out[f"{prefix}_tags"] = np.array(json.dumps(list(m.tag_names)))


def space_meta(prefix, sp, out, full):
    for name in ("coords", "rx", "jac", "bm", "geom"):
        out[f"{prefix}_sha_{name}"] = np.array(sha(getattr(sp, name)))
    for name in ("gid", "perm", "offsets"):
        out[f"{prefix}_sha_{name}"] = np.array(sha(getattr(sp.gs, name)))
    out[f"{prefix}_n_gid"] = np.array(sp.gs.n_gid)
    out[f"{prefix}_volume"] = np.array(sp.volume)
    out[f"{prefix}_warea_sum"] = np.array(float(sp.facet_warea.sum()))
    if full:
        for name in ("coords", "jac", "bm"):
            out[f"{prefix}_{name}"] = getattr(sp, name)
        for name in ("gid", "perm", "offsets"):
            out[f"{prefix}_{name}"] = getattr(sp.gs, name)
        out[f"{prefix}_facet_normal"] = sp.facet_normal
        out[f"{prefix}_facet_warea"] = sp.facet_warea


SPACES = {}


def gen_spaces():
    out = {}
    cases = {
        "box211": (gen_box_mesh((0.0, 2.0, 0.0, 1.0, 0.0, 1.0), (2, 1, 1)), 2, True),
        "cube222": (gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (2, 2, 2)), 4, True),
        "pbox322": (perturbed_box((3, 2, 2), 17), 7, True),
        "pbox543": (perturbed_box((5, 4, 3), 29, amp=0.12), 5, True),
        "tgv4": (gen_box_mesh((0.0, 2 * np.pi, 0.0, 2 * np.pi, 0.0, 2 * np.pi), (4, 4, 4)), 7, False),
        "tgv8": (gen_box_mesh((0.0, 2 * np.pi, 0.0, 2 * np.pi, 0.0, 2 * np.pi), (8, 8, 8)), 7, False),
        "rotor": (gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2,
                                        n_axial=2, n_upstream=4, n_downstream=5, n_front=3, n_back=3,
                                        geom_order=5), 5, True),
    }
    for key, (m, order, full) in cases.items():
        t0 = time.time()
        sp = build_space(m, make_basis(order))
        SPACES[key] = sp
        mesh_arrays(key, m, out)
        out[f"{key}_order"] = np.array(order)
        space_meta(key, sp, out, full)
        print(f"space {key}: E={m.n_elements} P={sp.gs.gid.size} {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(OUT, "spaces.npz"), **out)


def gen_operators():
    """Operator outputs on the perturbed 3x2x2 order-7 box (6144 points)."""
    sp = SPACES["pbox322"]
    rng = np.random.default_rng(0)
    u = rng.standard_normal(sp.shape)
    v = rng.standard_normal((3,) + sp.shape)
    c = rng.standard_normal((3,) + sp.shape)
    mask = np.ones(sp.shape)
    mask.reshape(-1)[sp.facet_flat.ravel()] = 0.0
    out = {"u": u, "v": v, "c": c, "mask": mask}
    out["ax_poisson"] = ops.laplace_local(sp, u)
    out["ax_helm"] = ops.helmholtz_local(sp, u, 0.3, 7.0)
    out["gop_poisson_masked"] = ops.make_global_op(sp, 1.0, 0.0, mask)(u)
    out["gop_helm_masked"] = ops.make_global_op(sp, 0.3, 7.0, mask)(u)
    out["gop_poisson"] = ops.make_global_op(sp, 1.0, 0.0)(u)
    out["gs_add"] = sp.gs.add(u)
    out["gs_avg"] = sp.gs.avg(u)
    out["gs_add_vec"] = sp.gs.add(v)
    out["gs_dot"] = np.array(sp.gs.dot(u, v[0]))
    out["integral"] = np.array(sp.integral(u))
    out["grad"] = ops.grad(sp, u)
    out["div"] = ops.div(sp, v)
    out["curl"] = ops.curl(sp, v)
    out["advect"] = ops.advect_vec(sp, c, v)
    out["wgd"] = ops.weak_grad_dot(sp, v)
    out["cfl"] = np.array(ops.cfl(sp, v, 0.01))
    out["jacobi_p"] = BlockJacobi(sp, 1.0, 0.0, mask).inv_diag
    out["jacobi_h"] = BlockJacobi(sp, 0.3, 7.0, mask).inv_diag
    out["ke"] = np.array(kinetic_energy(sp, v))
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **out)


def all_tags(spec):
    return {t: dict(spec) for t in ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")}


def poisson_case(ne, order=7, restart_gmres=20):
    sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (ne, ne, ne)), make_basis(order))
    mask = np.ones(sp.shape)
    mask.reshape(-1)[sp.facet_flat.ravel()] = 0.0
    f = sp.from_function(lambda x, y, z: 3.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y)
                         * np.sin(np.pi * z))
    exact = sp.from_function(lambda x, y, z: np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z))
    rhs = mask * sp.gs.add(sp.bm * f)
    a = ops.make_global_op(sp, 1.0, 0.0, mask)
    pc = BlockJacobi(sp, 1.0, 0.0, mask)
    res = {}
    t0 = time.time()
    info = pcg(a, rhs, tol=1e-8, max_iter=500, precond=pc, dot=sp.gs.dot)
    res["pcg"] = dict(iterations=info.iterations, residual=info.residual,
                      initial_residual=info.initial_residual, converged=info.converged,
                      err=float(np.abs(info.x - exact).max()), seconds=time.time() - t0,
                      x_l2=sp.l2_norm(info.x))
    if ne <= 8:
        info = gmres(a, rhs, tol=1e-8, max_iter=500, restart=restart_gmres, precond=pc, dot=sp.gs.dot)
        res["gmres"] = dict(iterations=info.iterations, residual=info.residual,
                            initial_residual=info.initial_residual, converged=info.converged,
                            err=float(np.abs(info.x - exact).max()), x_l2=sp.l2_norm(info.x))
        info = pcg(a, rhs, tol=1e-8, max_iter=500, dot=sp.gs.dot)
        res["cg_noprec"] = dict(iterations=info.iterations, residual=info.residual)
        # projection: solve twice with perturbed rhs
        proj = ProjectionSpace(sp.gs.dot)
        seq = []
        for k in range(3):
            r_k = rhs * (1.0 + 0.1 * k)
            x0, b = proj.prepare(r_k, a)
            inf = pcg(a, b, tol=1e-8, max_iter=500, precond=pc, dot=sp.gs.dot)
            proj.absorb(inf.x, a)
            seq.append(dict(iterations=inf.iterations, residual=inf.residual, count=proj.count))
        res["projection"] = seq
    return res


def enstrophy(sp, v):
    w = ops.curl(sp, v)
    return 0.5 * sp.integral(w[0] ** 2 + w[1] ** 2 + w[2] ** 2)


def tgv_case(ne, steps):
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, L), (ne, ne, ne)), make_basis(7))
    bset = BoundarySet(sp, all_tags({"kind": "symmetry"}))
    st = Stepper(sp, bset, nu=1.0 / 1600.0, dt=1e-2, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords
    v0 = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), np.zeros_like(x)])
    state = st.initial_state(v0)
    rows = [dict(step=0, ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel))]
    for _ in range(steps):
        t0 = time.time()
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, p_res=d.p_residual, v_it=list(d.v_iterations),
                         v_res=list(d.v_residual), cfl=d.cfl, div=d.div_norm,
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel),
                         seconds=time.time() - t0))
        print(f"tgv{ne} step {d.step}: p {d.p_iterations} v {d.v_iterations} ke {rows[-1]['ke']:.15g}",
              flush=True)
    return rows


def channel_case(counts, steps):
    """Config-4 analogue: Poiseuille inflow, outflow, no-slip walls, symmetric span."""
    Lx, Ly, Lz = 4 * np.pi / 8, 2.0, 4 * np.pi / 3 / 8
    m = gen_box_mesh((0.0, Lx, 0.0, Ly, 0.0, Lz), counts)
    sp = build_space(m, make_basis(5))

    def pois(x, y, z, t):
        out = np.zeros((3,) + np.shape(x))
        out[0] = 1.5 * y * (2.0 - y)
        return out

    specs = {"xlo": {"kind": "function", "fn": pois}, "xhi": {"kind": "outflow"},
             "ylo": {"kind": "noslip"}, "yhi": {"kind": "noslip"},
             "zlo": {"kind": "symmetry"}, "zhi": {"kind": "symmetry"}}
    bset = BoundarySet(sp, specs)
    st = Stepper(sp, bset, nu=1.0 / 2800.0, dt=2e-3, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords
    rng = np.random.default_rng(3)
    v0 = pois(x, y, z, 0.0)
    v0[1] += 0.05 * np.sin(np.pi * x / Lx) * np.sin(np.pi * y / 2.0) ** 2
    state = st.initial_state(v0)
    rows = []
    for _ in range(steps):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, p_res=d.p_residual, v_it=list(d.v_iterations),
                         v_res=list(d.v_residual), cfl=d.cfl, div=d.div_norm,
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print(f"channel step {d.step}: p {d.p_iterations} v {d.v_iterations}", flush=True)
    del rng
    return rows


KINDS_SPECS = {"xlo": {"kind": "inflow", "u_cl": 1.0, "h": 2.0}, "xhi": {"kind": "outflow"},
               "ylo": {"kind": "noslip"}, "yhi": {"kind": "taylor_green", "nu": 0.01},
               "zlo": {"kind": "symmetry"},
               "zhi": {"kind": "rotor", "u_spin": 0.3, "delta": 0.5, "center": (0.8, 0.0)}}


def channel_kinds_case(counts, steps):
    """Every analytic Dirichlet kind on one box: power-law inflow, decaying-vortex
    wall, spinning wall with its smoothed ramp (delta inside the face)."""
    Lx, Ly, Lz = 4 * np.pi / 8, 2.0, 4 * np.pi / 3 / 8
    sp = build_space(gen_box_mesh((0.0, Lx, 0.0, Ly, 0.0, Lz), counts), make_basis(5))
    st = Stepper(sp, BoundarySet(sp, KINDS_SPECS), nu=1.0 / 2800.0, dt=2e-3, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    state = st.initial_state(np.zeros((3,) + sp.shape))
    rows = []
    for _ in range(steps):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, p_res=d.p_residual, v_it=list(d.v_iterations),
                         v_res=list(d.v_residual), cfl=d.cfl, div=d.div_norm,
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print(f"channel_kinds step {d.step}: p {d.p_iterations} v {d.v_iterations}", flush=True)
    return rows


def gen_bcfun():
    """Reference boundary-value evaluators at sample points (bc.py:36-157)."""
    from semflow import analytic
    from semflow.bc import inflow_profile, rotor_smoothing, rotor_velocity

    rng = np.random.default_rng(11)
    x = rng.uniform(-1.0, 1.0, 400)
    y = np.concatenate([rng.uniform(-0.2, 2.2, 392), [0.0, 0.25, 0.5, 1.0, 2.0, -0.0, 1e-9, 0.5 - 1e-12]])
    z = rng.uniform(-1.0, 1.0, 400)
    x[:3] = 0.25
    z[:3] = 0.0
    x[3] = z[3] = 0.0          # on the rotor axis
    with np.errstate(all="ignore"):
        out = dict(x=x, y=y, z=z,
                   inflow=inflow_profile(y, 1.3, 2.0, 1.0 / 7.0),
                   inflow_sq=inflow_profile(y, 0.7, 2.0, 0.5),
                   ramp=rotor_smoothing(y, 0.9, 0.5),
                   rotor=rotor_velocity(x, y, z, 0.9, 0.5, (0.25, 0.0)),
                   tg=analytic.taylor_green_velocity(x, y, z, 0.37, 0.01))
    np.savez_compressed(os.path.join(OUT, "bcfun.npz"), **out)


def gen_ckpt():
    """A checkpoint written by the reference's own writer (output.py:69-84)."""
    from semflow.output import write_checkpoint

    rng = np.random.default_rng(21)
    arrays = {"vel_0": rng.standard_normal((3, 2, 3, 3, 3)), "prs": rng.standard_normal((2, 3, 3, 3)) * 1e-300,
              "scalar": np.array(np.pi), "proj_p_xs": rng.standard_normal((2, 54))}
    meta = {"case": "golden", "time": 0.125, "nsteps": 10, "primed": False, "n_vel_hist": 1,
            "n_nl_hist": 0, "last_order": 3, "projections": {"p": {"count": 2, "solves": 7}}, "forcing": None}
    write_checkpoint(os.path.join(OUT, "ref_state.ckpt"), arrays, meta)

    # the runner's diagnostics.csv row format (runner.py:92-99)
    from semflow.runner import _DIAG_HEADER, _diag_row
    from semflow.timestep import StepDiagnostics

    d = StepDiagnostics(step=7, time=0.07000000000000001, cfl=0.2012345678901234, div_norm=1.25e-5,
                        p_iterations=33, p_residual=9.87654321e-6, v_iterations=(4, 4, 3),
                        v_residual=(1e-9, 2.5e-9, 3.333e-9), wall_time=0.0123)
    with open(os.path.join(OUT, "diag_row.txt"), "w") as fh:
        fh.write(_DIAG_HEADER + "\n" + _diag_row(d) + "\n")

    # a TGV 3^3 state after 3 steps, checkpointed by the reference's runner, and
    # the diagnostics of 3 more steps of the uninterrupted run
    from types import SimpleNamespace

    from semflow.runner import _save_checkpoint

    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, L), (3, 3, 3)), make_basis(7))
    st = Stepper(sp, BoundarySet(sp, all_tags({"kind": "symmetry"})), nu=1.0 / 1600.0, dt=1e-2, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords
    state = st.initial_state(np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                                       np.zeros_like(x)]))
    for _ in range(3):
        state, _d = st.step(state)
    _save_checkpoint(os.path.join(OUT, "tgv3_step3.ckpt"), SimpleNamespace(name="tgv3"), state, st)
    rows = []
    for _ in range(3):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations),
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
    with open(os.path.join(OUT, "tgv3_restart.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


CYL_MESHES = {
    # the 1/208-scale analogue of config 5: 9728 elements, lx = 8
    "cyl_analogue": dict(diameter=1.0, xlim=(-50.0, 120.0), zlim=(-25.0, 25.0), height=10.0, n_azimuthal=32,
                         n_radial=8, n_axial=4, n_upstream=16, n_downstream=32, n_front=16, n_back=16,
                         geom_order=7),
    # automatic frame counts, explicit collar, 12 sectors
    "cyl_auto": dict(diameter=2.0, xlim=(-6.0, 9.0), zlim=(-5.0, 7.0), height=3.0, n_azimuthal=12, n_radial=3,
                     n_axial=2, collar=1.7, geom_order=4),
}

ROTOR_SPECS = {"inflow": {"kind": "inflow", "u_cl": 1.0, "h": 2.0}, "outflow": {"kind": "outflow"},
               "bottom": {"kind": "noslip"}, "top": {"kind": "symmetry"}, "span": {"kind": "symmetry"},
               "cylinder": {"kind": "rotor", "u_cl": 1.0, "alpha": 3.0, "delta": 0.25}}


def gen_cyl():
    """Cylinder-in-box meshes from the reference generator (mesh.py:231-438), the
    analogue's space maps, and 3 mini-rotor steps (pkg/cases/mini_rotor.json with
    the Jacobi pressure preconditioner)."""
    out = {}
    for key, kw in CYL_MESHES.items():
        m = gen_cylinder_box_mesh(**kw)
        for f in ("vertices", "elements", "facet_elem", "facet_face", "facet_tag", "curved_elem", "curved_coords"):
            out[f"{key}_sha_{f}"] = sha(np.asarray(getattr(m, f)))
            out[f"{key}_shape_{f}"] = np.asarray(np.shape(getattr(m, f)))
        if key == "cyl_analogue":
            t0 = time.time()
            sp = build_space(m, make_basis(7))
            print("analogue build_space", time.time() - t0, flush=True)
            for f in ("coords", "jac", "bm"):
                out[f"{key}_sha_{f}"] = sha(getattr(sp, f))
            for f in ("gid", "perm", "offsets"):
                out[f"{key}_sha_{f}"] = sha(getattr(sp.gs, f))
            out[f"{key}_n_gid"] = np.asarray(sp.gs.n_gid)
            cnt = np.diff(sp.gs.offsets)
            out[f"{key}_mult_hist"] = np.bincount(cnt)
    np.savez_compressed(os.path.join(OUT, "cylinder.npz"), **out)
    # the mini-rotor mesh in the reference's binary file format (mesh.py:444-466)
    from semflow.mesh import write_mesh

    write_mesh(gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                                     n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5),
               os.path.join(OUT, "mini_rotor.mesh"))

    m = gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                              n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5)
    sp = build_space(m, make_basis(5))
    st = Stepper(sp, BoundarySet(sp, ROTOR_SPECS), nu=1.0 / 100.0, dt=2e-3, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x = sp.coords
    v0 = np.zeros((3,) + sp.shape)
    v0[0] = 1.0
    state = st.initial_state(v0)
    rows = []
    for _ in range(3):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations), cfl=d.cfl,
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print("rotor", rows[-1], flush=True)
    del x
    with open(os.path.join(OUT, "rotor_steps.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


def gen_dealias():
    """Over-integration (operators.py:129-158) on the perturbed 3x2x2 order-7 box, the
    GL rule / interpolation matrix, and 3 TGV 4^3 steps with dealias=True."""
    from semflow.basis import gauss_legendre, interp_matrix

    sp = build_space(perturbed_box((3, 2, 2), 17), make_basis(7))
    rng = np.random.default_rng(0)
    rng.standard_normal(sp.shape)
    v = rng.standard_normal((3,) + sp.shape)
    c = rng.standard_normal((3,) + sp.shape)
    dl = ops.Dealias(sp)
    out = {"c": c, "v": v, "advect": ops.advect_vec(sp, c, v, dealias=dl), "wjac_f": dl.wjac_f,
           "interp": dl.interp}
    for m in (3, 8, 12):
        pts, wts = gauss_legendre(m)
        out[f"gl{m}_pts"], out[f"gl{m}_wts"] = pts, wts
        out[f"interp7_to_gl{m}"] = interp_matrix(make_basis(7), pts)
    out["interp_nodes"] = interp_matrix(make_basis(5), np.array([-1.0, 0.3, 1.0, make_basis(5).points[2]]))
    np.savez_compressed(os.path.join(OUT, "dealias.npz"), **out)
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, L), (4, 4, 4)), make_basis(7))
    st = Stepper(sp, BoundarySet(sp, all_tags({"kind": "symmetry"})), nu=1.0 / 1600.0, dt=1e-2, scheme_order=3,
                 dealias=True, pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords
    state = st.initial_state(np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                                       np.zeros_like(x)]))
    rows = []
    for _ in range(3):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations),
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print("dealias tgv4", rows[-1], flush=True)
    with open(os.path.join(OUT, "dealias_tgv4.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


TRIP = dict(x0=0.7, length_x=0.2, length_y=0.1, z_min=0.0, z_max=np.pi / 8, amp_steady=0.02,
            amp_unsteady=0.05, t_scale=2e-3, n_modes=6, seed=5)


def gen_trip():
    """Tripping force (forcing.py:24-133) values over several segments, its state,
    and 3 channel-box steps with it (test_runner.py:117-134 set-up)."""
    from semflow.forcing import TrippingForcing

    trip = TrippingForcing(**TRIP)
    rng = np.random.default_rng(8)
    x = rng.uniform(0.4, 1.0, 64)
    y = rng.uniform(0.0, 0.3, 64)
    z = np.concatenate([rng.uniform(-0.05, np.pi / 8 + 0.05, 60), [0.0, np.pi / 8, -1e-12, 0.2]])
    out = {"x": x, "y": y, "z": z}
    times = [-4e-3, 0.0, 1e-3, 2.5e-3, 9e-3, 9.5e-3, 2.1e-2]
    for k, t in enumerate(times):
        out[f"f{k}"] = trip.evaluate(x, y, z, t)
    out["times"] = np.array(times)
    np.savez_compressed(os.path.join(OUT, "trip.npz"), **out)
    with open(os.path.join(OUT, "trip_state.json"), "w") as fh:
        json.dump(trip.get_state(), fh)
    # channel box with the trip and Poiseuille inflow
    Lx, Ly, Lz = 4 * np.pi / 8, 2.0, 4 * np.pi / 3 / 8
    sp = build_space(gen_box_mesh((0.0, Lx, 0.0, Ly, 0.0, Lz), (6, 4, 3)), make_basis(5))

    def pois(x, y, z, t):
        o = np.zeros((3,) + np.shape(x))
        o[0] = 1.5 * y * (2.0 - y)
        return o

    specs = {"xlo": {"kind": "function", "fn": pois}, "xhi": {"kind": "outflow"},
             "ylo": {"kind": "noslip"}, "yhi": {"kind": "noslip"},
             "zlo": {"kind": "symmetry"}, "zhi": {"kind": "symmetry"}}
    st = Stepper(sp, BoundarySet(sp, specs), nu=1.0 / 2800.0, dt=2e-3, scheme_order=3,
                 forcing=TrippingForcing(**TRIP),
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    xs, ys, zs = sp.coords
    state = st.initial_state(pois(xs, ys, zs, 0.0))
    rows = []
    for _ in range(3):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations),
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print("trip channel", rows[-1], flush=True)
    with open(os.path.join(OUT, "trip_channel.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


def gen_primed():
    """Planar decaying vortex with taylor_green walls, started from an exact
    three-level history (timestep.py:174-200), 3 steps at full order."""
    from semflow import analytic

    L = 2 * np.pi
    nu = 0.01
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, 0.5 * np.pi), (4, 4, 2)), make_basis(6))
    specs = {t: {"kind": "taylor_green", "nu": nu} for t in ("xlo", "xhi", "ylo", "yhi")}
    specs.update({"zlo": {"kind": "symmetry"}, "zhi": {"kind": "symmetry"}})
    st = Stepper(sp, BoundarySet(sp, specs), nu=nu, dt=5e-3, scheme_order=3,
                 pressure=SolverOptions(tol=1e-8, max_iter=300, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-10, max_iter=200, precond="jacobi"))
    state = st.primed_state(lambda x, y, z, t: analytic.taylor_green_velocity(x, y, z, t, nu), 0.0,
                            prs_fn=lambda x, y, z, t: analytic.taylor_green_pressure(x, y, z, t, nu))
    rows = []
    for _ in range(3):
        state, d = st.step(state)
        exact = analytic.taylor_green_velocity(sp.x, sp.y, sp.z, state.time, nu)
        err = float(np.sqrt(sum(sp.integral((state.vel[l] - exact[l]) ** 2) for l in range(3))))
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations),
                         ke=kinetic_energy(sp, state.vel), err=err))
        print("primed tg", rows[-1], flush=True)
    with open(os.path.join(OUT, "primed_tg.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


def gen_schwarz():
    """Hybrid Schwarz preconditioner (precond.py:94-250): one application on a
    perturbed box, GMRES/PCG counts on the 4^3 Poisson box, 3 TGV 4^3 steps."""
    from semflow.precond import HybridSchwarz

    out = {}
    sp = build_space(perturbed_box((3, 2, 2), 17), make_basis(5))
    rng = np.random.default_rng(3)
    r = sp.gs.add(rng.standard_normal(sp.shape))
    mask = np.ones(sp.shape)
    mask.reshape(-1)[sp.facet_flat.ravel()] = 0.0
    for name, mk in (("masked", mask), ("free", None)):
        hs = HybridSchwarz(sp, mask=mk, lam_visc=1.0, lam_mass=0.0 if mk is not None else 0.5)
        out[f"apply_{name}"] = hs(r)
        out[f"wsqrt_{name}"] = hs.wsqrt
        out[f"coarse_diag_{name}"] = hs.coarse_inv_diag
    out["r"] = r
    np.savez_compressed(os.path.join(OUT, "schwarz.npz"), **out)
    res = {}
    sp4 = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (4, 4, 4)), make_basis(7))
    mask = np.ones(sp4.shape)
    mask.reshape(-1)[sp4.facet_flat.ravel()] = 0.0
    x, y, z = sp4.coords
    f = 3.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    rhs = mask * sp4.gs.add(sp4.bm * f)
    A = ops.make_global_op(sp4, 1.0, 0.0, mask)
    M = HybridSchwarz(sp4, mask=mask)
    info = gmres(A, rhs, tol=1e-8, max_iter=200, restart=20, precond=M, dot=sp4.gs.dot)
    res["poisson4_gmres"] = dict(iterations=info.iterations, residual=info.residual,
                                 x_l2=float(np.sqrt(sp4.integral(info.x ** 2))))
    info = pcg(A, rhs, tol=1e-8, max_iter=200, precond=M, dot=sp4.gs.dot)
    res["poisson4_pcg"] = dict(iterations=info.iterations, residual=info.residual)
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, L), (4, 4, 4)), make_basis(7))
    st = Stepper(sp, BoundarySet(sp, all_tags({"kind": "symmetry"})), nu=1.0 / 1600.0, dt=1e-2, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="schwarz"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords
    state = st.initial_state(np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                                       np.zeros_like(x)]))
    rows = []
    for _ in range(4):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations),
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print("schwarz tgv4", rows[-1], flush=True)
    res["tgv4"] = rows
    print(res["poisson4_gmres"], res["poisson4_pcg"])
    with open(os.path.join(OUT, "schwarz.json"), "w") as fh:
        json.dump(res, fh, indent=1)


def main():
    if "--schwarz" in sys.argv:
        gen_schwarz()
        return
    if "--primed" in sys.argv:
        gen_primed()
        return
    if "--trip" in sys.argv:
        gen_trip()
        return
    if "--dealias" in sys.argv:
        gen_dealias()
        return
    if "--cyl" in sys.argv:
        gen_cyl()
        return
    if "--bcfun" in sys.argv:
        gen_bcfun()
        return
    if "--ckpt" in sys.argv:
        gen_ckpt()
        return
    if "--update" in sys.argv:
        # recompute selected solver entries only: --update poisson4 poisson8 ...
        keys = sys.argv[sys.argv.index("--update") + 1:]
        path = os.path.join(OUT, "solvers.json")
        with open(path) as fh:
            sol = json.load(fh)
        for k in keys:
            if k.startswith("poisson"):
                sol[k] = poisson_case(int(k[len("poisson"):]))
            elif k.startswith("tgv"):
                sol[k] = tgv_case(int(k[3:]), 10)
            elif k == "channel_kinds":
                sol[k] = channel_kinds_case((6, 4, 3), 4)
        with open(path, "w") as fh:
            json.dump(sol, fh, indent=1)
        return
    skip_big = "--skip-big" in sys.argv
    gen_kernels()
    gen_basis()
    gen_spaces()
    gen_operators()
    sol = {"versions": {"numpy": np.__version__}}
    sol["poisson4"] = poisson_case(4)
    sol["poisson8"] = poisson_case(8)
    sol["tgv4"] = tgv_case(4, 10)
    sol["channel"] = channel_case((6, 4, 3), 4)
    if not skip_big:
        sol["tgv8"] = tgv_case(8, 10)
        sol["poisson32"] = poisson_case(32)
    with open(os.path.join(OUT, "solvers.json"), "w") as fh:
        json.dump(sol, fh, indent=1)


if __name__ == "__main__":
    main()
