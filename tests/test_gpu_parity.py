"""CUDA path vs the reference (golden fixtures) and the CPU oracle -- needs a B200.

Bars (BASELINE.json north_star): gather-scatter maps bit-exact; Ax / dssum within
1e-12 relative (production DFMA arithmetic) and bit-identical in exact mode;
identical Krylov iteration counts.
"""

import hashlib

import numpy as np
import pytest
import torch

from conftest import mesh_from_golden, rel_err

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture
def exact(monkeypatch):
    from paper_2207_07098_b200 import _device

    monkeypatch.setattr(_device, "EXACT", True)
    yield


# ------------------------------------------------------------------ kernel lane (plugin API)

@pytest.mark.parametrize("tag", ["n5", "n6", "n8"])
def test_lane_bitwise_vs_reference(cuda, golden_kernels, tag):
    from paper_2207_07098_b200 import kernels as K

    g = golden_kernels
    a, geo, b, u = g[f"{tag}_a"], g[f"{tag}_g"], g[f"{tag}_b"], g[f"{tag}_u"]
    for ax, fn in enumerate((K.apply_r, K.apply_s, K.apply_t)):
        assert np.array_equal(fn(a, u), g[f"{tag}_apply{ax}"])
        assert np.array_equal(fn(g[f"{tag}_rect"], u), g[f"{tag}_rect{ax}"])
    ur, us, ut = K.grad_ref(a, u)
    assert np.array_equal(ur, g[f"{tag}_ur"]) and np.array_equal(us, g[f"{tag}_us"])
    assert np.array_equal(ut, g[f"{tag}_ut"])
    for k, (lv, lm) in enumerate(((1.0, 0.0), (0.7, 2.5), (1.0, 0.3))):
        assert np.array_equal(K.ax_helmholtz_local(a, geo, b, u, lv, lm), g[f"{tag}_ax{k}"])


def test_lane_gather_scatter(cuda, golden_kernels):
    from paper_2207_07098_b200 import kernels as K

    g = golden_kernels
    sums = K.gs_gather(g["gs_vals"], g["gs_perm"], g["gs_off"])
    assert np.array_equal(sums, g["gs_sums"])
    out = np.zeros(g["gs_vals"].size)
    ret = K.gs_scatter(sums, g["gs_perm"], g["gs_off"], out)
    assert ret is out and np.array_equal(out, g["gs_scat"])


# ------------------------------------------------------------------ device space build

@pytest.mark.parametrize("key", ["box211", "cube222", "pbox322", "pbox543", "tgv4", "tgv8", "rotor"])
def test_device_build_space_bit_exact(cuda, golden_spaces, key):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.space import build_space

    g = golden_spaces
    m = mesh_from_golden(g, key)
    sp = build_space(m, make_basis(int(g[f"{key}_order"])), device=cuda)
    for name in ("coords", "jac", "bm", "rx"):
        assert sha(getattr(sp, name).cpu().numpy()) == str(g[f"{key}_sha_{name}"]), name
    for name in ("gid", "perm", "offsets"):
        assert sha(getattr(sp.gs, name).cpu().numpy()) == str(g[f"{key}_sha_{name}"]), name
    assert sp.gs.n_gid == int(g[f"{key}_n_gid"])
    assert abs(sp.volume - float(g[f"{key}_volume"])) <= 1e-13 * float(g[f"{key}_volume"])
    assert abs(float(sp.facet_warea.sum()) - float(g[f"{key}_warea_sum"])) <= 1e-12 * float(g[f"{key}_warea_sum"])


def test_device_geom_equals_oracle(cuda, oracle, golden_spaces):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.space import build_space

    m = mesh_from_golden(golden_spaces, "rotor")
    sp = build_space(m, make_basis(5), device=cuda)
    osp = oracle.build_space(m, oracle.make_basis(5))
    assert np.array_equal(sp.geom.cpu().numpy(), osp.geom)


# ------------------------------------------------------------------ operators

@pytest.fixture(scope="module")
def pbox(golden_spaces):
    import torch as _t

    if not _t.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.space import build_space

    return build_space(mesh_from_golden(golden_spaces, "pbox322"), make_basis(7), device="cuda:0")


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def test_operators_fast_mode(cuda, golden_ops, pbox):
    from paper_2207_07098_b200 import operators as ops
    from paper_2207_07098_b200.precond import BlockJacobi

    g, sp = golden_ops, pbox
    u, v, c, mask = _t(g["u"]), _t(g["v"]), _t(g["c"]), _t(g["mask"])
    tol = 1e-12
    assert rel_err(ops.laplace_local(sp, u).cpu().numpy(), g["ax_poisson"]) < tol
    assert rel_err(ops.helmholtz_local(sp, u, 0.3, 7.0).cpu().numpy(), g["ax_helm"]) < tol
    assert rel_err(ops.make_global_op(sp, 1.0, 0.0, mask)(u).cpu().numpy(), g["gop_poisson_masked"]) < tol
    assert rel_err(ops.make_global_op(sp, 0.3, 7.0, mask)(u).cpu().numpy(), g["gop_helm_masked"]) < tol
    assert rel_err(ops.make_global_op(sp, 1.0, 0.0)(u).cpu().numpy(), g["gop_poisson"]) < tol
    assert np.array_equal(sp.gs.add(u).cpu().numpy(), g["gs_add"])
    assert np.array_equal(sp.gs.avg(u).cpu().numpy(), g["gs_avg"])
    assert np.array_equal(sp.gs.add(v).cpu().numpy(), g["gs_add_vec"])
    assert rel_err(sp.gs.dot(u, v[0]), g["gs_dot"]) < 1e-13
    assert rel_err(sp.integral(u), g["integral"]) < 1e-13
    for name, got in (("grad", ops.grad(sp, u)), ("div", ops.div(sp, v)), ("curl", ops.curl(sp, v)),
                      ("advect", ops.advect_vec(sp, c, v)), ("wgd", ops.weak_grad_dot(sp, v))):
        assert rel_err(got.cpu().numpy(), g[name]) < tol, name
    assert rel_err(ops.cfl(sp, v, 0.01), g["cfl"]) < 1e-14
    assert rel_err(BlockJacobi(sp, 1.0, 0.0, mask).inv_diag.cpu().numpy(), g["jacobi_p"]) < 1e-15
    assert rel_err(BlockJacobi(sp, 0.3, 7.0, mask).inv_diag.cpu().numpy(), g["jacobi_h"]) < 1e-15


def test_operators_exact_mode_bitwise(cuda, exact, oracle, golden_ops, golden_spaces, pbox):
    """Exact mode reproduces the reference numba lane bit for bit (rx/bm-based
    operators vs the golden arrays; geom-based ones vs the oracle on the same geom)."""
    from paper_2207_07098_b200 import operators as ops

    g, sp = golden_ops, pbox
    u, v, c, mask = _t(g["u"]), _t(g["v"]), _t(g["c"]), _t(g["mask"])
    for name, got in (("grad", ops.grad(sp, u)), ("div", ops.div(sp, v)), ("curl", ops.curl(sp, v)),
                      ("advect", ops.advect_vec(sp, c, v)), ("wgd", ops.weak_grad_dot(sp, v))):
        assert np.array_equal(got.cpu().numpy(), g[name]), name
    assert ops.cfl(sp, v, 0.01) == float(g["cfl"])
    osp = oracle.build_space(mesh_from_golden(golden_spaces, "pbox322"), oracle.make_basis(7))
    un, mn = g["u"], g["mask"]
    assert np.array_equal(ops.laplace_local(sp, u).cpu().numpy(),
                          oracle.ax_helmholtz_local(osp.basis.dmat, osp.geom, osp.bm, un, 1.0, 0.0))
    for lv, lm in ((1.0, 0.0), (0.3, 7.0)):
        want = oracle.make_global_op(osp, lv, lm, mn)(un)
        assert np.array_equal(ops.make_global_op(sp, lv, lm, mask)(u).cpu().numpy(), want)


@pytest.fixture(scope="module")
def tgv8():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space

    L = 2 * np.pi
    return build_space(gen_box_mesh((0, L, 0, L, 0, L), (8, 8, 8)), make_basis(7), device="cuda:0")


def test_ax_dssum_config1_size(cuda, oracle, tgv8):
    """Assembled operator on the 8^3 lx=8 TGV mesh vs the oracle (<=1e-12), masked and not."""
    from paper_2207_07098_b200 import operators as ops

    sp = tgv8
    osp = oracle.build_space(oracle.gen_box_mesh((0, 2 * np.pi, 0, 2 * np.pi, 0, 2 * np.pi), (8, 8, 8)),
                             oracle.make_basis(7))
    un = np.random.default_rng(0).standard_normal(osp.shape)
    mn = np.ones(osp.shape)
    mn.reshape(-1)[osp.facet_flat.ravel()] = 0.0
    u, mask = _t(un), _t(mn)
    for lv, lm, mk in ((1.0, 0.0, None), (1.0, 0.0, mn), (1.0 / 1600, 183.3, mn)):
        want = oracle.make_global_op(osp, lv, lm, mk)(un)
        got = ops.make_global_op(sp, lv, lm, None if mk is None else mask)(u).cpu().numpy()
        assert rel_err(got, want) <= 1e-12
    w = ops.laplace_local(sp, u)
    assert np.array_equal(sp.gs.add(w).cpu().numpy(), osp.gs.add(w.cpu().numpy()))   # dssum bit-exact


def test_operator_is_deterministic(cuda, tgv8):
    from paper_2207_07098_b200 import operators as ops

    sp = tgv8
    u = torch.randn(sp.shape, dtype=torch.float64, device="cuda:0")
    a = ops.make_global_op(sp, 1.0, 0.0)
    x, y = a(u), a(u)
    assert torch.equal(x, y)
    d1, d2 = sp.gs.dot(x, u), sp.gs.dot(x, u)
    assert d1 == d2


# ------------------------------------------------------------------ solvers

def _poisson_dev(ne):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space

    sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (ne, ne, ne)), make_basis(7), device="cuda:0")
    mask = torch.ones(sp.shape, dtype=torch.float64, device=sp.device)
    mask.view(-1)[sp.facet_flat.reshape(-1)] = 0.0
    x, y, z = sp.coords
    f = 3.0 * np.pi ** 2 * torch.sin(np.pi * x) * torch.sin(np.pi * y) * torch.sin(np.pi * z)
    rhs = mask * sp.gs.add(sp.bm * f)
    return sp, mask, rhs


@pytest.mark.parametrize("ne", [4, 8])
def test_pcg_gmres_iteration_counts(cuda, golden_solvers, ne):
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.precond import BlockJacobi

    sp, mask, rhs = _poisson_dev(ne)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    M = BlockJacobi(sp, 1.0, 0.0, mask)
    want = golden_solvers[f"poisson{ne}"]
    info = krylov.pcg(A, rhs, tol=1e-8, max_iter=500, precond=M, dot=sp.gs.dot)
    assert info.converged and info.iterations == want["pcg"]["iterations"]
    # final residuals agree to the level the reference's own two lanes do
    # (numba vs numpy: 9.499e-9 vs 9.523e-9 at 32^3)
    assert rel_err(info.residual, want["pcg"]["residual"]) < 2e-2
    assert rel_err(sp.l2_norm(info.x), want["pcg"]["x_l2"]) < 1e-10
    # restart 20 (the Stepper's pressure setting); GMRES(10) here takes ~280
    # iterations and the reference's own numba and numpy lanes disagree on it
    # (278 vs 279), so it is not a meaningful parity case
    info = krylov.gmres(A, rhs, tol=1e-8, max_iter=500, restart=20, precond=M, dot=sp.gs.dot)
    assert info.iterations == want["gmres"]["iterations"]
    # the look-ahead (pipelined) GMRES takes the same iterations to the same x
    import os

    os.environ["SEMFLOW_B200_GMRES_PIPELINE"] = "1"
    try:
        info_p = krylov.gmres(A, rhs, tol=1e-8, max_iter=500, restart=20, precond=M, dot=sp.gs.dot)
    finally:
        del os.environ["SEMFLOW_B200_GMRES_PIPELINE"]
    assert info_p.iterations == info.iterations and torch.equal(info_p.x, info.x)
    info = krylov.pcg(A, rhs, tol=1e-8, max_iter=500, dot=sp.gs.dot)
    assert info.iterations == want["cg_noprec"]["iterations"]
    proj = krylov.ProjectionSpace(sp.gs.dot)
    for k, row in enumerate(want["projection"]):
        x0, b = proj.prepare(rhs * (1.0 + 0.1 * k), A)
        inf = krylov.pcg(A, b, tol=1e-8, max_iter=500, precond=M, dot=sp.gs.dot)
        proj.absorb(inf.x, A)
        assert inf.iterations == row["iterations"] and proj.count == row["count"]


def test_pcg_config2_42_iterations(cuda, golden_solvers):
    """Config 2 (32^3 Poisson, lx=8): the reference takes 42 Jacobi-PCG iterations."""
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.precond import BlockJacobi

    sp, mask, rhs = _poisson_dev(32)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    info = krylov.pcg(A, rhs, tol=1e-8, max_iter=500, precond=BlockJacobi(sp, 1.0, 0.0, mask), dot=sp.gs.dot)
    want = golden_solvers["poisson32"]["pcg"]
    assert info.converged and info.iterations == want["iterations"] == 42
    assert rel_err(info.residual, want["residual"]) < 2e-2
    assert rel_err(sp.l2_norm(info.x), want["x_l2"]) < 1e-10


def test_generic_solver_path_matches_fused(cuda):
    """Arbitrary callables take the generic path; it must agree with the fused one."""
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.precond import BlockJacobi

    sp, mask, rhs = _poisson_dev(4)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    M = BlockJacobi(sp, 1.0, 0.0, mask)
    fused = krylov.pcg(A, rhs, tol=1e-8, max_iter=500, precond=M, dot=sp.gs.dot)
    generic = krylov.pcg(lambda v: A(v), rhs, tol=1e-8, max_iter=500, precond=lambda r: M(r), dot=sp.gs.dot)
    assert fused.iterations == generic.iterations
    # the generic path rounds x += alpha p in two steps (torch), the fused one
    # uses DFMA: after 44 iterations the iterates differ at the ~1e-10 level
    assert rel_err(fused.x.cpu().numpy(), generic.x.cpu().numpy()) < 1e-8


def test_gmres_graph_replay_reuse(cuda, golden_solvers, monkeypatch):
    """Look-ahead GMRES replaying captured Arnoldi steps: the first solve captures,
    later solves (other right-hand sides) replay; every solve equals the
    un-captured path bit for bit and the reference's iteration count."""
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.precond import BlockJacobi

    sp, mask, rhs = _poisson_dev(4)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    M = BlockJacobi(sp, 1.0, 0.0, mask)
    monkeypatch.setenv("SEMFLOW_B200_GMRES_PIPELINE", "1")
    want_its = golden_solvers["poisson4"]["gmres"]["iterations"]
    results = []
    for scale in (1.0, 0.5, 1.0):
        info = krylov.gmres(A, rhs * scale, tol=1e-8 * scale, max_iter=500, restart=20, precond=M, dot=sp.gs.dot)
        results.append(info)
        assert info.iterations == want_its
    assert A._gmres_graphs.graphs          # captured steps exist and were reused
    monkeypatch.setenv("SEMFLOW_B200_GRAPHS", "0")
    plain = krylov.gmres(A, rhs, tol=1e-8, max_iter=500, restart=20, precond=M, dot=sp.gs.dot)
    assert torch.equal(plain.x, results[0].x) and torch.equal(plain.x, results[2].x)
