"""Hybrid overlapping Schwarz preconditioner on the device (reference
precond.py:94-250): one application vs the reference, Krylov counts, and the
TGV step with the reference's default pressure preconditioner."""
import json
import os

import numpy as np
import pytest
import torch

from conftest import mesh_from_golden, rel_err

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden_schwarz():
    with open(os.path.join(GOLDEN, "schwarz.json")) as fh:
        return json.load(fh), np.load(os.path.join(GOLDEN, "schwarz.npz"))


def test_schwarz_apply(cuda, golden_spaces, golden_schwarz):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.precond import HybridSchwarz
    from paper_2207_07098_b200.space import build_space

    _, g = golden_schwarz
    sp = build_space(mesh_from_golden(golden_spaces, "pbox322"), make_basis(5), device=cuda)
    r = torch.from_numpy(g["r"]).to(cuda)
    mask = torch.ones(sp.shape, dtype=torch.float64, device=cuda)
    mask.view(-1)[sp.facet_flat.reshape(-1)] = 0.0
    for name, mk, lm in (("masked", mask, 0.0), ("free", None, 0.5)):
        hs = HybridSchwarz(sp, mask=mk, lam_visc=1.0, lam_mass=lm)
        assert np.array_equal(hs.wsqrt.cpu().numpy(), g[f"wsqrt_{name}"][hs.gid_of_node.cpu().numpy()])
        assert rel_err(hs.coarse_inv_diag.cpu().numpy(), g[f"coarse_diag_{name}"]) < 1e-12
        assert rel_err(hs(r).cpu().numpy(), g[f"apply_{name}"]) < 1e-10, name
        assert torch.equal(hs(r), hs(r))          # deterministic


def test_schwarz_krylov_counts(cuda, golden_schwarz):
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.precond import HybridSchwarz
    from paper_2207_07098_b200.space import build_space

    res, _ = golden_schwarz
    sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (4, 4, 4)), make_basis(7), device=cuda)
    mask = torch.ones(sp.shape, dtype=torch.float64, device=cuda)
    mask.view(-1)[sp.facet_flat.reshape(-1)] = 0.0
    x, y, z = sp.coords
    f = 3.0 * np.pi ** 2 * torch.sin(np.pi * x) * torch.sin(np.pi * y) * torch.sin(np.pi * z)
    rhs = mask * sp.gs.add(sp.bm * f)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    M = HybridSchwarz(sp, mask=mask)
    info = krylov.gmres(A, rhs, tol=1e-8, max_iter=200, restart=20, precond=M, dot=sp.gs.dot)
    assert info.iterations == res["poisson4_gmres"]["iterations"]
    assert rel_err(float(np.sqrt(sp.integral(info.x ** 2))), res["poisson4_gmres"]["x_l2"]) < 1e-9
    info = krylov.pcg(A, rhs, tol=1e-8, max_iter=200, precond=M, dot=sp.gs.dot)
    assert info.iterations == res["poisson4_pcg"]["iterations"]


def test_schwarz_tgv_steps(cuda, golden_schwarz):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.bc import BoundarySet
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space
    from paper_2207_07098_b200.timestep import SolverOptions, Stepper, enstrophy, kinetic_energy

    res, _ = golden_schwarz
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, L), (4, 4, 4)), make_basis(7), device=cuda)
    tags = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")
    st = Stepper(sp, BoundarySet(sp, {t: {"kind": "symmetry"} for t in tags}), nu=1.0 / 1600.0, dt=1e-2,
                 scheme_order=3, pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="schwarz"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords.cpu().numpy()
    v0 = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), np.zeros_like(x)])
    state = st.initial_state(torch.from_numpy(v0).to(cuda))
    for row in res["tgv4"]:
        state, d = st.step(state)
        assert d.p_iterations == row["p_it"] and list(d.v_iterations) == row["v_it"], (d, row)
        assert rel_err(kinetic_energy(sp, state.vel), row["ke"]) < 1e-9
        assert rel_err(enstrophy(sp, state.vel), row["ens"]) < 1e-9


def test_schwarz_kernel_vs_host_restatement(cuda):
    """HybridSchwarz.apply_into against the numpy restatement of its stages on
    the same device-built structures (tests/test_schwarz_setup.py::_emulate)."""
    from test_schwarz_setup import _emulate

    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.precond import HybridSchwarz
    from paper_2207_07098_b200.space import build_space

    sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 2.0, 0.0, 1.0), (6, 5, 4)), make_basis(5), device=cuda)
    mask = torch.ones(sp.shape, dtype=torch.float64, device=cuda)
    mask.view(-1)[sp.facet_flat.reshape(-1)] = 0.0
    r = torch.randn(sp.shape, dtype=torch.float64, generator=torch.Generator().manual_seed(3)).to(cuda)
    for mk in (mask, None):
        hs = HybridSchwarz(sp, mask=mk, lam_visc=1.0, lam_mass=0.0 if mk is not None else 0.3)
        got = hs(r).cpu().numpy()
        want = _emulate(hs, r.cpu().numpy())
        assert rel_err(got, want) < 1e-13
        assert torch.equal(hs(r), hs(r))
        assert hs.n_classes <= 125


def test_schwarz_fused_gmres_matches_generic(cuda, monkeypatch):
    """The fused (graph-captured, flexible) GMRES with hybrid Schwarz against the
    generic torch loop: identical iteration counts, solutions to rounding."""
    from paper_2207_07098_b200 import krylov, operators as ops
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.precond import HybridSchwarz
    from paper_2207_07098_b200.space import build_space

    sp = build_space(gen_box_mesh((0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (8, 8, 8)), make_basis(7), device=cuda)
    mask = torch.ones(sp.shape, dtype=torch.float64, device=cuda)
    mask.view(-1)[sp.facet_flat.reshape(-1)] = 0.0
    x, y, z = sp.coords
    f = 3.0 * np.pi ** 2 * torch.sin(np.pi * x) * torch.sin(np.pi * y) * torch.sin(np.pi * z)
    rhs = mask * sp.gs.add(sp.bm * f)
    A = ops.make_global_op(sp, 1.0, 0.0, mask)
    M = HybridSchwarz(sp, mask=mask)
    fused = krylov.gmres(A, rhs, tol=1e-8, max_iter=200, restart=20, precond=M, dot=sp.gs.dot)
    again = krylov.gmres(A, rhs, tol=1e-8, max_iter=200, restart=20, precond=M, dot=sp.gs.dot)
    assert torch.equal(fused.x, again.x)                       # graph replay is deterministic
    gen = krylov._gmres_generic(A, rhs, 1e-8, 200, 20, M, sp.gs.dot, None)
    assert fused.iterations == gen.iterations and fused.converged
    assert rel_err(fused.x.cpu().numpy(), gen.x.cpu().numpy()) < 1e-9
