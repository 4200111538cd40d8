"""Over-integration (reference operators.py:129-158): GL rule and interpolation
matrix on CPU; the device Dealias operator and a dealiased TGV run on the GPU."""
import json
import os

import numpy as np
import pytest
import torch

from conftest import mesh_from_golden, rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden_dealias():
    return np.load(os.path.join(GOLDEN, "dealias.npz"))


def test_gauss_legendre_and_interp_bitwise(golden_dealias):
    from paper_2207_07098_b200.basis import gauss_legendre, interp_matrix, make_basis

    g = golden_dealias
    for m in (3, 8, 12):
        pts, wts = gauss_legendre(m)
        assert np.array_equal(pts, g[f"gl{m}_pts"]) and np.array_equal(wts, g[f"gl{m}_wts"])
        assert np.array_equal(interp_matrix(make_basis(7), pts), g[f"interp7_to_gl{m}"])
    b5 = make_basis(5)
    assert np.array_equal(interp_matrix(b5, np.array([-1.0, 0.3, 1.0, b5.points[2]])), g["interp_nodes"])
    with pytest.raises(ValueError, match="outside"):
        interp_matrix(b5, np.array([1.5]))


@pytest.mark.gpu
@pytest.mark.parametrize("exact", [False, True])
def test_dealias_advect(cuda, golden_dealias, golden_spaces, monkeypatch, exact):
    from paper_2207_07098_b200 import _device, operators as ops
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.space import build_space

    monkeypatch.setattr(_device, "EXACT", exact)
    g = golden_dealias
    sp = build_space(mesh_from_golden(golden_spaces, "pbox322"), make_basis(7), device=cuda)
    dl = ops.Dealias(sp)
    assert np.array_equal(dl.interp, g["interp"])
    c = torch.from_numpy(g["c"]).to(cuda)
    v = torch.from_numpy(g["v"]).to(cuda)
    got = ops.advect_vec(sp, c, v, dealias=dl).cpu().numpy()
    if exact:
        assert np.array_equal(dl.wjac_f.cpu().numpy(), g["wjac_f"])
        assert np.array_equal(got, g["advect"])
    else:
        assert rel_err(got, g["advect"]) < 1e-12


@pytest.mark.gpu
def test_dealiased_tgv_steps(cuda):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.bc import BoundarySet
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space
    from paper_2207_07098_b200.timestep import SolverOptions, Stepper, enstrophy, kinetic_energy

    with open(os.path.join(GOLDEN, "dealias_tgv4.json")) as fh:
        rows = json.load(fh)
    L = 2 * np.pi
    sp = build_space(gen_box_mesh((0.0, L, 0.0, L, 0.0, L), (4, 4, 4)), make_basis(7), device=cuda)
    tags = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")
    st = Stepper(sp, BoundarySet(sp, {t: {"kind": "symmetry"} for t in tags}), nu=1.0 / 1600.0, dt=1e-2,
                 scheme_order=3, dealias=True,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    x, y, z = sp.coords.cpu().numpy()
    v0 = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), np.zeros_like(x)])
    state = st.initial_state(torch.from_numpy(v0).to(cuda))
    for row in rows:
        state, d = st.step(state)
        assert d.p_iterations == row["p_it"] and list(d.v_iterations) == row["v_it"]
        assert rel_err(kinetic_energy(sp, state.vel), row["ke"]) < 1e-9
        assert rel_err(enstrophy(sp, state.vel), row["ens"]) < 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("order", [3, 5, 7])
def test_fused_dealias_equals_chain(cuda, monkeypatch, order):
    """sf_dealias_advect_f64 (one launch, fine grid in shared memory) against the
    contraction chain it replaces: bitwise in exact mode, with the sign applied."""
    from paper_2207_07098_b200 import _device, operators as ops
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space

    monkeypatch.setattr(_device, "EXACT", True)
    sp = build_space(gen_box_mesh((0.0, 1.3, 0.0, 1.0, 0.0, 0.7), (3, 2, 2)), make_basis(order), device=cuda)
    dl = ops.Dealias(sp)
    g = torch.Generator().manual_seed(order)
    c = torch.randn((3,) + sp.shape, generator=g, dtype=torch.float64).to(cuda)
    v = torch.randn((3,) + sp.shape, generator=g, dtype=torch.float64).to(cuda)
    fused = dl.advect_vec(c, v, sign=-1.0)
    cf = [dl._to_fine(c[l]) for l in range(3)]
    chain = -torch.stack([dl._advect_fine(cf, v[l]) for l in range(3)])
    assert torch.equal(fused, chain)
