"""Stochastic tripping force (reference forcing.py:24-133; tests/test_forcing.py):
identical random stream and state, field values to rounding, restart, and a
tripped channel run on the GPU."""
import json
import os

import numpy as np
import pytest
import torch

from conftest import rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TRIP = dict(x0=0.7, length_x=0.2, length_y=0.1, z_min=0.0, z_max=np.pi / 8, amp_steady=0.02,
            amp_unsteady=0.05, t_scale=2e-3, n_modes=6, seed=5)


def test_trip_values_and_stream_match_reference():
    from paper_2207_07098_b200.forcing import TrippingForcing

    g = np.load(os.path.join(GOLDEN, "trip.npz"))
    trip = TrippingForcing(**TRIP)
    for k, t in enumerate(g["times"]):
        f = trip.evaluate(g["x"], g["y"], g["z"], float(t)).numpy()
        want = g[f"f{k}"]
        assert np.array_equal(f == 0.0, want == 0.0)          # support: exactly zero outside
        assert np.max(np.abs(f - want)) <= 1e-14 * max(1.0, np.max(np.abs(want)))
    with open(os.path.join(GOLDEN, "trip_state.json")) as fh:
        want_state = json.load(fh)
    assert json.loads(json.dumps(trip.get_state())) == want_state


def test_trip_restart_and_validation():
    from paper_2207_07098_b200.forcing import TrippingForcing

    a = TrippingForcing(**TRIP)
    z = torch.linspace(0.0, np.pi / 8, 7, dtype=torch.float64)
    a.spanwise_signal(z, 5e-3)
    b = TrippingForcing(**TRIP)
    b.set_state(json.loads(json.dumps(a.get_state())))
    for t in (5.5e-3, 9e-3, 2e-2):
        assert torch.equal(a.spanwise_signal(z, t), b.spanwise_signal(z, t))
    with pytest.raises(ValueError, match="backwards"):
        a.spanwise_signal(z, 0.0)
    with pytest.raises(ValueError):
        TrippingForcing(**{**TRIP, "length_x": 0.0})
    zero = TrippingForcing(**{**TRIP, "amp_steady": 0.0, "amp_unsteady": 0.0})
    assert float(zero.evaluate(z, z, z, 1e-3).abs().max()) == 0.0


@pytest.mark.gpu
def test_tripped_channel_steps(cuda, tmp_path):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.bc import BoundarySet
    from paper_2207_07098_b200.checkpoint import load_state, save_state
    from paper_2207_07098_b200.forcing import TrippingForcing
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space
    from paper_2207_07098_b200.timestep import SolverOptions, Stepper, kinetic_energy, poiseuille

    with open(os.path.join(GOLDEN, "trip_channel.json")) as fh:
        rows = json.load(fh)
    Lx, Ly, Lz = 4 * np.pi / 8, 2.0, 4 * np.pi / 3 / 8
    sp = build_space(gen_box_mesh((0.0, Lx, 0.0, Ly, 0.0, Lz), (6, 4, 3)), make_basis(5), device=cuda)
    specs = {"xlo": {"kind": "function", "fn": poiseuille}, "xhi": {"kind": "outflow"},
             "ylo": {"kind": "noslip"}, "yhi": {"kind": "noslip"},
             "zlo": {"kind": "symmetry"}, "zhi": {"kind": "symmetry"}}

    def stepper():
        return Stepper(sp, BoundarySet(sp, specs), nu=1.0 / 2800.0, dt=2e-3, scheme_order=3,
                       forcing=TrippingForcing(**TRIP),
                       pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="jacobi"),
                       velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))

    st = stepper()
    x, y, z = sp.coords.cpu().numpy()
    state = st.initial_state(torch.from_numpy(poiseuille(x, y, z, 0.0)).to(cuda))
    for k, row in enumerate(rows):
        state, d = st.step(state)
        assert d.p_iterations == row["p_it"] and list(d.v_iterations) == row["v_it"]
        assert rel_err(kinetic_energy(sp, state.vel), row["ke"]) < 1e-7
        if k == 0:
            save_state(str(tmp_path / "trip.ckpt"), st, state)
    # restart after step 1 continues the random stream: bitwise the same steps 2-3
    st2 = stepper()
    resumed = load_state(str(tmp_path / "trip.ckpt"), st2)
    for _ in range(len(rows) - 1):
        resumed, _ = st2.step(resumed)
    assert torch.equal(resumed.vel, state.vel)


@pytest.mark.gpu
def test_force_field_equals_pointwise(cuda):
    """force_field evaluates g(z) and the envelope on the distinct coordinate
    values and gathers: bit-identical to the per-point expression."""
    import torch

    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.forcing import TrippingForcing
    from paper_2207_07098_b200.mesh import gen_box_mesh
    from paper_2207_07098_b200.space import build_space

    sp = build_space(gen_box_mesh((0.0, 4.0, 0.0, 2.0, 0.0, 3.0), (4, 3, 5)), make_basis(5), device=cuda)
    trip = TrippingForcing(x0=1.0, y0=0.2, length_x=0.7, length_y=0.3, z_min=0.5, z_max=2.5, amp_steady=0.1,
                           amp_unsteady=0.3, t_scale=0.14, n_modes=40, seed=3)
    ref = TrippingForcing(x0=1.0, y0=0.2, length_x=0.7, length_y=0.3, z_min=0.5, z_max=2.5, amp_steady=0.1,
                          amp_unsteady=0.3, t_scale=0.14, n_modes=40, seed=3)
    for t in (0.01, 0.2, 0.45):
        f = trip.force_field(sp, t)
        x, y, z = sp.coords
        want = ref.evaluate(x, y, z, t)
        assert torch.equal(f[1], want) and float(f[0].abs().max()) == 0.0 and float(f[2].abs().max()) == 0.0
