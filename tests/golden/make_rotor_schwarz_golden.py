"""The mini-rotor case with the reference's DEFAULT pressure preconditioner
(hybrid Schwarz, pkg/cases/mini_rotor.json: GMRES(20) tol 1e-5, projection on),
3 steps of the reference Stepper (run here only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_rotor_schwarz_golden.py

writes rotor_schwarz_steps.json (per-step iteration counts, CFL, kinetic energy,
enstrophy) for tests/test_gpu_stepper.py::test_mini_rotor_schwarz_steps.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from semflow.basis import make_basis  # noqa: E402
from semflow.bc import BoundarySet  # noqa: E402
from semflow import operators as ops  # noqa: E402
from semflow.diagnostics import kinetic_energy  # noqa: E402
from semflow.mesh import gen_cylinder_box_mesh  # noqa: E402
from semflow.space import build_space  # noqa: E402
from semflow.timestep import SolverOptions, Stepper  # noqa: E402

def enstrophy(sp, v):
    """0.5 (curl v, curl v), as tests/golden/make_golden.py records it."""
    w = ops.curl(sp, v)
    return 0.5 * sp.integral(w[0] ** 2 + w[1] ** 2 + w[2] ** 2)


SPECS = {"inflow": {"kind": "inflow", "u_cl": 1.0, "h": 2.0}, "outflow": {"kind": "outflow"},
         "bottom": {"kind": "noslip"}, "top": {"kind": "symmetry"}, "span": {"kind": "symmetry"},
         "cylinder": {"kind": "rotor", "u_cl": 1.0, "alpha": 3.0, "delta": 0.25}}


def main():
    m = gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                              n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5)
    sp = build_space(m, make_basis(5))
    st = Stepper(sp, BoundarySet(sp, SPECS), nu=1.0 / 100.0, dt=2e-3, scheme_order=3,
                 pressure=SolverOptions(tol=1e-5, max_iter=200, restart=20, precond="schwarz", projection=True),
                 velocity=SolverOptions(tol=1e-8, max_iter=100, precond="jacobi"))
    v0 = np.zeros((3,) + sp.shape)
    v0[0] = 1.0
    state = st.initial_state(v0)
    rows = []
    for _ in range(3):
        state, d = st.step(state)
        rows.append(dict(step=d.step, p_it=d.p_iterations, v_it=list(d.v_iterations), cfl=d.cfl,
                         ke=kinetic_energy(sp, state.vel), ens=enstrophy(sp, state.vel)))
        print("rotor schwarz", rows[-1], flush=True)
    with open(os.path.join(HERE, "rotor_schwarz_steps.json"), "w") as fh:
        json.dump({"elements": int(m.n_elements), "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
