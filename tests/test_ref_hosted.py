"""Reference-hosted drop-in proof.

The UNMODIFIED reference, vendored into ``baseline/_ref`` by tools/vendor_ref.sh
(pip install of /root/reference/pkg plus its test suite; git-ignored, shipped to
the GPU box with the snapshot), is driven through the b200 lane:

* ``test_reference_suite_on_b200_lane``: the reference's own 257 tests
  (pkg/tests/, incl. the LANES assertions test_kernels.py:68-95,140-155 and the
  dense-stiffness operator oracle test_operators.py:25-34) with
  ``kernels.install()`` applied to ``semflow.kernels`` and
  ``semflow.kernels._numba`` (tests/ref_lane_plugin.py);
* ``test_from_reference_space``: a reference ``FunctionSpace`` uploaded with
  ``space.from_reference`` gives our device operators the reference's results.

Nothing here reads /root/reference at run time.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "semflow_tests")

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "semflow")),
                       reason="baseline/_ref not vendored (tools/vendor_ref.sh)"),
]


def _env(tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env["NUMBA_CACHE_DIR"] = str(tmp_path / "numba_cache")
    env["SEMFLOW_B200_LANE_COUNTS"] = str(tmp_path / "lane_counts.json")
    return env


def test_reference_suite_on_b200_lane(tmp_path):
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\n")   # keep this repo's ini/conftest out of the reference run
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", str(ini), "-p", "no:cacheprovider",
           "-p", "ref_lane_plugin", REF_TESTS]
    res = subprocess.run(cmd, cwd=REF_TESTS, env=_env(tmp_path), capture_output=True, text=True,
                         timeout=1500)
    tail = "\n".join(res.stdout.splitlines()[-15:])
    log = os.environ.get("SEMFLOW_B200_REF_LOG")
    if log:
        with open(log, "w") as fh:
            fh.write(res.stdout + res.stderr)
    assert res.returncode == 0, tail + res.stderr[-2000:]
    with open(tmp_path / "lane_counts.json") as fh:
        counts = json.load(fh)
    assert counts["lane"] == "b200"
    # every plugin entry point was exercised by the reference's tests
    missing = [k for k, v in counts["calls"].items() if v == 0]
    assert not missing, (missing, counts)


def _ref_modules():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/semflow_numba_cache")
    from semflow import operators as rops
    from semflow.basis import make_basis
    from semflow.mesh import gen_box_mesh, gen_cylinder_box_mesh
    from semflow.space import build_space
    return rops, make_basis, gen_box_mesh, gen_cylinder_box_mesh, build_space


def test_from_reference_space():
    import torch

    from paper_2207_07098_b200 import operators as ops
    from paper_2207_07098_b200.space import from_reference

    rops, make_basis, gen_box_mesh, gen_cyl, rbuild = _ref_modules()
    meshes = [
        (gen_box_mesh((0.0, 1.5, 0.0, 1.0, 0.0, 2.0), (3, 2, 2)), 7),
        (gen_cyl(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                 n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5), 5),
    ]
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    for mesh, order in meshes:
        rsp = rbuild(mesh, make_basis(order))
        sp = from_reference(rsp, device=dev)
        u = rng.standard_normal(rsp.shape)
        ud = torch.from_numpy(u).to(dev)
        # gather-scatter: bitwise (same maps, same sequential order)
        assert np.array_equal(sp.gs.add(ud).cpu().numpy(), rsp.gs.add(u))
        mask = np.ones(rsp.shape)
        mask.reshape(-1)[np.asarray(rsp.facet_flat).ravel()] = 0.0
        md = torch.from_numpy(mask).to(dev)
        for lv, lm, mk in ((1.0, 0.0, None), (0.3, 7.0, mask)):
            want = rops.make_global_op(rsp, lv, lm, mk)(u)
            got = ops.make_global_op(sp, lv, lm, None if mk is None else md)(ud).cpu().numpy()
            err = np.abs(got - want).max() / np.abs(want).max()
            assert err <= 1e-12, (order, lv, lm, err)
        # glsc3 through the uploaded multiplicities
        d_ref = rsp.gs.dot(u, u)
        d = sp.gs.dot(ud, ud)
        d = float(d) if not torch.is_tensor(d) else float(d.item())
        assert abs(d - d_ref) <= 1e-13 * abs(d_ref)
