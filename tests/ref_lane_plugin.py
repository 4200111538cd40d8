"""pytest plugin: run the REFERENCE's own test suite with the b200 lane installed.

Loaded by tests/test_ref_hosted.py as ``-p ref_lane_plugin`` in a pytest run over
``baseline/_ref/semflow_tests`` (the unmodified reference tests, vendored by
tools/vendor_ref.sh).  At import it swaps the b200 lane into

* ``semflow.kernels`` -- the lane every reference operator resolves at call time
  (operators.py:18,47; space.py:47-48), and
* ``semflow.kernels._numba`` -- the module the reference's lane tests
  parametrise as ``LANES`` (pkg/tests/test_kernels.py:20-22), so the "numba"
  lane assertions (einsum oracles, lane agreement, thread-count invariance)
  run against the B200 kernels.

Every lane call is counted; the counts go to ``$SEMFLOW_B200_LANE_COUNTS`` at the
end of the session so the caller can prove the device lane really ran.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import semflow.kernels as _K  # noqa: E402  (the vendored reference)
import semflow.kernels._numba as _KNB  # noqa: E402

from paper_2207_07098_b200 import kernels as _b200  # noqa: E402

COUNTS = {name: 0 for name in _b200._EXPORTS}


def _counted(name):
    fn = getattr(_b200, name)

    def wrapper(*args, **kwargs):
        COUNTS[name] += 1
        return fn(*args, **kwargs)

    wrapper.__name__ = name
    wrapper.__doc__ = fn.__doc__
    return wrapper


_IMPORT_LANE = _K.LANE
for _mod in (_K, _KNB):
    _b200.install(_mod)
    for _name in _b200._EXPORTS:
        setattr(_mod, _name, _counted(_name))
# lane_name() keeps reporting the import-time selection: the reference's
# lane-selection tests (test_kernels.py:158-177) are about its env switch, not
# about which functions are bound
_K.LANE = _IMPORT_LANE


def pytest_report_header(config):
    return f"semflow.kernels: b200 device lane installed (selected lane {_K.LANE}; b200 device lane installed into kernels and kernels._numba)"


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("SEMFLOW_B200_LANE_COUNTS")
    if out:
        with open(out, "w") as fh:
            json.dump({"lane": _b200.LANE, "calls": COUNTS}, fh)
