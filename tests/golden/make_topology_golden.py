"""Record the REFERENCE's outcome on the topology cases (run here only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_topology_golden.py

For every recipe of tests/topology_cases.py: the reference ``Mesh.validate``
(mesh.py:95-147) and ``build_space`` (space.py:195-314) outcome -- the exception
class and message, or sha256 of gid/perm/offsets -- into topology.json.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from semflow.basis import make_basis  # noqa: E402
from semflow.mesh import Mesh  # noqa: E402
from semflow.space import build_space  # noqa: E402

import topology_cases  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(fn):
    try:
        return {"ok": True, "value": fn()}
    except Exception as exc:  # noqa: BLE001 -- the class name is the record
        return {"ok": False, "error": type(exc).__name__, "message": str(exc)}


def main():
    res = {}
    for name, (arrays, order) in topology_cases.cases().items():
        mesh = topology_cases.as_mesh(arrays, Mesh)
        val = outcome(lambda: (mesh.validate(), None)[1])

        def build():
            sp = build_space(mesh, make_basis(order))
            return {"gid": sha(sp.gs.gid), "perm": sha(sp.gs.perm), "offsets": sha(sp.gs.offsets),
                    "n_gid": int(sp.gs.n_gid)}

        res[name] = {"order": order, "validate": val, "build": outcome(build)}
        print(name, res[name]["validate"].get("error"), res[name]["build"].get("error"),
              res[name]["build"].get("message", "")[:90])
    with open(os.path.join(HERE, "topology.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
