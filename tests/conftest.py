"""Shared fixtures: golden data (generated from the reference), the CPU oracle,
and the `gpu` marker (tests that need a B200 and libsemflow_b200.so)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def load_npz(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


@pytest.fixture(scope="session")
def golden_kernels():
    return load_npz("kernels.npz")


@pytest.fixture(scope="session")
def golden_basis():
    return load_npz("basis.npz")


@pytest.fixture(scope="session")
def golden_spaces():
    return load_npz("spaces.npz")


@pytest.fixture(scope="session")
def golden_ops():
    return load_npz("operators.npz")


@pytest.fixture(scope="session")
def golden_bcfun():
    return load_npz("bcfun.npz")


@pytest.fixture(scope="session")
def golden_solvers():
    with open(os.path.join(GOLDEN, "solvers.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    import semflow_oracle

    semflow_oracle.lib()
    return semflow_oracle


def mesh_from_golden(g, key):
    """Rebuild a product Mesh from the arrays stored by make_golden.py."""
    from paper_2207_07098_b200.mesh import Mesh

    go = int(g[f"{key}_geom_order"])
    return Mesh(
        vertices=g[f"{key}_vertices"], elements=g[f"{key}_elements"],
        facet_elem=g[f"{key}_facet_elem"], facet_face=g[f"{key}_facet_face"],
        facet_tag=g[f"{key}_facet_tag"], tag_names=tuple(json.loads(str(g[f"{key}_tags"]))),
        curved_elem=g[f"{key}_curved_elem"], curved_coords=g[f"{key}_curved_coords"],
        geom_order=None if go < 0 else go)


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = float(np.abs(b).max()) if b.size else 0.0
    return float(np.abs(a - b).max()) / (den if den > 0 else 1.0)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_07098_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)
