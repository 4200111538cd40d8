"""Mesh validation and the geometric gather-scatter cross-check against the
reference's outcomes (tests/golden/topology.json from make_topology_golden.py).

CPU: ``topology.validate_mesh`` raises the reference's TopologyError with the
reference's message on every malformed mesh (mesh.py:95-147), and the pair
search / component labelling reproduce the reference's geometric grouping.
GPU: ``build_space`` raises what the reference's build_space raises
(GeometryError before TopologyError, space.py:224-291) or yields its maps bit for
bit -- including a mesh whose duplicated vertex ids make the topological groups
differ from the geometric ones.
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import topology_cases
from paper_2207_07098_b200 import errors, topology
from paper_2207_07098_b200.mesh import Mesh

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "topology.json")


def _gold():
    with open(GOLD) as fh:
        return json.load(fh)


CASES = topology_cases.cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_validate_matches_reference(name):
    want = _gold()[name]["validate"]
    mesh = topology_cases.as_mesh(CASES[name][0], Mesh)
    if want["ok"]:
        topology.validate_mesh(mesh)
    else:
        with pytest.raises(getattr(errors, want["error"])) as ei:
            topology.validate_mesh(mesh)
        assert str(ei.value) == want["message"]


def test_mesh_validate_method():
    mesh = topology_cases.as_mesh(CASES["hanging_2to1"][0], Mesh)
    with pytest.raises(errors.TopologyError, match="carries no boundary tag"):
        mesh.validate()
    assert topology_cases.as_mesh(CASES["valid_box"][0], Mesh).validate() is not None


def _coords(arrays, order):
    """Trilinear GLL coordinates (3, E, n, n, n) as the reference computes them."""
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.space import _wc

    b = make_basis(order)
    corners = np.asarray(arrays["vertices"])[np.asarray(arrays["elements"])]
    c = np.einsum("ecl,cp->lep", corners, _wc(b.points))
    return torch.from_numpy(c.reshape(3, -1, b.n, b.n, b.n))


def test_pairs_and_components_cpu():
    """Pair search vs brute force; components vs a host union-find."""
    rng = np.random.default_rng(3)
    arrays, order = CASES["split_face_half"]
    coords = _coords(arrays, order)
    tol = topology.gs_tolerance(topology_cases.as_mesh(arrays, Mesh))
    pairs = topology.coincident_pairs(coords, tol, chunk=37).numpy()
    pts = coords.reshape(3, -1).numpy().T
    d = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    i, j = np.nonzero(np.triu(d <= tol, 1))
    assert sorted(map(tuple, pairs)) == sorted(zip(i.tolist(), j.tolist()))
    # components: lowest index of each connected component
    P = pts.shape[0]
    lab = topology.components(torch.from_numpy(pairs), P).numpy()
    parent = list(range(P))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for a, b in pairs:
        ra, rb = find(a), find(b)
        parent[max(ra, rb)] = min(ra, rb)
    want = np.array([find(a) for a in range(P)])
    comp_min = {}
    for p in range(P):
        comp_min.setdefault(want[p], p)
    assert np.array_equal(lab, np.array([comp_min[want[p]] for p in range(P)]))
    # random jitter below tol keeps the pair set; a shuffled chunking changes nothing
    jit = coords + torch.from_numpy(rng.uniform(-1e-3, 1e-3, coords.shape)) * tol
    p2 = topology.coincident_pairs(jit, tol, chunk=1000).numpy()
    assert len(p2) == len(pairs)


def _sha(t):
    return hashlib.sha256(np.ascontiguousarray(t.cpu().numpy()).tobytes()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_build_space_matches_reference(name):
    from paper_2207_07098_b200.basis import make_basis
    from paper_2207_07098_b200.space import build_space

    want = _gold()[name]["build"]
    arrays, order = CASES[name]
    mesh = topology_cases.as_mesh(arrays, Mesh)
    if want["ok"]:
        sp = build_space(mesh, make_basis(order), device="cuda:0")
        g = sp.gs
        assert (_sha(g.gid), _sha(g.perm), _sha(g.offsets)) == \
            (want["value"]["gid"], want["value"]["perm"], want["value"]["offsets"])
        return
    with pytest.raises(getattr(errors, want["error"])) as ei:
        build_space(mesh, make_basis(order), device="cuda:0")
    msg = want["message"]
    if "degenerate element?" in msg:
        # the local point pair comes from cKDTree's traversal order
        msg = msg.split(": local points")[0]
        assert str(ei.value).startswith(msg)
    else:
        assert str(ei.value) == msg


def test_geometric_fallback_cpu():
    """Duplicated vertex ids on half of a shared face: the topological groups
    differ from the reference's geometric ones, and the builder's cross-check
    falls back to the tol-graph components -- the reference's maps (torch CPU)."""
    from paper_2207_07098_b200.space import build_gather_scatter

    arrays, order = CASES["split_face_half"]
    mesh = topology_cases.as_mesh(arrays, Mesh)
    coords = _coords(arrays, order)
    el = torch.from_numpy(mesh.elements)
    want = _gold()["split_face_half"]["build"]["value"]
    gid_t, _, _ = build_gather_scatter(el, coords, order + 1)            # topology only
    assert _sha(gid_t) != want["gid"]
    gid, perm, off = build_gather_scatter(el, coords, order + 1, tol=topology.gs_tolerance(mesh))
    assert (_sha(gid), _sha(perm), _sha(off)) == (want["gid"], want["perm"], want["offsets"])
    # conforming box: the cross-check agrees and changes nothing
    arrays, order = CASES["valid_box"]
    mesh = topology_cases.as_mesh(arrays, Mesh)
    coords = _coords(arrays, order)
    a = build_gather_scatter(torch.from_numpy(mesh.elements), coords, order + 1)
    b = build_gather_scatter(torch.from_numpy(mesh.elements), coords, order + 1,
                             tol=topology.gs_tolerance(mesh))
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    assert _sha(b[0]) == _gold()["valid_box"]["build"]["value"]["gid"]
