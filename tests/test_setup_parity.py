"""Product setup code vs the reference (CPU): basis, box mesh and the topological
gather-scatter numbering (run on torch CPU tensors; the same code runs on the
GPU in build_space)."""

import hashlib

import numpy as np
import pytest
import torch

from conftest import mesh_from_golden
from paper_2207_07098_b200.basis import make_basis
from paper_2207_07098_b200.mesh import gen_box_mesh
from paper_2207_07098_b200.space import build_gather_scatter, pack_bits


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("order", range(1, 11))
def test_basis_bitwise(golden_basis, order):
    b = make_basis(order)
    assert np.array_equal(b.points, golden_basis[f"p{order}"])
    assert np.array_equal(b.weights, golden_basis[f"w{order}"])
    assert np.array_equal(b.dmat, golden_basis[f"d{order}"])


@pytest.mark.parametrize("key,extent,counts", [
    ("tgv4", (0.0, 2 * np.pi, 0.0, 2 * np.pi, 0.0, 2 * np.pi), (4, 4, 4)),
    ("box211", (0.0, 2.0, 0.0, 1.0, 0.0, 1.0), (2, 1, 1)),
    ("cube222", (0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (2, 2, 2)),
])
def test_box_mesh_matches_reference(golden_spaces, key, extent, counts):
    g = golden_spaces
    m = gen_box_mesh(extent, counts)
    assert np.array_equal(m.vertices, g[f"{key}_vertices"])
    assert np.array_equal(m.elements, g[f"{key}_elements"])
    assert np.array_equal(m.facet_elem, g[f"{key}_facet_elem"])
    assert np.array_equal(m.facet_face, g[f"{key}_facet_face"])
    assert np.array_equal(m.facet_tag, g[f"{key}_facet_tag"])


@pytest.mark.parametrize("key", ["box211", "cube222", "pbox322", "pbox543", "tgv4", "rotor"])
def test_topological_numbering_is_bit_exact(oracle, golden_spaces, key):
    """gid / perm / offsets from topology + exact coordinates == reference KD-tree build."""
    g = golden_spaces
    m = mesh_from_golden(g, key)
    order = int(g[f"{key}_order"])
    sp = oracle.build_space(m, oracle.make_basis(order))   # exact reference coordinates
    assert sha(sp.coords) == str(g[f"{key}_sha_coords"])
    gid, perm, offsets = build_gather_scatter(torch.from_numpy(m.elements), torch.from_numpy(sp.coords),
                                              order + 1)
    assert sha(gid.numpy()) == str(g[f"{key}_sha_gid"])
    assert sha(perm.numpy()) == str(g[f"{key}_sha_perm"])
    assert sha(offsets.numpy()) == str(g[f"{key}_sha_offsets"])


def test_topological_numbering_permuted_vertices(oracle):
    """Vertex ids in arbitrary order (unstructured-style numbering) still group correctly."""
    m = oracle.gen_box_mesh((0.0, 1.0, 0.0, 2.0, 0.0, 1.0), (3, 2, 2))
    rng = np.random.default_rng(4)
    p = rng.permutation(m.vertices.shape[0])
    inv = np.empty_like(p)
    inv[p] = np.arange(p.size)
    m2 = oracle.Mesh(m.vertices[p], inv[m.elements], m.facet_elem, m.facet_face, m.facet_tag, m.tag_names,
                     m.curved_elem, m.curved_coords, None)
    sp = oracle.build_space(m2, oracle.make_basis(4))
    gid, perm, off = build_gather_scatter(torch.from_numpy(m2.elements), torch.from_numpy(sp.coords), 5)
    assert np.array_equal(gid.numpy(), sp.gs.gid)
    assert np.array_equal(perm.numpy(), sp.gs.perm)
    assert np.array_equal(off.numpy(), sp.gs.offsets)


def test_pack_bits_layout():
    flags = torch.zeros(2, 125, dtype=torch.bool)
    flags[0, 0] = True
    flags[0, 33] = True
    flags[1, 124] = True
    w = pack_bits(flags)
    assert w.shape == (2, 4)
    assert int(w[0, 0]) == 1 and int(w[0, 1]) == 2
    assert int(w[1, 3]) == (1 << (124 - 96))
    full = pack_bits(torch.ones(1, 64, dtype=torch.bool))
    assert int(full[0, 0]) == -1 and int(full[0, 1]) == -1
