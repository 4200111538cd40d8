"""Cylinder-in-box generator vs the reference's (mesh.py:231-438): bit-identical
vertices (first-appearance numbering), connectivity, facets and curved records."""
import hashlib
import os

import numpy as np
import pytest

from conftest import mesh_from_golden
from paper_2207_07098_b200.mesh import gen_cylinder_box_mesh

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cylinder.npz")
CYL_MESHES = {
    "cyl_analogue": dict(diameter=1.0, xlim=(-50.0, 120.0), zlim=(-25.0, 25.0), height=10.0, n_azimuthal=32,
                         n_radial=8, n_axial=4, n_upstream=16, n_downstream=32, n_front=16, n_back=16,
                         geom_order=7),
    "cyl_auto": dict(diameter=2.0, xlim=(-6.0, 9.0), zlim=(-5.0, 7.0), height=3.0, n_azimuthal=12, n_radial=3,
                     n_axial=2, collar=1.7, geom_order=4),
}
FIELDS = ("vertices", "elements", "facet_elem", "facet_face", "facet_tag", "curved_elem", "curved_coords")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden_cyl():
    return np.load(GOLDEN)


@pytest.mark.parametrize("key", sorted(CYL_MESHES))
def test_cylinder_mesh_bitwise(golden_cyl, key):
    m = gen_cylinder_box_mesh(**CYL_MESHES[key])
    for f in FIELDS:
        a = np.asarray(getattr(m, f))
        assert tuple(a.shape) == tuple(golden_cyl[f"{key}_shape_{f}"]), f
        assert sha(a) == str(golden_cyl[f"{key}_sha_{f}"]), f
    assert m.tag_names == ("inflow", "outflow", "bottom", "top", "span", "cylinder")


def test_mini_rotor_mesh_bitwise(golden_spaces):
    ref = mesh_from_golden(golden_spaces, "rotor")
    m = gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                              n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5)
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(m, f)), np.asarray(getattr(ref, f))), f


def test_config5_element_count_formula():
    """2 023 424 elements (documented formula, mesh.py:259-263)."""
    a, nr, nax, up, down, fr, bk = 32, 32, 52, 64, 128, 64, 64
    E = nax * (4 * a * nr + a * (up + down + fr + bk) + (up + down) * (fr + bk))
    assert E == 2023424
    m = gen_cylinder_box_mesh(1.0, (-50.0, 120.0), (-25.0, 25.0), 10.0, n_azimuthal=16, n_radial=2, n_axial=3,
                              n_upstream=3, n_downstream=5, n_front=2, n_back=4, geom_order=2)
    a, nr, nax, up, down, fr, bk = 4, 2, 3, 3, 5, 2, 4
    assert m.elements.shape[0] == nax * (4 * a * nr + a * (up + down + fr + bk) + (up + down) * (fr + bk))


def test_cylinder_validation():
    with pytest.raises(ValueError, match="multiple of 4"):
        gen_cylinder_box_mesh(1.0, (-4, 6), (-4, 4), 2.0, n_azimuthal=6)
    with pytest.raises(ValueError, match="collar"):
        gen_cylinder_box_mesh(1.0, (-4, 6), (-4, 4), 2.0, collar=0.4)
    with pytest.raises(ValueError, match="strictly contain"):
        gen_cylinder_box_mesh(1.0, (-0.5, 6), (-4, 4), 2.0)


def test_mesh_file_roundtrip_and_reference_file(tmp_path):
    """read_mesh / write_mesh (mesh.py:444-560): the reference-written file reads to
    our generator's mesh and rewrites byte for byte; damage is reported by section."""
    from paper_2207_07098_b200.errors import MeshFormatError
    from paper_2207_07098_b200.mesh import gen_box_mesh, read_mesh, write_mesh

    ref_path = os.path.join(os.path.dirname(__file__), "golden", "mini_rotor.mesh")
    m = read_mesh(ref_path)
    g = gen_cylinder_box_mesh(1.0, (-4.0, 6.0), (-4.0, 4.0), 2.0, n_azimuthal=8, n_radial=2, n_axial=2,
                              n_upstream=4, n_downstream=5, n_front=3, n_back=3, geom_order=5)
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(m, f)), np.asarray(getattr(g, f))), f
    assert m.tag_names == g.tag_names and m.geom_order == 5
    out = tmp_path / "again.mesh"
    write_mesh(g, str(out))
    blob = open(ref_path, "rb").read()
    assert out.read_bytes() == blob
    box = gen_box_mesh((0, 1, 0, 1, 0, 1), (2, 3, 1))
    write_mesh(box, str(tmp_path / "box.mesh"))
    b2 = read_mesh(str(tmp_path / "box.mesh"))
    assert b2.geom_order is None and np.array_equal(b2.elements, box.elements)
    bad = tmp_path / "bad.mesh"
    bad.write_bytes(blob[:-16])
    with pytest.raises(MeshFormatError) as exc:
        read_mesh(str(bad))
    assert exc.value.section == "curved_coords"
    bad.write_bytes(b"NOTAMESH" + blob[8:])
    with pytest.raises(MeshFormatError, match="magic"):
        read_mesh(str(bad))
    bad.write_bytes(blob + b"\0")
    with pytest.raises(MeshFormatError, match="trailing") as exc:
        read_mesh(str(bad))
    assert exc.value.section == "end"
