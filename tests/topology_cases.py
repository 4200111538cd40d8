"""Malformed and unusual meshes for the topology checks (reference mesh.py:95-147,
space.py:265-314).  Each recipe returns plain arrays; tests/golden/
make_topology_golden.py runs the REFERENCE's Mesh.validate / build_space on them
and records the outcome (exception class + message, or sha256 of the maps).
"""

import numpy as np

TAGS = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")


def box(counts, extent=(0.0, 1.0, 0.0, 1.0, 0.0, 1.0)):
    """Same arrays as gen_box_mesh (bit-identical to the reference generator)."""
    from paper_2207_07098_b200.mesh import gen_box_mesh

    m = gen_box_mesh(extent, counts)
    return dict(vertices=m.vertices.copy(), elements=m.elements.copy(), facet_elem=m.facet_elem.copy(),
                facet_face=m.facet_face.copy(), facet_tag=m.facet_tag.copy(), tag_names=TAGS)


def _hanging():
    """One unit element next to four half-size elements on its xhi face (2:1,
    non-conforming): the big face and the four small faces are all 'exterior'
    and untagged."""
    big = box((1, 1, 1), (0.0, 1.0, 0.0, 1.0, 0.0, 1.0))
    small = box((1, 2, 2), (1.0, 1.5, 0.0, 1.0, 0.0, 1.0))
    nv = big["vertices"].shape[0]
    verts = np.concatenate([big["vertices"], small["vertices"]])
    elems = np.concatenate([big["elements"], small["elements"] + nv])
    fe = np.concatenate([big["facet_elem"], small["facet_elem"] + 1])
    ff = np.concatenate([big["facet_face"], small["facet_face"]])
    ft = np.concatenate([big["facet_tag"], small["facet_tag"]])
    keep = ~(((fe == 0) & (ff == 1)) | ((fe >= 1) & (ff == 0)))
    return dict(vertices=verts, elements=elems, facet_elem=fe[keep], facet_face=ff[keep],
                facet_tag=ft[keep], tag_names=TAGS)


def _split_face(all_four):
    """2x1x1 box; element 1 uses duplicated vertex ids (same coordinates) for the
    shared face -- all four corners, or only the two at y=1 -- and both halves of
    the cut are tagged, so Mesh.validate passes."""
    m = box((2, 1, 1))
    v = m["vertices"]
    el = m["elements"].copy()
    shared = [int(c) for c in el[1, [0, 2, 4, 6]]]          # element 1's r=-1 face
    if not all_four:
        shared = [c for c in shared if v[c, 1] == 1.0]
    new_ids = {}
    verts = [v]
    for c in shared:
        new_ids[c] = v.shape[0] + len(new_ids)
        verts.append(v[c][None])
    for k in range(8):
        if int(el[1, k]) in new_ids:
            el[1, k] = new_ids[int(el[1, k])]
    fe = np.concatenate([m["facet_elem"], [0, 1]])
    ff = np.concatenate([m["facet_face"], [1, 0]])
    ft = np.concatenate([m["facet_tag"], [1, 0]])
    return dict(vertices=np.concatenate(verts), elements=el, facet_elem=fe, facet_face=ff,
                facet_tag=ft, tag_names=TAGS)


def _thin():
    """A 2x1x1 box whose first element is 1e-11 thick in x (positive Jacobian,
    GLL points of that element closer than the gather-scatter tolerance)."""
    m = box((2, 1, 1))
    v = m["vertices"].copy()
    v[v[:, 0] == 0.0, 0] = 0.5 - 1e-11
    return dict(m, vertices=v)


def _collapsed():
    """Element 0 has one edge collapsed to a point (zero Jacobian there)."""
    m = box((2, 1, 1))
    v = m["vertices"].copy()
    el = m["elements"]
    v[el[0, 1]] = v[el[0, 0]]
    return dict(m, vertices=v)


def cases():
    """name -> (arrays, order)."""
    out = {}
    out["valid_box"] = (box((2, 2, 2)), 3)
    m = box((2, 1, 1))
    out["nonconforming_3"] = (dict(m, elements=np.concatenate([m["elements"], m["elements"][:1]])), 3)
    out["hanging_2to1"] = (_hanging(), 3)
    out["untagged_exterior"] = (dict(m, facet_elem=m["facet_elem"][1:], facet_face=m["facet_face"][1:],
                                     facet_tag=m["facet_tag"][1:]), 3)
    out["tagged_twice"] = (dict(m, facet_elem=np.concatenate([m["facet_elem"], m["facet_elem"][3:4]]),
                                facet_face=np.concatenate([m["facet_face"], m["facet_face"][3:4]]),
                                facet_tag=np.concatenate([m["facet_tag"], m["facet_tag"][3:4]])), 3)
    out["interior_tagged"] = (dict(m, facet_elem=np.concatenate([m["facet_elem"], [0]]),
                                   facet_face=np.concatenate([m["facet_face"], [1]]),
                                   facet_tag=np.concatenate([m["facet_tag"], [0]])), 3)
    el = m["elements"].copy()
    el[1, 3] = m["vertices"].shape[0]
    out["vertex_out_of_range"] = (dict(m, elements=el), 3)
    out["facet_elem_out_of_range"] = (dict(m, facet_elem=np.where(np.arange(m["facet_elem"].size) == 2, 7,
                                                                   m["facet_elem"])), 3)
    out["facet_face_out_of_range"] = (dict(m, facet_face=np.where(np.arange(m["facet_face"].size) == 2, 6,
                                                                   m["facet_face"])), 3)
    out["facet_tag_out_of_range"] = (dict(m, facet_tag=np.where(np.arange(m["facet_tag"].size) == 2, 6,
                                                                 m["facet_tag"])), 3)
    out["split_face_all"] = (_split_face(True), 3)
    out["split_face_half"] = (_split_face(False), 3)
    out["thin_element"] = (_thin(), 3)
    out["collapsed_edge"] = (_collapsed(), 3)
    return out


def as_mesh(arrays, mesh_cls):
    a = arrays
    return mesh_cls(vertices=np.asarray(a["vertices"], dtype=np.float64),
                    elements=np.asarray(a["elements"], dtype=np.int64),
                    facet_elem=np.asarray(a["facet_elem"], dtype=np.int64),
                    facet_face=np.asarray(a["facet_face"], dtype=np.int64),
                    facet_tag=np.asarray(a["facet_tag"], dtype=np.int64),
                    tag_names=tuple(a["tag_names"]))
