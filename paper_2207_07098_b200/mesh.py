"""Hexahedral mesh container and the structured box generator (setup only).

Field-compatible with the reference ``semflow.mesh.Mesh`` (mesh.py:38-93), so a
mesh produced by the reference generators (box, cylinder-in-box, file reader)
can be handed to :func:`paper_2207_07098_b200.space.build_space` unchanged.
``gen_box_mesh`` restates mesh.py:154-219: vertices from ``np.linspace`` laid
out x-fastest, element corners in the r-fastest corner order, elements numbered
x fastest then y then z, boundary facets tagged (xlo, xhi, ylo, yhi, zlo, zhi).
"""

from dataclasses import dataclass, field

import numpy as np

#: corner indices of each local face: 0 r=-1, 1 r=+1, 2 s=-1, 3 s=+1, 4 t=-1, 5 t=+1
FACE_CORNERS = ((0, 2, 4, 6), (1, 3, 5, 7), (0, 1, 4, 5), (2, 3, 6, 7), (0, 1, 2, 3), (4, 5, 6, 7))


@dataclass
class Mesh:
    vertices: np.ndarray
    elements: np.ndarray
    facet_elem: np.ndarray
    facet_face: np.ndarray
    facet_tag: np.ndarray
    tag_names: tuple
    curved_elem: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    curved_coords: np.ndarray = field(default_factory=lambda: np.zeros((0, 2, 2, 2, 3)))
    geom_order: int | None = None

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def n_elements(self):
        return self.elements.shape[0]

    @property
    def n_facets(self):
        return self.facet_elem.shape[0]


def gen_box_mesh(extent, counts, tags=None):
    """Cartesian box of affine hexahedra (reference mesh.py:154)."""
    tags = tuple(tags) if tags is not None else ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")
    if len(tags) != 6:
        raise ValueError("tags must name the 6 box sides")
    nx, ny, nz = (int(c) for c in counts)
    if min(nx, ny, nz) < 1:
        raise ValueError(f"element counts must be >= 1, got {counts}")
    ext = list(extent)
    if len(ext) == 6:
        ext = [(ext[0], ext[1]), (ext[2], ext[3]), (ext[4], ext[5])]
    lo = [float(a) for a, _ in ext]
    hi = [float(b) for _, b in ext]
    if any(h <= l for l, h in zip(lo, hi)):
        raise ValueError(f"degenerate extent {extent}")
    axes = [np.linspace(lo[d], hi[d], c + 1) for d, c in enumerate((nx, ny, nz))]
    # vertex id = i + (nx+1) (j + (ny+1) k): x fastest
    zz, yy, xx = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    vertices = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1).astype(np.float64)

    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    corner = np.arange(8)
    ci = i[:, None] + (corner & 1)[None, :]
    cj = j[:, None] + ((corner >> 1) & 1)[None, :]
    ck = k[:, None] + ((corner >> 2) & 1)[None, :]
    elements = (ci + (nx + 1) * (cj + (ny + 1) * ck)).astype(np.int64)

    names = []
    for t in tags:
        if t not in names:
            names.append(t)
    tag_idx = [names.index(t) for t in tags]
    eid = np.arange(nx * ny * nz, dtype=np.int64)
    on_face = (i == 0, i == nx - 1, j == 0, j == ny - 1, k == 0, k == nz - 1)
    # reference order: per element (in element order) faces 0..5
    fe = np.concatenate([eid[m] for m in on_face])
    ff = np.concatenate([np.full(int(m.sum()), f, dtype=np.int64) for f, m in enumerate(on_face)])
    order = np.lexsort((ff, fe))
    fe, ff = fe[order], ff[order]
    ft = np.asarray(tag_idx, dtype=np.int64)[ff]
    return Mesh(vertices=vertices, elements=elements, facet_elem=fe, facet_face=ff,
                facet_tag=ft, tag_names=tuple(names))
