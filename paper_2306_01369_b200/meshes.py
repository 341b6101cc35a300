"""Triangle meshes for baked SDF tools (meshes.py / sdf.py:248-426 of the reference).

Meshes are ``(vertices (V, 3) float64, faces (T, 3) int64)`` with outward,
counter-clockwise winding.  The generators produce the same vertex and face
order as the reference's, so ``mesh_content_hash`` (the GSDF cache key) agrees.
``triangle_table`` packs what the device baker needs per triangle: corners and
the angle-weighted pseudonormals of the face, its three edges and its three
corners (sdf.py:265-297, Baerentzen & Aanaes), computed on the host in the
reference's numpy operation order.
"""

from __future__ import annotations

import hashlib

import numpy as np


class MeshError(ValueError):
    """meshes.py:14 (not watertight, empty, unreadable)."""


def mesh_volume(vertices: np.ndarray, faces: np.ndarray) -> float:
    """Signed volume (divergence theorem), positive for outward winding (meshes.py:18-23)."""
    a, b, c = (vertices[faces[:, k]] for k in range(3))
    return float(np.einsum("ij,ij->i", a, np.cross(b, c)).sum() / 6.0)


def ensure_outward(vertices: np.ndarray, faces: np.ndarray) -> np.ndarray:
    """Reverse every face when the signed volume is negative (meshes.py:26-30)."""
    return faces[:, ::-1].copy() if mesh_volume(vertices, faces) < 0.0 else faces


def open_edge_count(faces: np.ndarray) -> int:
    """Directed edges whose opposite edge is missing (meshes.py:33-37)."""
    directed = set()
    for i, j, k in np.asarray(faces).tolist():
        directed.update(((i, j), (j, k), (k, i)))
    return sum((b, a) not in directed for a, b in directed)


def check_watertight(vertices: np.ndarray, faces: np.ndarray) -> None:
    """meshes.py:40-45."""
    if len(faces) == 0:
        raise MeshError("mesh has no triangles")
    n_open = open_edge_count(faces)
    if n_open:
        raise MeshError(f"mesh is not watertight: {n_open} open edges")


def mesh_content_hash(vertices: np.ndarray, faces: np.ndarray) -> bytes:
    """SHA-256 of the float64 vertex and int64 face bytes (sdf.py:422-426)."""
    h = hashlib.sha256(np.ascontiguousarray(vertices, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(faces, dtype=np.int64).tobytes())
    return h.digest()


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------
def make_box_mesh(half_extents) -> tuple[np.ndarray, np.ndarray]:
    """Axis-aligned box, 8 corners (index 4 ix + 2 iy + iz), 12 triangles (meshes.py:96-117)."""
    h = np.asarray(half_extents, dtype=np.float64)
    sgn = np.array([[sx, sy, sz] for sx in (-1.0, 1.0) for sy in (-1.0, 1.0) for sz in (-1.0, 1.0)])
    v = sgn * h
    # one quad per side (-x, +x, -y, +y, -z, +z), split along its first diagonal
    sides = ((0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3))
    f = np.array([t for a, b, c, d in sides for t in ((a, b, c), (a, c, d))], dtype=np.int64)
    return v, ensure_outward(v, f)


def make_bucket_mesh(half_extents, wall: float) -> tuple[np.ndarray, np.ndarray]:
    """An excavator bucket: the box of ``half_extents`` with a box-shaped
    cavity open at the top (walls and floor ``wall`` thick), as ONE closed
    genus-0 mesh (16 vertices, 28 triangles) so the baked SDF's sign is
    well defined everywhere (sdf.py:357-391).  Vertices: outer bottom 0-3,
    outer top 4-7, cavity top 8-11, cavity bottom 12-15, each ring
    counter-clockwise seen from +z."""
    hx, hy, hz = (float(a) for a in half_extents)
    w = float(wall)
    if not (0.0 < w < min(hx, hy, hz)):
        raise MeshError("bucket wall must be thinner than every half extent")
    ix, iy = hx - w, hy - w
    ring = np.array([[-1.0, -1.0], [1.0, -1.0], [1.0, 1.0], [-1.0, 1.0]])
    v = np.concatenate([
        np.column_stack([ring * [hx, hy], np.full(4, -hz)]),
        np.column_stack([ring * [hx, hy], np.full(4, hz)]),
        np.column_stack([ring * [ix, iy], np.full(4, hz)]),
        np.column_stack([ring * [ix, iy], np.full(4, -hz + w)]),
    ])
    f = [(0, 2, 1), (0, 3, 2), (12, 13, 14), (12, 14, 15)]  # outer bottom (-z), cavity floor (+z)
    for k in range(4):
        n = (k + 1) % 4
        f += [(k, n, 4 + n), (k, 4 + n, 4 + k)]                  # outer side
        f += [(4 + k, 4 + n, 8 + n), (4 + k, 8 + n, 8 + k)]      # rim (+z)
        f += [(12 + k, 8 + n, 12 + n), (12 + k, 8 + k, 8 + n)]  # cavity wall (faces the cavity)
    f = np.array(f, dtype=np.int64)
    check_watertight(v, f)
    return v, ensure_outward(v, f)


def make_icosphere(subdivisions: int = 2, radius: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Icosahedron refined ``subdivisions`` times, midpoints pushed to the sphere (meshes.py:51-93)."""
    g = (1.0 + np.sqrt(5.0)) / 2.0
    v = np.array([(-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0), (0, -1, g), (0, 1, g),
                  (0, -1, -g), (0, 1, -g), (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1)],
                 dtype=np.float64)
    f = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
                  (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
                  (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)
    v = v / np.linalg.norm(v, axis=1, keepdims=True)
    for _ in range(subdivisions):
        pts = [np.asarray(p) for p in v.tolist()]
        mid: dict[tuple[int, int], int] = {}

        def midpoint(i: int, j: int) -> int:
            key = (min(i, j), max(i, j))
            if key not in mid:
                m = pts[i] + pts[j]
                pts.append(m / np.linalg.norm(m))
                mid[key] = len(pts) - 1
            return mid[key]

        out = []
        for a, b, c in f.tolist():
            ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
            out.extend(((a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)))
        v = np.array(pts)
        f = np.array(out, dtype=np.int64)
    return v * radius, f


def make_gear_mesh(n_teeth: int = 8, root_radius: float = 0.6, tip_radius: float = 1.0,
                   thickness: float = 0.4, helix_angle: float = 0.4,
                   n_layers: int = 8) -> tuple[np.ndarray, np.ndarray]:
    """Helical gear: a star profile (per tooth: root, root, tip, tip at 0, .3,
    .45, .75 of the pitch) extruded over ``n_layers`` twisted layers, capped by
    fans from the two axis points (meshes.py:120-171)."""
    pitch = 2.0 * np.pi / n_teeth
    fr = np.array([0.0, 0.3, 0.45, 0.75])
    rr = np.array([root_radius, root_radius, tip_radius, tip_radius])
    ang = (np.arange(n_teeth)[:, None] * pitch + fr[None, :] * pitch).reshape(-1)
    rad = np.tile(rr, n_teeth)
    m = ang.size
    zs = np.linspace(-thickness / 2.0, thickness / 2.0, n_layers + 1)
    rows = []
    for z in zs:
        a = ang + helix_angle * (z / thickness + 0.5)
        rows.extend((x, y, z) for x, y in zip(rad * np.cos(a), rad * np.sin(a)))
    bottom, top = len(rows), len(rows) + 1
    rows.extend(((0.0, 0.0, zs[0]), (0.0, 0.0, zs[-1])))
    tris = []
    for layer in range(n_layers):
        lo, hi = layer * m, (layer + 1) * m
        for k in range(m):
            kn = (k + 1) % m
            tris.extend(((lo + k, lo + kn, hi + kn), (lo + k, hi + kn, hi + k)))
    t0 = n_layers * m
    for k in range(m):
        kn = (k + 1) % m
        tris.extend(((bottom, kn, k), (top, t0 + k, t0 + kn)))
    v = np.array(rows, dtype=np.float64)
    return v, ensure_outward(v, np.array(tris, dtype=np.int64))


# ---------------------------------------------------------------------------
# device triangle table
# ---------------------------------------------------------------------------
TRI_DOUBLES = 30  # a, b, c, face normal, 3 edge pseudonormals, 3 corner pseudonormals


def pseudonormals(vertices: np.ndarray, faces: np.ndarray):
    """(face_n (T,3), edge_pn (T,3,3), corner_pn (T,3,3)) as MeshDistance builds
    them (sdf.py:257-297): unit face normals; vertex normals weighted by the
    corner angle, accumulated face by face in corner order; edge normals = the
    normalised sum of the two adjacent face normals (edge e of a face joins
    corners e and e + 1)."""
    V = np.asarray(vertices, dtype=np.float64)
    F = np.asarray(faces, dtype=np.int64)
    a, b, c = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    n = np.cross(b - a, c - a)
    face_n = n / np.linalg.norm(n, axis=1, keepdims=True)
    vert = np.zeros_like(V)
    for k in range(3):
        i0 = F[:, k]
        e1 = V[F[:, (k + 1) % 3]] - V[i0]
        e2 = V[F[:, (k + 2) % 3]] - V[i0]
        cosang = np.einsum("ij,ij->i", e1, e2) / (np.linalg.norm(e1, axis=1) * np.linalg.norm(e2, axis=1))
        np.add.at(vert, i0, face_n * np.arccos(np.clip(cosang, -1.0, 1.0))[:, None])
    vert = vert / np.maximum(np.linalg.norm(vert, axis=1, keepdims=True), 1e-300)
    sums: dict[tuple[int, int], object] = {}
    edges = [((i, j), (j, k), (k, i)) for i, j, k in F.tolist()]
    for t, es in enumerate(edges):
        for u, w in es:
            key = (min(u, w), max(u, w))
            sums[key] = sums.get(key, 0.0) + face_n[t]
    edge_pn = np.zeros((len(F), 3, 3))
    for t, es in enumerate(edges):
        for e, (u, w) in enumerate(es):
            s = sums[(min(u, w), max(u, w))]
            edge_pn[t, e] = s / max(np.linalg.norm(s), 1e-300)
    return face_n, edge_pn, vert[F]


def triangle_table(vertices: np.ndarray, faces: np.ndarray) -> np.ndarray:
    """(T, 30) float64 rows for gg_bake_mesh_sdf (see include/granusim_b200.h)."""
    V = np.asarray(vertices, dtype=np.float64)
    F = np.asarray(faces, dtype=np.int64)
    face_n, edge_pn, corner_pn = pseudonormals(V, F)
    tab = np.empty((len(F), TRI_DOUBLES))
    tab[:, 0:3], tab[:, 3:6], tab[:, 6:9] = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    tab[:, 9:12] = face_n
    tab[:, 12:21] = edge_pn.reshape(-1, 9)
    tab[:, 21:30] = corner_pn.reshape(-1, 9)
    return np.ascontiguousarray(tab)
