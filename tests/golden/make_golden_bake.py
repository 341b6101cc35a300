"""Golden mesh SDFs from the REAL reference baker (meshes.py, sdf.py:248-419).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \\
        python tests/golden/make_golden_bake.py

Three meshes: the config-4 scoop box (make_box_mesh([0.15, 0.1, 0.04])), a
small helical gear and a 2-level icosphere.  For each: vertices, faces, the
pseudonormals MeshDistance builds, bake_mesh_sdf's grid (origin, spacing,
dims, float64 values, mesh hash) and signed distances at seeded points
(uniform in the padded box, plus points on vertices, edge midpoints and face
centroids).  Saved as tests/golden/bake.npz.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

import granusim
from granusim import meshes as rm
from granusim import sdf as rsdf

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__

cases = {
    "box": (rm.make_box_mesh([0.15, 0.1, 0.04]), 0.01),
    "gear": (rm.make_gear_mesh(n_teeth=6, root_radius=0.06, tip_radius=0.1, thickness=0.04,
                               helix_angle=0.4, n_layers=4), 0.008),
    "ico": (rm.make_icosphere(2, radius=0.1), 0.01),
}
rng = np.random.default_rng(7)
z = {}
for name, ((v, f), h) in cases.items():
    md = rsdf.MeshDistance(v, f)
    g = rsdf.bake_mesh_sdf(v, f, spacing=h)
    lo, hi = v.min(0) - 0.03, v.max(0) + 0.03
    pts = [rng.uniform(lo, hi, size=(400, 3)), v,
           0.5 * (v[f[:, 0]] + v[f[:, 1]]), (v[f[:, 0]] + v[f[:, 1]] + v[f[:, 2]]) / 3.0]
    pts = np.concatenate(pts)
    z[f"{name}_vertices"], z[f"{name}_faces"] = v, f
    z[f"{name}_face_n"], z[f"{name}_edge_pn"], z[f"{name}_corner_pn"] = md.face_n, md.edge_pn, md.corner_pn
    z[f"{name}_origin"], z[f"{name}_spacing"], z[f"{name}_dims"] = g.origin, g.spacing, np.asarray(g.dims)
    z[f"{name}_values"] = g.values
    z[f"{name}_hash"] = np.frombuffer(g.mesh_hash, dtype=np.uint8)
    z[f"{name}_points"], z[f"{name}_sd"] = pts, md.signed_distance(pts)
    print(name, len(f), "triangles", tuple(g.dims), "knots")
np.savez_compressed(OUT / "bake.npz", **z)
