"""Mesh SDF baking: host mesh generators and
pseudonormals vs the reference (CPU), device baker vs the reference's
bake_mesh_sdf / MeshDistance.signed_distance (GPU).  Fixtures:
tests/golden/bake.npz (tests/golden/make_golden_bake.py, the real reference).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2306_01369_b200 import meshes as M

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "bake.npz")
CASES = {
    "box": (lambda: M.make_box_mesh([0.15, 0.1, 0.04]), 0.01),
    "gear": (lambda: M.make_gear_mesh(n_teeth=6, root_radius=0.06, tip_radius=0.1, thickness=0.04,
                                      helix_angle=0.4, n_layers=4), 0.008),
    "ico": (lambda: M.make_icosphere(2, radius=0.1), 0.01),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_generators_match_reference(name):
    v, f = CASES[name][0]()
    np.testing.assert_array_equal(v, GOLD[f"{name}_vertices"])
    np.testing.assert_array_equal(f, GOLD[f"{name}_faces"])
    assert M.mesh_content_hash(v, f) == GOLD[f"{name}_hash"].tobytes()
    M.check_watertight(v, f)


@pytest.mark.parametrize("name", sorted(CASES))
def test_pseudonormals_match_reference(name):
    v, f = CASES[name][0]()
    fn, en, cn = M.pseudonormals(v, f)
    np.testing.assert_array_equal(fn, GOLD[f"{name}_face_n"])
    np.testing.assert_array_equal(en, GOLD[f"{name}_edge_pn"])
    np.testing.assert_array_equal(cn, GOLD[f"{name}_corner_pn"])
    tab = M.triangle_table(v, f)
    assert tab.shape == (len(f), M.TRI_DOUBLES) and tab.flags.c_contiguous
    np.testing.assert_array_equal(tab[:, 3:6], v[f[:, 1]])
    np.testing.assert_array_equal(tab[:, 12:21].reshape(-1, 3, 3), en)


def test_open_mesh_rejected():
    v, f = M.make_box_mesh([1.0, 1.0, 1.0])
    with pytest.raises(M.MeshError, match="not watertight"):
        M.check_watertight(v, f[:-1])
    with pytest.raises(M.MeshError, match="no triangles"):
        M.check_watertight(v, f[:0])
    assert M.mesh_volume(v, f) == pytest.approx(8.0)
    assert M.mesh_volume(v, f[:, ::-1]) == pytest.approx(-8.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_baked_grid_bit_exact(name):
    from paper_2306_01369_b200.sdf import bake_mesh_sdf

    (v, f), h = CASES[name][0](), CASES[name][1]
    g = bake_mesh_sdf(v, f, spacing=h)
    np.testing.assert_array_equal(g.origin, GOLD[f"{name}_origin"])
    np.testing.assert_array_equal(g.spacing, GOLD[f"{name}_spacing"])
    np.testing.assert_array_equal(g.dims, GOLD[f"{name}_dims"])
    ref = GOLD[f"{name}_values"]
    bad = np.flatnonzero(g.values.reshape(-1) != ref.reshape(-1))
    assert bad.size == 0, (bad.size, np.abs(g.values.reshape(-1) - ref.reshape(-1)).max())
    assert g.mesh_hash == GOLD[f"{name}_hash"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_signed_distance_points_bit_exact(name):
    from paper_2306_01369_b200.sdf import MeshDistance

    v, f = CASES[name][0]()
    md = MeshDistance(v, f)
    sd = md.signed_distance(GOLD[f"{name}_points"])
    np.testing.assert_array_equal(sd, GOLD[f"{name}_sd"])
    assert md.signed_distance(GOLD[f"{name}_points"][0]) == GOLD[f"{name}_sd"][0]


@pytest.mark.gpu
def test_baked_tool_in_a_step():
    """A baked box mesh tool behaves like the analytic Box it samples."""
    import paper_2306_01369_b200 as gg
    from paper_2306_01369_b200.sdf import bake_mesh_sdf

    v, f = M.make_box_mesh([0.15, 0.1, 0.04])
    grid = bake_mesh_sdf(v, f, spacing=0.01)
    pos = gg.lattice_bed(2000).astype(np.float32).astype(np.float64)
    top = float(pos[:, 2].max())
    cx, cy = float(np.median(pos[:, 0])), float(np.median(pos[:, 1]))
    reps = {}
    for nm, geom in (("grid", grid), ("box", gg.Box([0.15, 0.1, 0.04]))):
        sc = gg.Scene(particles=gg.ParticleSet(pos.copy(), np.zeros_like(pos)),
                      bodies=[gg.RigidBody(gg.HalfSpace(), name="floor"),
                              gg.RigidBody(geom, gg.StaticDriver(gg.make_pose(np.eye(3), [cx, cy, top])),
                                           name="tool")],
                      params=gg.MaterialParams(timestep=5e-4))
        _, reps[nm] = gg.step(sc)
    assert reps["grid"].n_body_contacts > 0
    assert abs(reps["grid"].n_body_contacts - reps["box"].n_body_contacts) <= 0.02 * reps["box"].n_body_contacts + 2
