"""Depth rendering on the device (render.py) against
images made by the real reference renderer (tests/golden/render.npz, from
make_golden_render.py).

Tolerance: depth is float64 on both sides, stored float32.  Sphere tracing
stops within eps = 1e-4 of a surface and the two implementations round their
ray arithmetic differently, so a traced depth may differ by ~eps; a pixel on
a silhouette may flip between hit and miss.  Bar: |d - d_ref| <= 2e-4 m on
>= 99% of the pixels, and no more than 1% of pixels beyond it.
"""

import numpy as np
import pytest

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.render import CAMERA_DTYPE, DepthCamera, render_batch, render_depth
from helpers import GOLDEN


def golden():
    with np.load(GOLDEN / "render.npz") as z:
        return {k: z[k] for k in z.files}


def camera(g, p):
    kind = "perspective" if int(g[p + "_kind"]) == 0 else "orthographic"
    w, h = (int(v) for v in g[p + "_wh"])
    return DepthCamera(kind=kind, pose=g[p + "_pose"], width=w, height=h, fov=float(g[p + "_fov"]),
                       extent=tuple(g[p + "_extent"]), far=float(g[p + "_far"]))


def close(img, ref, tol=2e-4, frac=0.01):
    assert img.shape == ref.shape and img.dtype == np.float32
    bad = np.abs(img.astype(np.float64) - ref.astype(np.float64)) > tol
    assert bad.mean() <= frac, (bad.mean(), np.abs(img - ref).max())


def test_camera_validation_and_layout():
    with pytest.raises(ValueError):
        DepthCamera(width=0)
    with pytest.raises(ValueError):
        DepthCamera(far=0.0)
    with pytest.raises(ValueError):
        DepthCamera(kind="fisheye")
    assert CAMERA_DTYPE.itemsize == 4 * 4 + 16 * 8 + 8 + 16 + 8


def env_scene(g, k):
    x = g[f"c{k}_x"]
    r = float(g[f"c{k}_radius"])
    blade = gg.RigidBody(gg.Box(g[f"c{k}_blade_half"]), driver=gg.StaticDriver(g[f"c{k}_blade_pose"]),
                         name="blade")
    blade.update(0.0)
    sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="ground"), blade],
                  params=gg.MaterialParams(radius=r))
    for b in sc.bodies:
        b.update(0.0)
    return sc


@pytest.mark.gpu
def test_env_cameras_match_reference():
    g = golden()
    for k in range(int(g["n_env_cases"])):
        sc = env_scene(g, k)
        close(render_depth(sc, camera(g, f"c{k}_ego")), g[f"c{k}_ego_depth"])
        close(render_depth(sc, camera(g, f"c{k}_sky")), g[f"c{k}_sky_depth"])


@pytest.mark.gpu
def test_primitives_and_grid_match_reference():
    g = golden()
    x = g["p_x"]
    grid = gg.SdfGrid(g["p_grid_origin"], g["p_grid_spacing"], np.array(g["p_grid_values"].shape),
                      g["p_grid_values"])
    bodies = [gg.RigidBody(gg.Sphere(0.3), driver=gg.StaticDriver(g["p_sphere_pose"])),
              gg.RigidBody(gg.Cylinder(0.25, 0.4), driver=gg.StaticDriver(g["p_cyl_pose"])),
              gg.RigidBody(grid, driver=gg.StaticDriver(g["p_grid_pose"]))]
    for b in bodies:
        b.update(0.0)
    sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)), bodies=bodies,
                  params=gg.MaterialParams(radius=float(g["p_radius"])))
    close(render_depth(sc, camera(g, "p_persp")), g["p_persp_depth"])
    close(render_depth(sc, camera(g, "p_ortho")), g["p_ortho_depth"])


@pytest.mark.gpu
def test_batch_render_equals_single_scene_render():
    from paper_2306_01369_b200.batch import SceneBatch

    g = golden()
    scenes = [env_scene(g, k) for k in range(int(g["n_env_cases"]))]
    for sc in scenes:  # the batch needs equal particle counts
        sc.particles = gg.ParticleSet(sc.particles.positions[:300], sc.particles.velocities[:300])
    singles = [env_scene(g, k) for k in range(int(g["n_env_cases"]))]
    for sc in singles:
        sc.particles = gg.ParticleSet(sc.particles.positions[:300], sc.particles.velocities[:300])
    batch = SceneBatch(scenes)
    ego = [camera(g, f"c{k}_ego") for k in range(len(scenes))]
    sky = camera(g, "c0_sky")
    E_ego, E_sky = render_batch(batch, [ego[0], sky], [np.stack([c.pose for c in ego]), None])
    for k, sc in enumerate(singles):
        assert np.array_equal(E_ego[k], render_depth(sc, ego[k]))
        assert np.array_equal(E_sky[k], render_depth(sc, sky))
    batch.close()
