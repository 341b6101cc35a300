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


@pytest.mark.gpu
def test_splat_equals_brute_force():
    """The splatting renderer (mode 1: each particle tests only the pixels its
    sphere can cover) gives bitwise the image of the default (mode 0: every
    pixel tests every particle, the reference's algorithm)."""
    from paper_2306_01369_b200 import _native as N

    g = golden()
    try:
        for k in range(int(g["n_env_cases"])):
            sc = env_scene(g, k)
            imgs = {}
            for mode in (0, 1):
                N.lib().gg_set_render_mode(mode)
                imgs[mode] = (render_depth(sc, camera(g, f"c{k}_ego")),
                              render_depth(sc, camera(g, f"c{k}_sky")))
            assert np.array_equal(imgs[0][0], imgs[1][0])
            assert np.array_equal(imgs[0][1], imgs[1][1])
        # a dense random cloud seen from inside and around it
        rng = np.random.default_rng(1)
        x = rng.uniform(-1.0, 1.0, size=(3000, 3))
        sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)), bodies=[],
                      params=gg.MaterialParams(radius=0.03))
        cams = [DepthCamera(kind="perspective", pose=gg.make_pose(gg.so3_exp(np.array([0.3, -0.2, 0.1])),
                                                                 np.array([0.1, 0.0, -0.2])),
                            width=64, height=48, fov=1.7, far=5.0),
                DepthCamera(kind="orthographic", pose=gg.make_pose(np.eye(3), np.array([0.0, 0.0, -3.0])),
                            width=50, height=40, extent=(2.5, 2.0), far=9.0)]
        for cam in cams:
            N.lib().gg_set_render_mode(0)
            a = render_depth(sc, cam)
            N.lib().gg_set_render_mode(1)
            b = render_depth(sc, cam)
            assert np.array_equal(a, b)
            assert (a < cam.far).mean() > 0.3
    finally:
        N.lib().gg_set_render_mode(0)
