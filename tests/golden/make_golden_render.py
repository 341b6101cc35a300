"""Golden depth images from the REAL reference renderer (render.py).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_render.py

BulldozerEnv(n_particles=400) seeds 0 and 1: after reset and after one control
step with a fixed action, the ego and sky depth images the env observes
(envs.py:180-205) plus everything needed to re-render them: particle
positions (float32-representable), body poses, camera poses.  Also a scene
with a Sphere, a Cylinder and a baked SdfGrid body seen by both camera kinds.
Saved as tests/golden/render.npz.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

import granusim
from granusim import sdf as rsdf
from granusim.envs import BulldozerEnv, BulldozerEnvConfig
from granusim.kinematics import make_pose, so3_exp
from granusim.render import DepthCamera, render_depth
from granusim.scene import MaterialParams, ParticleSet, RigidBody, Scene

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731


def cam_rec(prefix, cam, pose, out):
    out[prefix + "_kind"] = np.array(0 if cam.kind == "perspective" else 1)
    out[prefix + "_wh"] = np.array([cam.width, cam.height])
    out[prefix + "_pose"] = np.asarray(pose, float)
    out[prefix + "_fov"] = np.array(cam.fov)
    out[prefix + "_extent"] = np.array(cam.extent, float)
    out[prefix + "_far"] = np.array(cam.far)


def main():
    out = {}
    cfg = BulldozerEnvConfig(n_particles=400)
    k = 0
    for seed in (0, 1):
        env = BulldozerEnv(cfg)
        env.reset(seed)
        sc = env.scene
        sc.particles.positions[:] = f32(sc.particles.positions)
        for stage in range(2):
            if stage == 1:
                env.step(np.array([0.8, 0.3]))
                sc.particles.positions[:] = f32(sc.particles.positions)
            obs_pose = env.driver.pose_at(sc.t)
            vehicle = obs_pose.copy()
            vehicle[:3, 3] -= obs_pose[:3, :3] @ env.driver.base_pose[:3, 3]
            ego_cam = DepthCamera(kind="perspective", pose=vehicle @ env.ego_camera.pose, width=36,
                                  height=36, fov=env.ego_camera.fov, far=cfg.far)
            p = f"c{k}"
            out[p + "_x"] = sc.particles.positions.copy()
            out[p + "_radius"] = np.array(sc.params.radius)
            out[p + "_blade_pose"] = np.asarray(sc.bodies[1].pose, float)
            out[p + "_blade_half"] = np.array(cfg.blade_half_extents, float)
            cam_rec(p + "_ego", ego_cam, ego_cam.pose, out)
            cam_rec(p + "_sky", env.sky_camera, env.sky_camera.pose, out)
            out[p + "_ego_depth"] = render_depth(sc, ego_cam)
            out[p + "_sky_depth"] = render_depth(sc, env.sky_camera)
            k += 1
    out["n_env_cases"] = np.array(k)
    # primitives + grid scene
    rng = np.random.default_rng(7)
    x = f32(rng.uniform([-1, -1, 0.0], [1, 1, 0.6], size=(300, 3)))
    sph = RigidBody(rsdf.Sphere(0.3), name="s")
    sph.pose = make_pose(np.eye(3), np.array([0.5, 0.2, 0.9]))
    cyl = RigidBody(rsdf.Cylinder(0.25, 0.4), name="c")
    cyl.pose = make_pose(so3_exp(np.array([0.3, 0.0, 0.2])), np.array([-0.6, -0.3, 0.6]))
    grid = rsdf.bake_mesh_sdf(*__import__("granusim.meshes", fromlist=["x"]).make_box_mesh(
        np.array([0.2, 0.3, 0.15])), spacing=0.05)
    gb = RigidBody(grid, name="g")
    gb.pose = make_pose(so3_exp(np.array([0.0, 0.4, 0.1])), np.array([0.1, -0.7, 0.5]))
    sc = Scene(particles=ParticleSet(x, np.zeros_like(x)), bodies=[sph, cyl, gb],
               params=MaterialParams(radius=0.04))
    persp = DepthCamera(kind="perspective", pose=make_pose(
        np.array([[1.0, 0, 0], [0, -1.0, 0], [0, 0, -1.0]]) @ so3_exp(np.array([0.2, 0.1, 0.0])),
        np.array([0.0, 0.0, 3.0])), width=40, height=30, fov=1.0, far=8.0)
    ortho = DepthCamera(kind="orthographic", pose=make_pose(
        np.array([[1.0, 0, 0], [0, -1.0, 0], [0, 0, -1.0]]), np.array([0.0, 0.0, 4.0])),
        width=48, height=32, extent=(3.0, 2.0), far=10.0)
    out["p_x"] = x
    out["p_radius"] = np.array(0.04)
    out["p_sphere_pose"] = sph.pose
    out["p_cyl_pose"] = cyl.pose
    out["p_grid_pose"] = gb.pose
    out["p_grid_values"] = np.asarray(grid.values, float)
    out["p_grid_origin"] = np.asarray(grid.origin, float)
    out["p_grid_spacing"] = np.asarray(grid.spacing, float)
    cam_rec("p_persp", persp, persp.pose, out)
    cam_rec("p_ortho", ortho, ortho.pose, out)
    out["p_persp_depth"] = render_depth(sc, persp)
    out["p_ortho_depth"] = render_depth(sc, ortho)
    np.savez_compressed(OUT / "render.npz", **out)
    print({k: np.shape(v) for k, v in out.items() if k.endswith("depth")})


if __name__ == "__main__":
    main()
