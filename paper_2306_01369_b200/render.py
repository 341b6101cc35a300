"""Depth cameras rendered on the device (render.py of the reference).

``DepthCamera`` and ``render_depth(scene, camera)`` keep the reference's
interface (render.py:19-135): depth along the ray, ``far`` where nothing is
hit, camera frame +x right / +y down / +z forward, ``attach_body`` following a
body's pose.  The image is computed by ``gg_render_depth`` from the resident
particle state (no host copy of the bed): particles as spheres (exact float64
near root after a float32 pre-filter), bodies by float64 sphere tracing.
``render_batch`` renders every env of a ``SceneBatch`` in one launch.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import engine_for
from .kinematics import identity_pose

CAMERA_DTYPE = np.dtype(
    [
        ("kind", "<i4"),
        ("width", "<i4"),
        ("height", "<i4"),
        ("reserved", "<i4"),
        ("pose", "<f8", (16,)),
        ("fov", "<f8"),
        ("extent", "<f8", (2,)),
        ("far", "<f8"),
    ],
    align=True,
)


@dataclass
class DepthCamera:
    """render.py:19-32 (same fields and validation)."""

    kind: str = "perspective"
    pose: np.ndarray = field(default_factory=identity_pose)
    width: int = 36
    height: int = 36
    fov: float = np.pi / 3
    extent: tuple = (10.0, 10.0)
    far: float = 100.0
    attach_body: int | None = None

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("camera resolution must be at least 1x1")
        if self.far <= 0:
            raise ValueError("camera far plane must be positive")
        if self.kind not in ("perspective", "orthographic"):
            raise ValueError(f"unknown camera kind {self.kind!r}")


def camera_record(cam, pose: np.ndarray | None = None, out=None):
    """gg_camera record of ``cam`` at world pose ``pose`` (default cam.pose)."""
    rec = np.zeros((), dtype=CAMERA_DTYPE) if out is None else out
    rec["kind"] = 0 if cam.kind == "perspective" else 1
    rec["width"], rec["height"] = int(cam.width), int(cam.height)
    rec["pose"] = np.asarray(cam.pose if pose is None else pose, dtype=np.float64).reshape(16)
    rec["fov"] = float(cam.fov)
    rec["extent"] = np.asarray(cam.extent, dtype=np.float64)
    rec["far"] = float(cam.far)
    return rec


def _render(ctx, cams: np.ndarray, n_cams: int, per_env: bool, bodies: np.ndarray, nb: int,
            n_envs: int, sizes) -> list[np.ndarray]:
    total = sum(h * w for h, w in sizes)
    out = np.empty(n_envs * total, dtype=np.float32)
    st = N.lib().gg_render_depth(ctx, N.ptr(np.ascontiguousarray(cams)), n_cams, int(per_env),
                                 N.ptr(np.ascontiguousarray(bodies)) if nb else None, nb,
                                 N.ptr(out))
    N.check(ctx, st, "gg_render_depth")
    out = out.reshape(n_envs, total)
    imgs, o = [], 0
    for h, w in sizes:
        imgs.append(out[:, o:o + h * w].reshape(n_envs, h, w))
        o += h * w
    return imgs


def render_depth(scene, camera: DepthCamera) -> np.ndarray:
    """Depth image (height, width) float32 meters (render.py:119-135)."""
    pose = None
    if camera.attach_body is not None:
        pose = np.asarray(scene.bodies[camera.attach_body].pose) @ np.asarray(camera.pose)
    if scene.particles.count == 0:
        raise ValueError("render_depth on the device needs at least one particle")
    eng = engine_for(scene)
    eng.prepare(scene)
    nb = len(scene.bodies)
    rows = np.zeros(max(nb, 1), dtype=N.BODY_DTYPE)
    for b, body in enumerate(scene.bodies):
        eng.body_row(body, float(scene.params.radius), rows[b])
    cam = camera_record(camera, pose)
    return _render(eng.ctx, cam.reshape(1), 1, False, rows, nb, 1,
                   [(camera.height, camera.width)])[0][0]


def render_batch(batch, cameras: list, poses: list | None = None) -> list[np.ndarray]:
    """Render camera c of every env of ``batch`` (a SceneBatch) at its last
    committed state and body poses.  ``poses[c]`` (E, 4, 4) gives per-env
    world poses of camera c (None: cameras[c].pose for all envs).  Returns
    one (E, height, width) float32 array per camera."""
    E, C = batch.E, len(cameras)
    per_env = poses is not None and any(p is not None for p in poses)
    if per_env:
        recs = np.zeros((E, C), dtype=CAMERA_DTYPE)
        for c, cam in enumerate(cameras):
            one = camera_record(cam)
            for f in ("kind", "width", "height", "fov", "extent", "far"):
                recs[f][:, c] = one[f]
            P = cam.pose if poses[c] is None else poses[c]
            recs["pose"][:, c] = np.broadcast_to(np.asarray(P, np.float64), (E, 4, 4)).reshape(E, 16)
    else:
        recs = np.zeros(C, dtype=CAMERA_DTYPE)
        for c, cam in enumerate(cameras):
            recs[c] = camera_record(cam)
    return _render(batch.ctx, recs, C, per_env, batch.last_bodies(), batch.nb, E,
                   [(cam.height, cam.width) for cam in cameras])
