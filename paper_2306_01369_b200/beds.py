"""Synthetic particle beds and the benchmark scenes.

* ``lattice_bed``   compressed cubic lattice on a floor (single-step stress input)
* ``column_scene``  the reference's ``make_column_scene`` (envs.py:351-390):
                    jittered lattice in a cylindrical tube with a floor
* ``hero_scene``    config 2: a settled column plus a Box scoop
                    (``sdf.Box([0.15, 0.1, 0.04])``, envs.py:283-287) on the
                    ExcavationEnv 7-joint chain (envs.py:250-266) moving at a
                    constant joint velocity 0.3 x limits (what a constant
                    action does in ExcavationEnv.step, envs.py:336-341)

``JointTrajectoryDriver`` is that constant-velocity chain written as a pure
function of time, so a whole batch of body poses can be evaluated at once
(``pose_batch``) instead of one Python FK per step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kinematics import ChainLink, KinematicChain, MotionDriver, make_pose
from .scene import CylinderRegion, MaterialParams, ParticleSet, RigidBody, Scene, seed_particles_grid
from .sdf import Box, HalfSpace, Tube


def lattice_bed(n: int, r: float = 0.05, s: float = 0.99, jitter: float = 0.01,
                seed: int = 0) -> np.ndarray:
    """SURVEY.md §8d generator: nx = ny = round(n^(1/3)), nz = ceil(n / (nx ny));
    x = idx * (2 r s) + (0, 0, r s) + U(-jitter r, jitter r); first n points."""
    nx = max(int(round(n ** (1.0 / 3.0))), 1)
    nz = int(np.ceil(n / (nx * nx)))
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(nx), np.arange(nz), indexing="ij")
    idx = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3).astype(np.float64)
    rng = np.random.default_rng(seed)
    pts = idx * (2.0 * r * s) + np.array([0.0, 0.0, r * s])
    pts = pts + rng.uniform(-jitter * r, jitter * r, size=pts.shape)
    return pts[:n]


def lattice_scene(n: int, r: float = 0.05, seed: int = 0, **params_kw) -> Scene:
    pos = lattice_bed(n, r=r, seed=seed)
    params = MaterialParams(radius=r, **params_kw)
    floor = RigidBody(HalfSpace(), name="floor")
    return Scene(particles=ParticleSet(pos, np.zeros_like(pos)), bodies=[floor], params=params,
                 seed=seed)


def column_scene(n_particles: int, r: float = 0.05, aspect: float = 4.0, params=None,
                 jitter: float = 0.2, seed: int = 0) -> Scene:
    """Jittered lattice in a tube of aspect ``aspect`` on a floor (envs.py:351-390)."""
    params = params or MaterialParams(radius=r, friction=0.5)
    r = params.radius
    vol = n_particles * (2.0 * r) ** 3
    radius = max((vol / (np.pi * 2.0 * aspect)) ** (1.0 / 3.0), 3.0 * r)
    height = 2.0 * aspect * radius
    ps = seed_particles_grid(CylinderRegion([0.0, 0.0], radius, 0.0, height), r, jitter=jitter,
                             rng=np.random.default_rng(seed))
    while ps.count < n_particles:
        height *= 1.5
        ps = seed_particles_grid(CylinderRegion([0.0, 0.0], radius, 0.0, height), r,
                                 jitter=jitter, rng=np.random.default_rng(seed))
    x = ps.positions[:n_particles].copy()
    bodies = [RigidBody(HalfSpace(), name="floor"), RigidBody(Tube(radius), name="wall")]
    return Scene(particles=ParticleSet(x, np.zeros_like(x)), bodies=bodies, params=params,
                 seed=seed)


make_column_scene = column_scene


# ---------------------------------------------------------------------------
# batched forward kinematics for a constant-joint-velocity chain
# ---------------------------------------------------------------------------
def _skew(a: np.ndarray) -> np.ndarray:
    return np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])


def _rot_batch(axis: np.ndarray, theta: np.ndarray) -> np.ndarray:
    """so3_exp(axis * theta) for a unit axis and T angles -> (T, 3, 3)."""
    K = _skew(axis)
    K2 = K @ K
    th = np.asarray(theta, dtype=np.float64)
    big = np.abs(th) >= 1e-12
    R = np.eye(3) + np.sin(th)[:, None, None] * K + (1.0 - np.cos(th))[:, None, None] * K2
    small = np.eye(3) + th[:, None, None] * K  # first-order branch of so3_exp
    return np.where(big[:, None, None], R, small)


@dataclass
class JointTrajectoryDriver(MotionDriver):
    """Link ``link_index`` of ``chain`` with q(t) = q0 + qd * t."""

    chain: KinematicChain
    link_index: int
    qd: np.ndarray
    q0: np.ndarray | None = None

    def __post_init__(self):
        lim = np.array([l.velocity_limit for l in self.chain.links])
        self.qd = np.clip(np.asarray(self.qd, dtype=np.float64), -lim, lim)
        self.q0 = np.zeros(len(self.chain.links)) if self.q0 is None else np.asarray(self.q0, float)

    def pose_batch(self, ts: np.ndarray):
        ts = np.asarray(ts, dtype=np.float64)
        T = len(ts)
        links = self.chain.links
        poses, w_sp, v_sp = [], [], []
        for i, link in enumerate(links):
            parent = (np.broadcast_to(self.chain.base_pose, (T, 4, 4)) if link.parent < 0
                      else poses[link.parent])
            joint = parent @ link.origin
            axis_w = joint[:, :3, :3] @ link.axis
            q = self.q0[i] + self.qd[i] * ts
            local = np.zeros((T, 4, 4))
            local[:, 3, 3] = 1.0
            if link.joint_type == "revolute":
                local[:, :3, :3] = _rot_batch(link.axis, q)
                wj = axis_w * self.qd[i]
                vj = -np.cross(wj, joint[:, :3, 3])
            else:
                local[:, :3, :3] = np.eye(3)
                local[:, :3, 3] = link.axis[None, :] * q[:, None]
                wj = np.zeros((T, 3))
                vj = axis_w * self.qd[i]
            poses.append(joint @ local)
            if link.parent < 0:
                w_sp.append(wj)
                v_sp.append(vj)
            else:
                w_sp.append(w_sp[link.parent] + wj)
                v_sp.append(v_sp[link.parent] + vj)
        k = self.link_index
        P = poses[k]
        w = w_sp[k]
        v = v_sp[k] + np.cross(w, P[:, :3, 3])
        return P, w, v

    def pose_at(self, t):
        return self.pose_batch(np.array([t]))[0][0]

    def twist_at(self, t):
        _, w, v = self.pose_batch(np.array([t]))
        return w[0], v[0]


@dataclass
class DigDriver(MotionDriver):
    """One digging pass of a bucket (analytic pose and twist, so a batch of
    steps is evaluated with array operations).  Until ``t0`` the bucket
    waits at ``start``; over ``duration`` seconds it travels ``length``
    metres along the horizontal unit vector ``direction`` while dipping to
    ``depth`` below its start height on a half sine and pitching from
    ``pitch0`` to ``pitch1`` (radians, about the horizontal axis
    ``z x direction``); afterwards it rises at ``lift_speed`` m/s.  The body
    frame origin follows the path; twist = (pitch rate x axis, path velocity)."""

    start: np.ndarray
    direction: np.ndarray
    length: float
    depth: float
    duration: float
    pitch0: float = 0.0
    pitch1: float = 0.0
    t0: float = 0.0
    lift_speed: float = 0.0

    def __post_init__(self):
        self.start = np.asarray(self.start, dtype=np.float64)
        d = np.asarray(self.direction, dtype=np.float64)
        d = d - np.array([0.0, 0.0, d[2]])
        self.direction = d / np.linalg.norm(d)
        ax = np.cross([0.0, 0.0, 1.0], self.direction)
        self.axis = ax / np.linalg.norm(ax)

    def pose_batch(self, ts):
        ts = np.atleast_1d(np.asarray(ts, dtype=np.float64))
        T = len(ts)
        u = (ts - self.t0) / self.duration
        s = np.clip(u, 0.0, 1.0)
        inside = (u > 0.0) & (u < 1.0)
        after = np.maximum(ts - self.t0 - self.duration, 0.0)
        ez = np.array([0.0, 0.0, 1.0])
        pos = (self.start[None, :] + self.direction[None, :] * (self.length * s)[:, None]
               - ez[None, :] * (self.depth * np.sin(np.pi * s))[:, None]
               + ez[None, :] * (self.lift_speed * after)[:, None])
        pitch = self.pitch0 + (self.pitch1 - self.pitch0) * s
        P = np.zeros((T, 4, 4))
        P[:, :3, :3] = _rot_batch(self.axis, pitch)
        P[:, :3, 3] = pos
        P[:, 3, 3] = 1.0
        rate = np.where(inside, 1.0 / self.duration, 0.0)
        v = (self.direction[None, :] * (self.length * rate)[:, None]
             - ez[None, :] * (self.depth * np.pi * np.cos(np.pi * s) * rate)[:, None]
             + ez[None, :] * np.where(u >= 1.0, self.lift_speed, 0.0)[:, None])
        w = self.axis[None, :] * ((self.pitch1 - self.pitch0) * rate)[:, None]
        return P, w, v

    def pose_at(self, t):
        return self.pose_batch([t])[0][0]

    def twist_at(self, t):
        _, w, v = self.pose_batch([t])
        return w[0], v[0]


def excavation_chain(base_translation=(0.0, 0.0, 0.0)) -> KinematicChain:
    """ExcavationEnv._build_chain (envs.py:250-266), base moved by a translation."""
    up, side = np.array([0.0, 0.0, 1.0]), np.array([0.0, 1.0, 0.0])
    axes = [up, side, up, side, up, side, np.array([1.0, 0.0, 0.0])]
    heights = [0.3, 0.3, 0.25, 0.25, 0.2, 0.15, 0.1]
    links = [
        ChainLink(parent=k - 1, origin=make_pose(np.eye(3), np.array([0.0, 0.0, heights[k]])),
                  joint_type="revolute", axis=axes[k], velocity_limit=1.0)
        for k in range(7)
    ]
    return KinematicChain(links, base_pose=make_pose(np.eye(3), np.asarray(base_translation, float)))


def add_scoop(scene: Scene, action: float = 0.3, depth: float = 0.05) -> RigidBody:
    """Attach the ExcavationEnv scoop so it starts ``depth`` below the bed top."""
    x = scene.particles.positions
    top = float(x[:, 2].max()) + scene.params.radius
    cx, cy = float(np.median(x[:, 0])), float(np.median(x[:, 1]))
    chain = excavation_chain((cx, cy, top - depth - 1.55))
    limits = np.array([l.velocity_limit for l in chain.links])
    driver = JointTrajectoryDriver(chain, 6, qd=action * limits)
    scoop = RigidBody(Box(np.array([0.15, 0.1, 0.04])), driver=driver, name="scoop")
    scoop.update(scene.t)
    scene.bodies.append(scoop)
    scene.chains["arm"] = chain
    return scoop


# the config-4 excavator bucket (bench.py bed1m): 2.4 m wide, 1.2 m deep,
# 1.2 m tall outside, 15 cm walls, baked at 5 cm
BUCKET1M_HALF = (0.6, 1.2, 0.6)
BUCKET1M_WALL = 0.15
BUCKET1M_SPACING = 0.05


def excavator_dig(x: np.ndarray, t_now: float, half=BUCKET1M_HALF, speed: float = 1.0,
                  length: float = 5.0, lead: float = 1.0) -> "DigDriver":
    """A front-loader pass of the config-4 bucket into the flank of a settled
    pile ``x``: mouth facing +x (pitch pi/2: the bucket's local +z is world
    +x, its width along y), bottom 10 cm above the floor, lip 10 cm before
    the point of the pile's -x flank (along the y centre band) where the
    pile is as tall as the bucket; it drives ``length`` m into
    the pile at ``speed`` m/s while curling the mouth up to 0.3 rad, then
    lifts at 0.5 m/s.  The pass started ``lead`` seconds before ``t_now``,
    so at t_now the bucket is already ``lead * speed`` m into the pile."""
    x = np.asarray(x, dtype=np.float64)
    yc = float(np.median(x[:, 1]))
    top = 2.0 * half[0] + 0.1  # the bucket's top above the floor
    # the flank: the first 0.25 m slice along the y centre band (from -x) in
    # which the pile reaches the bucket's top
    band = np.abs(x[:, 1] - yc) < half[1]
    xb = x[band]
    lo = float(xb[:, 0].min())
    idx = np.floor((xb[:, 0] - lo) / 0.25).astype(np.int64)
    zmax = np.zeros(int(idx.max()) + 1)
    np.maximum.at(zmax, idx, xb[:, 2])
    hit = np.nonzero(zmax >= top)[0]
    x_edge = lo + 0.25 * float(hit[0] if len(hit) else 0)
    start = np.array([x_edge - 0.1 - half[2], yc, half[0] + 0.1])
    return DigDriver(start=start, direction=np.array([1.0, 0.0, 0.0]), length=length, depth=0.0,
                     duration=length / speed, pitch0=0.5 * np.pi, pitch1=0.3, t0=t_now - lead,
                     lift_speed=0.5)


def hero_scene(n: int = 50_000, seed: int = 0, r: float = 0.05) -> Scene:
    """Config 2 before settling: column bed (aspect 1) + floor + tube wall."""
    params = MaterialParams(radius=r, friction=0.5, timestep=1e-3)
    return column_scene(n, r=r, aspect=1.0, params=params, seed=seed)
