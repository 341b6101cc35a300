"""Bulldozer task on the device: scene builder, reward, and the batched env
(SURVEY.md §8e config 3 / §8f rank 1).

``bulldozer_scene`` builds exactly the scene ``BulldozerEnv._build_scene``
does (envs.py:144-178): a jittered lattice bed truncated to ``n_particles``,
a ground half-space and a Box blade on a ``TrackSteeringDriver``.
``BatchedBulldozerEnv`` runs E such envs in one ``SceneBatch``: actions for
all envs in one array, the tracked vehicles advanced with array math
(``TrackSteeringBatch``), ``frame_skip`` physics substeps per control step as
one device batch, and the reward (``bulldozer_reward``, envs.py:61-70)
reduced per env on the device (``gg_env_box_stats``) so no particle state
crosses PCIe.  Observations are the reference's (``EnvObservation``,
envs.py:73-78): the 36x36 ego and 72x36 sky depth images rendered on the
device for every env in one launch (``render_batch``), and the vehicle pose.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .batch import SceneBatch, StaticBatch, TrackSteeringBatch
from .render import DepthCamera, render_batch
from .kinematics import TrackSteeringDriver, TrackSteeringState, make_pose
from .scene import BoxRegion, MaterialParams, ParticleSet, RigidBody, Scene, seed_particles_grid
from .sdf import Box, HalfSpace


@dataclass
class GoalBox:
    """Axis-aligned goal region (envs.py:39-58)."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        self.min = np.asarray(self.min, dtype=np.float64)
        self.max = np.asarray(self.max, dtype=np.float64)
        if not np.all(self.min < self.max):
            raise ValueError("goal box requires min < max componentwise")

    def contains(self, points: np.ndarray) -> np.ndarray:
        p = np.atleast_2d(points)
        return np.all((p >= self.min) & (p <= self.max), axis=1)

    def distance(self, points: np.ndarray) -> np.ndarray:
        p = np.atleast_2d(points)
        d = np.maximum(np.maximum(self.min - p, p - self.max), 0.0)
        return np.linalg.norm(d, axis=1)


def bulldozer_reward(positions: np.ndarray, goal: GoalBox) -> float:
    """Host version of the reward (envs.py:61-70)."""
    p = np.atleast_2d(positions)
    n = len(p)
    if n == 0:
        raise ValueError("reward is undefined for zero particles")
    inside = goal.contains(p)
    d = goal.distance(p)
    return float(np.where(inside, 100.0 / n, -d / n).sum())


@dataclass
class BulldozerEnvConfig:
    """envs.py:82-99 (same defaults)."""

    n_particles: int = 400
    radius: float = 0.05
    friction: float = 0.5
    timestep: float = 2e-3
    frame_skip: int = 10
    time_budget: float = 20.0
    scale_v: float = 1.0
    scale_omega: float = 1.0
    bed_min: tuple = (-1.0, -1.0, 0.05)
    bed_max: tuple = (1.0, 1.0, 0.45)
    goal_min: tuple = (1.5, -1.0, 0.0)
    goal_max: tuple = (3.0, 1.0, 1.0)
    blade_half_extents: tuple = (0.05, 0.5, 0.25)
    blade_offset: float = 0.45
    jitter: float = 0.3
    sky_extent: tuple = (8.0, 4.0)
    sky_height: float = 6.0
    far: float = 20.0


@dataclass
class BatchObservation:
    """EnvObservation (envs.py:73-78) for E envs."""

    ego: np.ndarray   # (E, 36, 36) float32 depth, meters
    sky: np.ndarray   # (E, 36, 72) float32 depth, meters
    pose: np.ndarray  # (E, 3) vehicle (x, y, yaw)


def ego_camera(cfg: BulldozerEnvConfig) -> DepthCamera:
    """The cockpit camera in the vehicle frame (envs.py:117-136)."""
    tilt = make_pose(np.array([[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]]).T,
                     np.array([-0.2, 0.0, 0.8]))
    pitch = 0.35
    tilt[:3, :3] = tilt[:3, :3] @ np.array([[np.cos(pitch), 0.0, -np.sin(pitch)], [0.0, 1.0, 0.0],
                                             [np.sin(pitch), 0.0, np.cos(pitch)]])
    return DepthCamera(kind="perspective", pose=tilt, width=36, height=36, fov=np.pi / 2.5,
                       far=cfg.far)


def sky_camera(cfg: BulldozerEnvConfig) -> DepthCamera:
    """The overhead orthographic camera (envs.py:137-148)."""
    pose = make_pose(np.array([[1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, -1.0]]),
                     np.array([0.0, 0.0, cfg.sky_height]))
    return DepthCamera(kind="orthographic", pose=pose, width=72, height=36, extent=cfg.sky_extent,
                       far=cfg.far)


def blade_base_pose(cfg: BulldozerEnvConfig) -> np.ndarray:
    return make_pose(np.eye(3), np.array([cfg.blade_offset, 0.0, cfg.blade_half_extents[2]]))


def bulldozer_scene(seed: int, cfg: BulldozerEnvConfig | None = None) -> Scene:
    """The scene of ``BulldozerEnv._build_scene(seed)`` (envs.py:144-178)."""
    cfg = cfg or BulldozerEnvConfig()
    rng = np.random.default_rng(seed)
    params = MaterialParams(radius=cfg.radius, friction=cfg.friction, timestep=cfg.timestep)
    particles = seed_particles_grid(BoxRegion(np.array(cfg.bed_min), np.array(cfg.bed_max)),
                                    cfg.radius, jitter=cfg.jitter, rng=rng)
    if particles.count > cfg.n_particles:
        particles = ParticleSet(particles.positions[: cfg.n_particles],
                                particles.velocities[: cfg.n_particles])
    ground = RigidBody(HalfSpace(), name="ground")
    driver = TrackSteeringDriver(state=TrackSteeringState(x=-2.0, y=0.0, theta=0.0), z=0.0,
                                 scale_v=cfg.scale_v, scale_omega=cfg.scale_omega,
                                 base_pose=blade_base_pose(cfg))
    blade = RigidBody(Box(np.array(cfg.blade_half_extents)), driver=driver, name="blade")
    return Scene(particles=particles, bodies=[ground, blade], params=params, seed=seed)


class BatchedBulldozerEnv:
    """E bulldozer envs in lock step on one device (BulldozerEnv, envs.py:102-230).

    ``reset(seeds)`` -> observation; ``step(actions (E, 2))`` ->
    (observation, rewards (E,), dones (E,), info) with info holding the
    per-env StepReport arrays of the last substep and the particles inside
    the goal box.  The observation is a ``BatchObservation`` (ego and sky
    depth images + poses; render=False: the (E, 3) poses alone).  All envs
    share one episode clock, as a synchronous vector env does."""

    action_shape = (2,)

    def __init__(self, n_envs: int, config: BulldozerEnvConfig | None = None, device: int = 0,
                 render: bool = True):
        if n_envs < 1:
            raise ValueError("n_envs must be >= 1")
        self.n_envs = n_envs
        self.config = config or BulldozerEnvConfig()
        cfg = self.config
        self.device = device
        self.episode_length = int(round(cfg.time_budget / (cfg.frame_skip * cfg.timestep)))
        self.goal = GoalBox(cfg.goal_min, cfg.goal_max)
        self.batch: SceneBatch | None = None
        self.driver: TrackSteeringBatch | None = None
        self._steps = 0
        self.render = render
        self.ego_camera = ego_camera(self.config)
        self.sky_camera = sky_camera(self.config)

    def reset(self, seeds=None):
        E = self.n_envs
        seeds = np.arange(E) if seeds is None else np.asarray(seeds, dtype=np.int64)
        if len(seeds) != E:
            raise ValueError(f"need {E} seeds, got {len(seeds)}")
        cfg = self.config
        scenes = [bulldozer_scene(int(s), cfg) for s in seeds]
        self.driver = TrackSteeringBatch(np.full(E, -2.0), np.zeros(E), np.zeros(E), z=0.0,
                                         scale_v=cfg.scale_v, scale_omega=cfg.scale_omega,
                                         base_pose=blade_base_pose(cfg))
        if self.batch is not None:
            self.batch.close()
        self.batch = SceneBatch(scenes, body_drivers={0: StaticBatch(E), 1: self.driver},
                                device=self.device)
        self._steps = 0
        return self._observe()

    def _observe(self):
        """BatchObservation (render=True) or the (E, 3) poses alone."""
        d = self.driver
        pose = np.stack([d.x, d.y, d.theta], axis=1)
        if not self.render:
            return pose
        # the camera rides the vehicle frame, not the blade offset (envs.py:182-186)
        blade, _, _ = d.pose_now()
        vehicle = blade.copy()
        vehicle[:, :3, 3] -= np.einsum("eij,j->ei", blade[:, :3, :3], d.base_pose[:3, 3])
        ego_poses = vehicle @ self.ego_camera.pose
        ego, sky = render_batch(self.batch, [self.ego_camera, self.sky_camera], [ego_poses, None])
        return BatchObservation(ego=ego, sky=sky, pose=pose)

    def goal_stats(self):
        """(rewards (E,), particles inside the goal box (E,)) on the device."""
        E = self.n_envs
        rew = np.zeros(E)
        ins = np.zeros(E, dtype=np.int64)
        N.check(self.batch.ctx, N.lib().gg_env_box_stats(
            self.batch.ctx, N.ptr(self.goal.min), N.ptr(self.goal.max), N.ptr(rew), N.ptr(ins)),
            "gg_env_box_stats")
        return rew, ins

    def step(self, actions):
        if self.batch is None:
            raise RuntimeError("step called before reset")
        a = np.asarray(actions, dtype=np.float64)
        if a.shape != (self.n_envs, 2):
            raise ValueError(f"actions shape must be ({self.n_envs}, 2), got {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValueError("action must be finite")
        self.driver.command(a)
        reps, _ = self.batch.run_raw(self.config.frame_skip)
        rew, ins = self.goal_stats()
        self._steps += 1
        done = np.full(self.n_envs, self._steps >= self.episode_length)
        last = reps[-1]
        info = {"n_contacts": last["n_contacts"].copy(),
                "max_penetration": last["max_penetration"].copy(),
                "kinetic_energy": last["kinetic_energy"].copy(),
                "in_goal": ins, "t": self.batch.t.copy()}
        return self._observe(), rew, done, info

    def close(self) -> None:
        if self.batch is not None:
            self.batch.close()
            self.batch = None
