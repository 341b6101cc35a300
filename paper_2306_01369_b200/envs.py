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
from .batch import ChainBatch, SceneBatch, StaticBatch, TrackSteeringBatch
from .render import DepthCamera, render_batch
from .kinematics import (
    ChainLink,
    ChainLinkDriver,
    KinematicChain,
    TrackSteeringDriver,
    TrackSteeringState,
    make_pose,
)
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
        # the ground and the blade's TrackSteeringDriver run on the device:
        # no per-substep body tables are packed or uploaded
        self.device_drivers = self.batch.drive_on_device()
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
        reps, _ = self.batch.run_raw(self.config.frame_skip, last_only=True)
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


# ---------------------------------------------------------------------------
# Excavation: the 7-joint arm with a Box scoop (envs.py:233-348)
# ---------------------------------------------------------------------------
def excavation_links() -> list:
    """The ExcavationEnv chain (envs.py:250-266): 7 revolute joints, axes
    up/side alternating then x, link heights 0.3 ... 0.1, velocity limit 1."""
    up, side = np.array([0.0, 0.0, 1.0]), np.array([0.0, 1.0, 0.0])
    axes = [up, side, up, side, up, side, np.array([1.0, 0.0, 0.0])]
    heights = [0.3, 0.3, 0.25, 0.25, 0.2, 0.15, 0.1]
    return [ChainLink(parent=k - 1, origin=make_pose(np.eye(3), np.array([0.0, 0.0, heights[k]])),
                      joint_type="revolute", axis=axes[k], velocity_limit=1.0) for k in range(7)]


def excavation_scene(seed: int, n_particles: int = 300, timestep: float = 2e-3) -> Scene:
    """The scene of ``ExcavationEnv.reset(seed)`` (envs.py:268-292)."""
    rng = np.random.default_rng(seed)
    params = MaterialParams(radius=0.05, timestep=timestep)
    particles = seed_particles_grid(BoxRegion(np.array([0.2, -0.6, 0.05]), np.array([1.4, 0.6, 0.35])),
                                    params.radius, jitter=0.3, rng=rng)
    if particles.count > n_particles:
        particles = ParticleSet(particles.positions[:n_particles], particles.velocities[:n_particles])
    chain = KinematicChain(excavation_links())
    scoop = RigidBody(Box(np.array([0.15, 0.1, 0.04])), driver=ChainLinkDriver(chain, 6), name="scoop")
    ground = RigidBody(HalfSpace(), name="ground")
    return Scene(particles=particles, bodies=[ground, scoop], params=params, seed=seed)


class BatchedExcavationEnv:
    """E excavation envs in lock step (ExcavationEnv, envs.py:233-348): the
    joints of all arms advance with array math (``ChainBatch``), the scoop
    poses go to the device as one body table per substep batch, and the
    observation (36x36 ego camera on the end effector, 72x36 sky) is rendered
    on the device.  Task-less like the reference: reward 0."""

    action_shape = (7,)

    def __init__(self, n_envs: int, n_particles: int = 300, frame_skip: int = 10,
                 time_budget: float = 20.0, timestep: float = 2e-3, device: int = 0,
                 render: bool = True):
        if n_envs < 1:
            raise ValueError("n_envs must be >= 1")
        self.n_envs, self.n_particles = n_envs, n_particles
        self.frame_skip, self.timestep = frame_skip, timestep
        self.episode_length = int(round(time_budget / (frame_skip * timestep)))
        self.device, self.render = device, render
        self.batch: SceneBatch | None = None
        self.chain: ChainBatch | None = None
        self._steps = 0
        self.sky_camera = DepthCamera(
            kind="orthographic",
            pose=make_pose(np.array([[1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, -1.0]]),
                           np.array([0.7, 0.0, 4.0])),
            width=72, height=36, extent=(4.0, 2.0), far=10.0)
        self.ego_local = make_pose(np.array([[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]]).T,
                                   np.array([0.0, 0.0, 0.2]))
        self.ego_camera = DepthCamera(kind="perspective", width=36, height=36, far=10.0)

    def reset(self, seeds=None):
        E = self.n_envs
        seeds = np.arange(E) if seeds is None else np.asarray(seeds, dtype=np.int64)
        if len(seeds) != E:
            raise ValueError(f"need {E} seeds, got {len(seeds)}")
        scenes = [excavation_scene(int(s), self.n_particles, self.timestep) for s in seeds]
        counts = {sc.particles.count for sc in scenes}
        if len(counts) != 1:
            raise ValueError(f"seeded beds differ in size {sorted(counts)}: lower n_particles")
        self.chain = ChainBatch(excavation_links(), E, link_index=6)
        if self.batch is not None:
            self.batch.close()
        self.batch = SceneBatch(scenes, body_drivers={0: StaticBatch(E), 1: self.chain},
                                device=self.device)
        # the ground and the arm's forward kinematics run on the device
        self.device_drivers = self.batch.drive_on_device()
        self._steps = 0
        return self._observe()

    def _observe(self):
        P, _, _ = self.chain.fk()
        end = P[:, -1]
        yaw = np.arctan2(end[:, 1, 0], end[:, 0, 0])
        pose = np.stack([end[:, 0, 3], end[:, 1, 3], yaw], axis=1)
        if not self.render:
            return pose
        ego, sky = render_batch(self.batch, [self.ego_camera, self.sky_camera],
                                [end @ self.ego_local, None])
        return BatchObservation(ego=ego, sky=sky, pose=pose)

    def step(self, actions):
        if self.batch is None:
            raise RuntimeError("step called before reset")
        a = np.asarray(actions, dtype=np.float64)
        if a.shape != (self.n_envs, 7):
            raise ValueError(f"actions shape must be ({self.n_envs}, 7), got {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValueError("action must be finite")
        self.chain.command(np.clip(a, -1.0, 1.0) * self.chain.limits)
        reps, _ = self.batch.run_raw(self.frame_skip, last_only=True)
        self._steps += 1
        done = np.full(self.n_envs, self._steps >= self.episode_length)
        info = {"n_contacts": reps[-1]["n_contacts"].copy(), "t": self.batch.t.copy()}
        return self._observe(), np.zeros(self.n_envs), done, info

    def close(self) -> None:
        if self.batch is not None:
            self.batch.close()
            self.batch = None
