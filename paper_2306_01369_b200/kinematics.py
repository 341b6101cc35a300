"""Kinematic body drivers (host side; evaluated once per body per step).

Mirrors the reference's driver interface (kinematics.py:105-322): a driver
returns the body pose (4x4) and twist (omega, v_origin) at time t, and a
velocity-controlled kinematic chain drives links.  These run on the host
because a scene has a handful of bodies; their outputs are packed into the
per-step body tables the device consumes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def identity_pose() -> np.ndarray:
    return np.eye(4)


def make_pose(rotation: np.ndarray, translation: np.ndarray) -> np.ndarray:
    T = np.eye(4)
    T[:3, :3] = rotation
    T[:3, 3] = translation
    return T


def skew(w: np.ndarray) -> np.ndarray:
    wx, wy, wz = (float(c) for c in w)
    return np.array([[0.0, -wz, wy], [wz, 0.0, -wx], [-wy, wx, 0.0]])


def so3_exp(w: np.ndarray) -> np.ndarray:
    """Rodrigues' formula; first-order near zero (kinematics.py:39-47)."""
    w = np.asarray(w, dtype=np.float64)
    angle = np.linalg.norm(w)
    if angle < 1e-12:
        return np.eye(3) + skew(w)
    K = skew(w / angle)
    return np.eye(3) + np.sin(angle) * K + (1.0 - np.cos(angle)) * (K @ K)


def so3_log(R: np.ndarray) -> np.ndarray:
    axis = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    angle = np.arccos(np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0))
    if angle < 1e-9:
        return axis / 2.0
    return angle / (2.0 * np.sin(angle)) * axis


def se3_inverse(T: np.ndarray) -> np.ndarray:
    R = T[:3, :3]
    return make_pose(R.T, -R.T @ T[:3, 3])


def rotation_error(R: np.ndarray) -> float:
    return float(np.abs(R.T @ R - np.eye(3)).max())


class MotionDriver:
    """pose_at(t) -> 4x4, twist_at(t) -> (omega, v_origin), world frame."""

    def pose_at(self, t: float) -> np.ndarray:
        raise NotImplementedError

    def twist_at(self, t: float):
        raise NotImplementedError


@dataclass
class StaticDriver(MotionDriver):
    pose: np.ndarray = field(default_factory=identity_pose)

    def pose_at(self, t):
        return self.pose

    def twist_at(self, t):
        return np.zeros(3), np.zeros(3)

    def pose_batch(self, ts):
        T = len(ts)
        return np.broadcast_to(np.asarray(self.pose, dtype=np.float64), (T, 4, 4)), np.zeros((T, 3)), np.zeros((T, 3))


@dataclass
class SpinDriver(MotionDriver):
    """Constant angular rate about a world axis through ``center``."""

    axis: np.ndarray
    rate: float
    center: np.ndarray = field(default_factory=lambda: np.zeros(3))
    base_pose: np.ndarray = field(default_factory=identity_pose)
    phase: float = 0.0

    def __post_init__(self):
        a = np.asarray(self.axis, dtype=np.float64)
        self.axis = a / np.linalg.norm(a)
        self.center = np.asarray(self.center, dtype=np.float64)

    def pose_at(self, t):
        R = so3_exp(self.axis * (self.rate * t + self.phase))
        return make_pose(R, self.center - R @ self.center) @ self.base_pose

    def twist_at(self, t):
        omega = self.axis * self.rate
        return omega, np.cross(omega, self.pose_at(t)[:3, 3] - self.center)

    def pose_batch(self, ts):
        ts = np.asarray(ts, dtype=np.float64)
        th = self.rate * ts + self.phase
        K = skew(self.axis)
        K2 = K @ K
        R = np.eye(3) + np.sin(th)[:, None, None] * K + (1.0 - np.cos(th))[:, None, None] * K2
        small = np.abs(th) < 1e-12
        if small.any():
            R[small] = np.eye(3) + th[small, None, None] * K
        spin = np.zeros((len(ts), 4, 4))
        spin[:, :3, :3] = R
        spin[:, :3, 3] = self.center - R @ self.center
        spin[:, 3, 3] = 1.0
        P = spin @ self.base_pose
        omega = self.axis * self.rate
        return P, np.broadcast_to(omega, (len(ts), 3)), np.cross(omega, P[:, :3, 3] - self.center)


@dataclass
class ScriptedDriver(MotionDriver):
    """Pose from a callable; twist by central differences."""

    sampler: object
    fd_step: float = 1e-5

    def pose_at(self, t):
        return self.sampler(t)

    def twist_at(self, t):
        h = self.fd_step
        A, B = self.sampler(t - h), self.sampler(t + h)
        omega = so3_log(B[:3, :3] @ A[:3, :3].T) / (2.0 * h)
        return omega, (B[:3, 3] - A[:3, 3]) / (2.0 * h)


@dataclass
class ChainLink:
    parent: int
    origin: np.ndarray
    joint_type: str
    axis: np.ndarray
    velocity_limit: float = np.inf

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64)
        a = np.asarray(self.axis, dtype=np.float64)
        norm = np.linalg.norm(a)
        if norm == 0:
            raise ValueError("joint axis must be nonzero")
        self.axis = a / norm
        if self.joint_type not in ("revolute", "prismatic"):
            raise ValueError(f"unknown joint type {self.joint_type!r}")


class KinematicChain:
    """Velocity-controlled kinematic tree (kinematics.py:256-306)."""

    def __init__(self, links: list[ChainLink], base_pose: np.ndarray | None = None):
        for i, link in enumerate(links):
            if not -1 <= link.parent < i:
                raise ValueError(f"link {i}: parent {link.parent} does not precede it (tree required)")
        self.links = links
        self.base_pose = identity_pose() if base_pose is None else np.asarray(base_pose)
        self.q = np.zeros(len(links))
        self.qd = np.zeros(len(links))

    def fk(self, q: np.ndarray | None = None):
        q = self.q if q is None else np.asarray(q, dtype=np.float64)
        poses: list[np.ndarray] = []
        spatial: list[tuple[np.ndarray, np.ndarray]] = []  # (omega, v at world origin)
        for i, link in enumerate(self.links):
            parent = self.base_pose if link.parent < 0 else poses[link.parent]
            joint = parent @ link.origin
            axis_w = joint[:3, :3] @ link.axis
            if link.joint_type == "revolute":
                local = make_pose(so3_exp(link.axis * q[i]), np.zeros(3))
                w_j = axis_w * self.qd[i]
                v_j = -np.cross(w_j, joint[:3, 3])
            else:
                local = make_pose(np.eye(3), link.axis * q[i])
                w_j = np.zeros(3)
                v_j = axis_w * self.qd[i]
            poses.append(joint @ local)
            w_p, v_p = (np.zeros(3), np.zeros(3)) if link.parent < 0 else spatial[link.parent]
            spatial.append((w_p + w_j, v_p + v_j))
        twists = [(w, v + np.cross(w, poses[i][:3, 3])) for i, (w, v) in enumerate(spatial)]
        return poses, twists

    def advance(self, qd_cmd: np.ndarray, dt: float) -> None:
        lim = np.array([link.velocity_limit for link in self.links])
        self.qd = np.clip(np.asarray(qd_cmd, dtype=np.float64), -lim, lim)
        self.q = self.q + dt * self.qd


@dataclass
class ChainLinkDriver(MotionDriver):
    chain: KinematicChain
    link_index: int

    def pose_at(self, t):
        return self.chain.fk()[0][self.link_index]

    def twist_at(self, t):
        return self.chain.fk()[1][self.link_index]

    def pose_batch(self, ts):
        # the chain does not move inside one batch (nothing advances it)
        poses, twists = self.chain.fk()
        w, v = twists[self.link_index]
        T = len(ts)
        return (np.broadcast_to(poses[self.link_index], (T, 4, 4)), np.broadcast_to(w, (T, 3)),
                np.broadcast_to(v, (T, 3)))


@dataclass
class TrackSteeringState:
    x: float = 0.0
    y: float = 0.0
    theta: float = 0.0


def track_steering_advance(state, action, dt, scale_v=1.0, scale_omega=1.0) -> TrackSteeringState:
    a = np.clip(np.asarray(action, dtype=np.float64), -1.0, 1.0)
    theta = state.theta + dt * scale_omega * a[1]
    return TrackSteeringState(
        x=state.x + dt * scale_v * a[0] * np.cos(theta),
        y=state.y + dt * scale_v * a[0] * np.sin(theta),
        theta=theta,
    )


@dataclass
class TrackSteeringDriver(MotionDriver):
    state: TrackSteeringState = field(default_factory=TrackSteeringState)
    z: float = 0.0
    scale_v: float = 1.0
    scale_omega: float = 1.0
    base_pose: np.ndarray = field(default_factory=identity_pose)
    _action: np.ndarray = field(default_factory=lambda: np.zeros(2))

    def command(self, action) -> None:
        self._action = np.clip(np.asarray(action, dtype=np.float64), -1.0, 1.0)

    def advance(self, dt: float) -> None:
        self.state = track_steering_advance(self.state, self._action, dt, self.scale_v,
                                            self.scale_omega)

    def pose_at(self, t):
        R = so3_exp(np.array([0.0, 0.0, self.state.theta]))
        return make_pose(R, np.array([self.state.x, self.state.y, self.z])) @ self.base_pose

    def twist_at(self, t):
        omega = np.array([0.0, 0.0, self.scale_omega * self._action[1]])
        heading = np.array([np.cos(self.state.theta), np.sin(self.state.theta), 0.0])
        ref = np.array([self.state.x, self.state.y, self.z])
        return omega, self.scale_v * self._action[0] * heading + np.cross(
            omega, self.pose_at(t)[:3, 3] - ref
        )
