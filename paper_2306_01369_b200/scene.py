"""Scene state types with the reference's attribute API (scene.py:47-185).

``ParticleSet`` here is device-aware: once a scene has been stepped on the
GPU its arrays are mirrors of the device state, downloaded lazily when read
and re-uploaded before the next step if they may have been modified (any
read hands out a mutable array, so a read marks the mirror dirty).  Plain
reference ``ParticleSet`` objects are accepted too; they are synchronised
eagerly every step (stepper.py:102-106 mutates them in place).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError
from .kinematics import KinematicChain, MotionDriver, StaticDriver, identity_pose, rotation_error
from .sdf import SdfGeometry

DEFAULT_PARTICLE_MASS = 1.0


@dataclass
class MaterialParams:
    radius: float = 0.05
    particle_mass: float = DEFAULT_PARTICLE_MASS
    friction: float = 0.5
    baumgarte_alpha: float = 0.2
    timestep: float = 1e-3
    solver_iterations: int = 10
    gravity: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -9.81]))
    gamma: float = 1.0

    def __post_init__(self):
        self.gravity = np.asarray(self.gravity, dtype=np.float64)
        self.validate()

    def validate(self) -> None:
        checks = [
            (self.radius > 0, f"radius must be > 0, got {self.radius}"),
            (self.particle_mass > 0, f"particle_mass must be > 0, got {self.particle_mass}"),
            (self.friction >= 0, f"friction must be >= 0, got {self.friction}"),
            (0.0 <= self.baumgarte_alpha <= 1.0,
             f"baumgarte_alpha must be in [0, 1], got {self.baumgarte_alpha}"),
            (self.timestep > 0, f"timestep must be > 0, got {self.timestep}"),
            (isinstance(self.solver_iterations, (int, np.integer)) and self.solver_iterations >= 1,
             f"solver_iterations must be a positive integer, got {self.solver_iterations}"),
            (self.gravity.shape == (3,) and bool(np.all(np.isfinite(self.gravity))),
             f"gravity must be a finite 3-vector, got {self.gravity}"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValidationError(msg)


def _as_state_array(a) -> np.ndarray:
    return np.atleast_2d(np.asarray(a, dtype=np.float64)).reshape(-1, 3)


class ParticleSet:
    """Particle positions/velocities, float64 (n, 3), device-mirrored."""

    def __init__(self, positions, velocities):
        self._x = np.array(_as_state_array(positions), dtype=np.float64, order="C")
        self._v = np.array(_as_state_array(velocities), dtype=np.float64, order="C")
        self._engine = None       # engine whose device copy is authoritative
        self._host_dirty = True   # host arrays may differ from the device copy
        self.validate()

    # -- device mirror protocol (used by engine.py) --------------------------
    def _refresh(self) -> None:
        eng = self._engine
        if eng is not None and eng.device_newer:
            eng.download_into(self._x, self._v)

    @property
    def positions(self) -> np.ndarray:
        self._refresh()
        self._host_dirty = True
        return self._x

    @positions.setter
    def positions(self, value) -> None:
        self._refresh()
        self._x = np.array(_as_state_array(value), dtype=np.float64, order="C")
        self._host_dirty = True

    @property
    def velocities(self) -> np.ndarray:
        self._refresh()
        self._host_dirty = True
        return self._v

    @velocities.setter
    def velocities(self, value) -> None:
        self._refresh()
        self._v = np.array(_as_state_array(value), dtype=np.float64, order="C")
        self._host_dirty = True

    @property
    def count(self) -> int:
        return self._x.shape[0]

    def validate(self) -> None:
        self._refresh()
        if self._x.shape != self._v.shape:
            raise ValidationError(
                f"positions and velocities must have equal shape, got "
                f"{self._x.shape} vs {self._v.shape}"
            )
        if not np.all(np.isfinite(self._x)):
            raise ValidationError("positions must be finite")
        if not np.all(np.isfinite(self._v)):
            raise ValidationError("velocities must be finite")

    # copies and pickles carry the CURRENT state: download first, and the copy
    # owns only host arrays (its next step uploads them to its own context)
    def __deepcopy__(self, memo):
        self._refresh()
        new = ParticleSet.__new__(ParticleSet)
        memo[id(self)] = new
        new._x = self._x.copy()
        new._v = self._v.copy()
        new._engine = None
        new._host_dirty = True
        return new

    def __getstate__(self):
        self._refresh()
        return {"_x": self._x.copy(), "_v": self._v.copy()}

    def __setstate__(self, state):
        self._x = state["_x"]
        self._v = state["_v"]
        self._engine = None
        self._host_dirty = True

    @staticmethod
    def empty() -> "ParticleSet":
        return ParticleSet(np.zeros((0, 3)), np.zeros((0, 3)))

    def __repr__(self) -> str:
        return f"ParticleSet(count={self.count})"


@dataclass
class CyclicBoundary:
    z_min: float
    z_max: float

    def __post_init__(self):
        if not self.z_min < self.z_max:
            raise ValidationError(
                f"cyclic boundary requires z_min < z_max, got [{self.z_min}, {self.z_max}]"
            )


class RigidBody:
    """Kinematically driven body (scene.py:130-166)."""

    def __init__(self, geometry: SdfGeometry, driver: MotionDriver | None = None, name: str = "",
                 spec: dict | None = None):
        self.geometry = geometry
        self.driver = driver or StaticDriver()
        self.name = name
        self.spec = spec
        self.pose = identity_pose()
        self.omega = np.zeros(3)
        self.v_origin = np.zeros(3)
        self.update(0.0)

    def update(self, t: float) -> None:
        self.pose = np.asarray(self.driver.pose_at(t), dtype=np.float64)
        self.omega, self.v_origin = self.driver.twist_at(t)
        self.validate()

    def validate(self) -> None:
        R = self.pose[:3, :3]
        err = rotation_error(R)
        if err > 1e-6 or abs(np.linalg.det(R) - 1.0) > 1e-6:
            raise ValidationError(f"body {self.name!r}: rotation is not orthonormal (residual {err:.3e})")

    def velocity_at(self, points: np.ndarray) -> np.ndarray:
        p = np.atleast_2d(points)
        return self.v_origin + np.cross(self.omega, p - self.pose[:3, 3])


@dataclass
class Scene:
    particles: ParticleSet
    bodies: list
    params: MaterialParams
    boundary: CyclicBoundary | None = None
    t: float = 0.0
    hashmap_size: int | None = None
    chains: dict = field(default_factory=dict)
    seed: int = 0
    config: dict | None = None

    def validate(self) -> None:
        self.params.validate()
        self.particles.validate()
        for body in self.bodies:
            body.validate()


# ---------------------------------------------------------------------------
# Particle seeding (scene.py:192-261) — host-side scene construction.
# ---------------------------------------------------------------------------
@dataclass
class BoxRegion:
    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        self.min = np.asarray(self.min, dtype=np.float64)
        self.max = np.asarray(self.max, dtype=np.float64)
        if not np.all(self.min < self.max):
            raise ValidationError("box region requires min < max componentwise")


@dataclass
class CylinderRegion:
    center: np.ndarray
    radius: float
    z_min: float
    z_max: float

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=np.float64)
        if not (self.radius > 0 and self.z_min < self.z_max):
            raise ValidationError("cylinder region requires radius > 0 and z_min < z_max")


def _lattice_axis(lo: float, hi: float, r: float, spacing: float) -> np.ndarray:
    room = (hi - lo) - 2.0 * r
    if room < -1e-12:
        raise ValidationError("region too small for even one particle of this radius")
    count = int(np.floor(max(room, 0.0) / spacing + 1e-9)) + 1
    first = (lo + hi) / 2.0 - (count - 1) * spacing / 2.0
    return first + spacing * np.arange(count)


def seed_particles_grid(region, r: float, jitter: float = 0.0, rng=None) -> ParticleSet:
    """Cubic-lattice seeding with jitter (scene.py:226-261)."""
    if not 0.0 <= jitter < 1.0:
        raise ValidationError(f"jitter must be in [0, 1), got {jitter}")
    spacing = 2.0 * r + 2.0 * jitter * r * np.sqrt(3.0)
    if isinstance(region, BoxRegion):
        axes = [_lattice_axis(region.min[a], region.max[a], r, spacing) for a in range(3)]
        grid = np.meshgrid(*axes, indexing="ij")
        pts = np.stack(grid, axis=-1).reshape(-1, 3)
    elif isinstance(region, CylinderRegion):
        R = region.radius
        xs = _lattice_axis(region.center[0] - R, region.center[0] + R, r, spacing)
        ys = _lattice_axis(region.center[1] - R, region.center[1] + R, r, spacing)
        zs = _lattice_axis(region.z_min, region.z_max, r, spacing)
        pts = np.stack(np.meshgrid(xs, ys, zs, indexing="ij"), axis=-1).reshape(-1, 3)
        rho = np.hypot(pts[:, 0] - region.center[0], pts[:, 1] - region.center[1])
        pts = pts[rho <= R - r + 1e-12]
        if len(pts) == 0:
            raise ValidationError("region too small for even one particle of this radius")
    else:
        raise ValidationError(f"unknown region type {type(region).__name__}")
    if jitter > 0:
        rng = rng or np.random.default_rng(0)
        pts = pts + rng.uniform(-jitter * r, jitter * r, size=pts.shape)
    return ParticleSet(pts, np.zeros_like(pts))


__all__ = [
    "BoxRegion",
    "CyclicBoundary",
    "CylinderRegion",
    "KinematicChain",
    "MaterialParams",
    "ParticleSet",
    "RigidBody",
    "Scene",
    "ValidationError",
    "seed_particles_grid",
]
