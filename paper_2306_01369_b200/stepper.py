"""``step``/``run`` on the GPU — the drop-in boundary (stepper.py:57-189).

``step(scene, mode, step_index)`` and ``run(scene, n_steps, ...)`` keep the
reference signatures, mutate the scene the same way (``scene.t``, body
poses, particle state) and return ``StepReport`` objects with the same
fields.  The physics runs as the sm_100a kernel schedule in
csrc/gg_kernels.cuh; ``run`` enqueues the whole batch as CUDA-graph
replays and synchronises once.
"""

from __future__ import annotations

import enum
import struct
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import _mode_code, engine_for, raise_status


class PipelineMode(enum.Enum):
    ONE_LOOP = "one-loop"
    TWO_LOOPS_FUSED = "two-loops-fused"
    TWO_LOOPS_SPLIT = "two-loops-split"


@dataclass
class StepReport:
    wall_time: float = 0.0
    n_contacts: int = 0
    n_candidates: int = 0
    candidate_hit_rate: float = 0.0
    max_penetration: float = 0.0
    kinetic_energy: float = 0.0
    n_body_contacts: int = 0
    n_coincident_skipped: int = 0
    n_degenerate_skipped: int = 0
    max_cone_violation: float = 0.0
    min_normal_impulse: float = 0.0
    body_momentum: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    step_index: int = -1


def _make_report(rec, bm: np.ndarray, step_index: int, wall: float) -> StepReport:
    n_pp = int(rec["n_contacts"])
    n_cand = int(rec["n_candidates"])
    mn = float(rec["min_normal_impulse"])
    return StepReport(
        wall_time=wall,
        n_contacts=n_pp,
        n_candidates=n_cand,
        candidate_hit_rate=n_pp / max(n_cand, 1),
        max_penetration=float(rec["max_penetration"]),
        kinetic_energy=float(rec["kinetic_energy"]),
        n_body_contacts=int(rec["n_body_contacts"]),
        n_coincident_skipped=int(rec["n_coincident"]),
        n_degenerate_skipped=int(rec["n_degenerate"]),
        max_cone_violation=float(rec["max_cone_violation"]),
        min_normal_impulse=mn if np.isfinite(mn) else 0.0,
        body_momentum=np.array(bm, dtype=np.float64).reshape(-1, 3),
        step_index=step_index,
    )


def _empty_steps(scene, n_steps: int, indices) -> list[StepReport]:
    """n == 0: the reference still advances time and bodies (stepper.py:65-67)."""
    out = []
    for k in range(n_steps):
        t0 = time.perf_counter()
        scene.t += scene.params.timestep
        for body in scene.bodies:
            body.update(scene.t)
        out.append(StepReport(wall_time=time.perf_counter() - t0,
                              body_momentum=np.zeros((len(scene.bodies), 3)),
                              step_index=indices[k]))
    return out


def advance(scene, n_steps: int, mode=PipelineMode.TWO_LOOPS_SPLIT, first_index: int = -1,
            index_stride: int = 1) -> list[StepReport]:
    """Run n_steps steps as one device batch; step k is labelled
    first_index + k * index_stride in reports and errors."""
    indices = [first_index + k * index_stride for k in range(n_steps)]
    if n_steps == 0:
        return []
    mcode = _mode_code(mode)
    if scene.particles.count == 0:
        return _empty_steps(scene, n_steps, indices)
    t_start = time.perf_counter()
    eng = engine_for(scene)
    eng.prepare(scene)
    t_before = scene.t
    table, ts = eng.body_tables(scene, n_steps)
    nb = len(scene.bodies)
    reps, bm, done, status, msg = eng.run_batch(table, nb, mcode)
    if done:
        eng.finish(scene)
    if status != N.GG_OK:
        # leave time and bodies where the failing step left them
        scene.t = float(ts[done]) if done < n_steps else scene.t
        for body in scene.bodies:
            body.update(scene.t)
        raise_status(status, msg, indices[done] if done < n_steps else indices[-1])
    wall = (time.perf_counter() - t_start) / n_steps
    del t_before
    return [_make_report(reps[k], bm[k], indices[k], wall) for k in range(n_steps)]


def step(scene, mode: PipelineMode = PipelineMode.TWO_LOOPS_SPLIT, step_index: int = -1):
    """Advance the scene by one timestep in place (stepper.py:57-135)."""
    return scene, advance(scene, 1, mode, step_index)[0]


def apply_cyclic_boundary(particles, boundary):
    """Host-side helper kept for API parity (stepper.py:138-144); the device
    applies the same rule inside k_integrate."""
    x = particles.positions
    z = x[:, 2]
    z[z < boundary.z_min] += boundary.z_max - boundary.z_min
    return particles


@dataclass
class Trajectory:
    dt: float
    stride: int
    positions: list = field(default_factory=list)
    velocities: list | None = None

    def record(self, particles) -> None:
        self.positions.append(np.asarray(particles.positions, dtype=np.float32).copy())
        if self.velocities is not None:
            self.velocities.append(np.asarray(particles.velocities, dtype=np.float32).copy())


def run(scene, n_steps: int, mode: PipelineMode = PipelineMode.TWO_LOOPS_SPLIT,
        snapshot_stride: int = 0, record_velocities: bool = False):
    """``step`` n_steps times (stepper.py:162-189), batched on the device
    between snapshots."""
    if n_steps < 0:
        raise ValueError("n_steps must be >= 0")
    traj = Trajectory(dt=scene.params.timestep, stride=snapshot_stride,
                      velocities=[] if record_velocities else None)
    if snapshot_stride > 0:
        traj.record(scene.particles)
    reports: list[StepReport] = []
    chunk = snapshot_stride if snapshot_stride > 0 else max(n_steps, 1)
    k = 0
    while k < n_steps:
        m = min(chunk, n_steps - k)
        reports.extend(advance(scene, m, mode, first_index=k))
        k += m
        if snapshot_stride > 0 and k % snapshot_stride == 0:
            traj.record(scene.particles)
    return traj, reports


# ---------------------------------------------------------------------------
# GTRJ trajectory file (stepper.py:196-239): header + little-endian float32.
# ---------------------------------------------------------------------------
TRAJ_MAGIC = b"GTRJ"
TRAJ_VERSION = 1


def save_trajectory(path: str, traj: Trajectory) -> None:
    n_p = traj.positions[0].shape[0] if traj.positions else 0
    with_v = traj.velocities is not None
    with open(path, "wb") as fh:
        fh.write(TRAJ_MAGIC)
        fh.write(struct.pack("<IIdII", TRAJ_VERSION, n_p, traj.dt, max(traj.stride, 0),
                             int(with_v)))
        for k, pos in enumerate(traj.positions):
            fh.write(np.ascontiguousarray(pos, dtype="<f4").tobytes())
            if with_v:
                fh.write(np.ascontiguousarray(traj.velocities[k], dtype="<f4").tobytes())


def load_trajectory(path: str) -> Trajectory:
    with open(path, "rb") as fh:
        if fh.read(4) != TRAJ_MAGIC:
            raise ValueError(f"{path!r} is not a trajectory file")
        version, n_p, dt, stride, with_v = struct.unpack("<IIdII", fh.read(24))
        if version != TRAJ_VERSION:
            raise ValueError(f"unsupported trajectory version {version}")
        blob = fh.read()
    traj = Trajectory(dt=dt, stride=stride, velocities=[] if with_v else None)
    if n_p == 0:
        return traj
    per = n_p * 3 * (2 if with_v else 1)
    frames = np.frombuffer(blob, dtype="<f4")
    for off in range(0, len(frames) - per + 1, per):
        f = frames[off : off + per]
        traj.positions.append(f[: n_p * 3].reshape(n_p, 3).copy())
        if with_v:
            traj.velocities.append(f[n_p * 3 :].reshape(n_p, 3).copy())
    return traj
