"""Shared test helpers: golden-fixture loading and scene construction."""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from paper_2306_01369_b200 import sdf as gsdf
from paper_2306_01369_b200.kinematics import MotionDriver
from paper_2306_01369_b200.scene import CyclicBoundary, MaterialParams, ParticleSet, RigidBody, Scene

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden_cases() -> list[str]:
    names = json.loads((GOLDEN / "cases.json").read_text())
    return [n for n in names if n not in ("hash_kats", "config1_run")]


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@dataclass
class FixedTwistDriver(MotionDriver):
    """Pose/twist frozen at recorded values (the body state the reference
    step saw at t + dt)."""

    pose: np.ndarray
    omega: np.ndarray
    v_origin: np.ndarray

    def pose_at(self, t):
        return self.pose

    def twist_at(self, t):
        return self.omega.copy(), self.v_origin.copy()


@dataclass
class BodyState:
    geometry: object
    pose: np.ndarray
    omega: np.ndarray
    v_origin: np.ndarray


def geometry_from(g: dict, i: int):
    kind = str(g[f"body{i}_kind"])
    if kind == "Sphere":
        return gsdf.Sphere(float(g[f"body{i}_radius"]))
    if kind == "HalfSpace":
        hs = gsdf.HalfSpace(offset=float(g[f"body{i}_offset"]))
        hs.normal = np.array(g[f"body{i}_normal"], dtype=np.float64)  # already unit: keep bits
        return hs
    if kind == "Box":
        return gsdf.Box(g[f"body{i}_half_extents"])
    if kind == "Cylinder":
        return gsdf.Cylinder(float(g[f"body{i}_radius"]), float(g[f"body{i}_half_height"]))
    if kind == "Tube":
        return gsdf.Tube(float(g[f"body{i}_radius"]))
    if kind == "SdfGrid":
        return gsdf.SdfGrid(g[f"body{i}_origin"], g[f"body{i}_spacing"], g[f"body{i}_dims"],
                            g[f"body{i}_values"])
    raise ValueError(kind)


def body_states(g: dict) -> list[BodyState]:
    return [
        BodyState(geometry_from(g, i), g[f"body{i}_pose"], g[f"body{i}_omega"], g[f"body{i}_v_origin"])
        for i in range(int(g["n_bodies"]))
    ]


def params_from(g: dict) -> MaterialParams:
    return MaterialParams(radius=float(g["radius"]), particle_mass=float(g["mass"]),
                          friction=float(g["friction"]), baumgarte_alpha=float(g["alpha"]),
                          timestep=float(g["dt"]), solver_iterations=int(g["iters"]),
                          gravity=g["gravity"], gamma=float(g["gamma"]))


def boundary_from(g: dict):
    return CyclicBoundary(float(g["z_min"]), float(g["z_max"])) if bool(g["has_boundary"]) else None


def scene_from(g: dict) -> Scene:
    """Our Scene for a golden case, bodies frozen at the recorded post-update state."""
    bodies = [
        RigidBody(b.geometry, FixedTwistDriver(b.pose, b.omega, b.v_origin), name=f"b{i}")
        for i, b in enumerate(body_states(g))
    ]
    return Scene(particles=ParticleSet(g["x0"].copy(), g["v0"].copy()), bodies=bodies,
                 params=params_from(g), boundary=boundary_from(g), t=float(g["t0"]),
                 hashmap_size=int(g["n_h"]))


def rel_err(a: np.ndarray, b: np.ndarray) -> float:
    """max|a - b| / max(1, max|b|) — the normalisation of test_acceptance.py:206-207."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max())))


def directed_rows(owner, kind, other) -> np.ndarray:
    rows = np.stack([np.asarray(owner), np.asarray(kind), np.asarray(other)], axis=1).astype(np.int64)
    if len(rows) == 0:
        return rows.reshape(0, 3)
    return rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]
