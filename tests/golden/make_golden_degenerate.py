"""Golden fixture with degenerate SDF gradients (sdf.py:19, 472-512): particles
exactly at sphere centres and on a capped cylinder's axis penetrate with a zero
gradient, so the reference drops the contact and counts it in n_degenerate.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \\
        python tests/golden/make_golden_degenerate.py

Writes tests/golden/degenerate.npz and adds it to cases.json.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as mg  # noqa: E402  (the reference harness: one_step_case)
from granusim import sdf as rsdf  # noqa: E402
from granusim.kinematics import StaticDriver, make_pose  # noqa: E402
from granusim.scene import MaterialParams, RigidBody  # noqa: E402

OUT = Path(__file__).resolve().parent
rng = np.random.default_rng(21)
centres = mg.f32(np.array([[0.1, 0.2, 0.3], [-0.25, 0.0, 0.35], [0.3, -0.3, 0.5]]))
x = rng.uniform([-0.5, -0.5, 0.0], [0.5, 0.5, 0.7], size=(600, 3))
x[:3] = centres                      # at the sphere centres: zero gradient
x[3] = mg.f32(np.array([0.0, 0.3, 0.2]))  # on the cylinder axis at its centre
bodies = [RigidBody(rsdf.Sphere(0.08), StaticDriver(make_pose(np.eye(3), c)), name=f"ball{i}")
          for i, c in enumerate(centres)]
bodies.append(RigidBody(rsdf.Cylinder(0.07, 0.1), StaticDriver(make_pose(np.eye(3), x[3])), name="cyl"))
bodies.append(RigidBody(rsdf.HalfSpace(), StaticDriver(), name="floor"))
name = mg.one_step_case("degenerate", x, np.zeros_like(x), MaterialParams(), bodies)
g = np.load(OUT / f"{name}.npz")
print(name, "n_degenerate", int(g["rep_n_degenerate"]), "body contacts", int(g["rep_n_body_contacts"]))
cases = json.loads((OUT / "cases.json").read_text())
if name not in cases:
    cases.insert(len(cases) - 1, name)  # before config1_run (a run, not a one-step case)
    (OUT / "cases.json").write_text(json.dumps(cases, indent=1))
