"""bench.py plumbing on CPU: argument parsing, the hero50k scene from the
committed settled state, the byte model and the reference arm's JSON line
(oracle port, tiny sample)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_hero_scene_from_settled_state():
    class A:
        workload = "hero50k"
        settle = 0

    sc, desc = bench.make_scene(A, with_gpu=False)
    assert sc.particles.count == 50_000 and desc["workload"] == "hero50k"
    assert np.isfinite(sc.particles.positions).all()
    assert len(sc.bodies) >= 3  # floor, wall, scoop


def test_bytes_model_matches_survey_formula():
    m = bench.bytes_model(n_h=1 << 21, S=10, c_pp=5.3, c_b=0.0)
    # B = 228 + 16P + 48S + (S+1)(20 c_pp + 32 c_b), P = 3
    assert m["radix_passes"] == 3
    assert abs(m["step_per_particle"] - (228 + 48 + 480 + 11 * 20 * 5.3)) < 1e-9


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-seconds", "0.5"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "particle-steps/s"
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port"
