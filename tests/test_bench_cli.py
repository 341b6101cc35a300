"""bench.py plumbing on CPU: argument parsing, the hero50k scene from the
committed settled state, the byte model and the reference arm's JSON line
(oracle port, tiny sample)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

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


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["--workload", "hero50k", "--steps", "3", "--warmup", "3", "--cpu-seconds", "0.5", "--profile-steps", "1"],
    ["--workload", "bed1m", "--steps", "3", "--warmup", "3", "--settle-bed", "250", "--no-cpu-baseline",
     "--profile-steps", "1"],
    ["--workload", "envs", "--envs", "16", "--steps", "20", "--warmup", "3", "--no-cpu-baseline",
     "--profile-steps", "1"],
    ["--workload", "slab", "--slab-particles", "100000", "--steps", "3", "--warmup", "3",
     "--no-cpu-baseline"],
], ids=["hero50k", "bed1m", "envs", "slab"])
def test_bench_line_contract(args):
    """Every workload prints ONE JSON line with the contract's keys (GPU)."""
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks",
                "gpu_launches"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["peak"] > 0 and 0 < d["roofline"]["frac"] < 1
