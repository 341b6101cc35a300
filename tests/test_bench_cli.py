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


def test_bed1m_scene_from_committed_state():
    """The default workload (config 4): the committed settled pile with the
    bucket 1 m into its flank, built without a GPU (both arms use it)."""
    class A:
        workload = "bed1m"

    sc, desc = bench.make_scene(A, with_gpu=False)
    assert sc.particles.count == 1_000_000 and desc["workload"] == "bed1m"
    assert [b.name for b in sc.bodies] == ["floor", "bucket"]
    x = sc.particles.positions
    pose = np.asarray(sc.bodies[1].driver.pose_at(sc.t))
    local = (x - pose[:3, 3]) @ pose[:3, :3]
    inside = (np.abs(local) < [0.7, 1.3, 0.7]).all(axis=1)
    assert inside.sum() > 1000  # the bucket is working in the pile


def test_workload_sample_is_bounded_and_near_the_tool():
    class A:
        workload = "bed1m"

    sc, _ = bench.make_scene(A, with_gpu=False)
    x, v = sc.particles._x, sc.particles._v
    xs, vs, what = bench.workload_sample(sc, x, v, 5000)
    assert xs.shape == (5000, 3) and "tool" in what
    c = np.asarray(sc.bodies[-1].driver.pose_at(sc.t))[:3, 3]
    assert np.abs(xs - c).max() < 3.0


def test_bytes_model_matches_survey_formula():
    m = bench.bytes_model(n_h=1 << 21, S=10, c_pp=5.3, c_b=0.0)
    # B = 228 + 16P + 48S + (S+1)(20 c_pp + 32 c_b), P = 3
    assert m["radix_passes"] == 3
    assert abs(m["step_per_particle"] - (228 + 48 + 480 + 11 * 20 * 5.3)) < 1e-9


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                          "--ref-seconds", "0.3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "particle-steps/s"
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["host_cores"] >= 1
    assert line["steps"] == 2 and line["warmup"] == 1 and line["config"]["workload"] == "bed1m"


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["--workload", "hero50k", "--steps", "3", "--warmup", "3", "--cpu-seconds", "0.5", "--profile-steps", "1"],
    ["--workload", "bed1m", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--profile-steps", "1"],
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


@pytest.mark.gpu
def test_both_arms_print_the_same_config():
    """The driver compares the arms' config dicts: run-specific details live
    under "run", so config is identical."""
    ours = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                           "--profile-steps", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    ref = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3",
                          "--ref-seconds", "0.3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert ours.returncode == 0 and ref.returncode == 0, (ours.stderr[-2000:], ref.stderr[-2000:])
    a = json.loads(ours.stdout.strip().splitlines()[-1])
    b = json.loads(ref.stdout.strip().splitlines()[-1])
    assert a["config"] == b["config"] and a["metric"] == b["metric"] and a["unit"] == b["unit"]


def test_roofline_traffic_resolves_for_each_top_kernel():
    """roofline.traffic comes from the committed profiles/ncu_summary.json;
    kernel names there are normalised (templated kernels included) so the
    lookup the bench line makes finds a number for every top kernel."""
    for kernel, wl in (("k_solve", "bed1m"), ("k_solve", "envs"), ("k_step_fused", "hero50k")):
        t = bench.ncu_traffic(kernel, wl)
        assert t is not None and t > 0, (kernel, wl)
