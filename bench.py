#!/usr/bin/env python
"""bench.py — particle-steps/s of the GranularGym timestep on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload hero50k|bed1m]
    python bench.py --impl reference ...        # the reference CPU path (oracle port)

Workloads (BASELINE.json configs):
  hero50k  config 2: 50k settled column bed (floor + tube wall) with the
           ExcavationEnv Box scoop on its 7-joint chain, joints at 0.3 x limits,
           dt = 5e-4, 10 PJA sweeps.  Initial state: bench_data/hero50k_settled.npz
           (settled once on the GPU, shared by both arms), else settled at start.
  bed1m    config 4 scale: lattice_bed(1e6) on a floor with a spinning grid SDF tool.
  slab     config 5: lattice_bed(8e6) on a floor, slab-decomposed along x over the
           N ranks (SlabBed: migration + ghost halo + per-sweep w halo, NCCL P2P);
           total work fixed as N grows ("scaling": "strong").
  envs     config 3: 4096 BulldozerEnv scenes x 2000 particles (r = 0.025), ground
           + blade on TrackSteering drivers with fixed random actions, physics
           substeps only; env e runs on rank e mod N (no communication), so the
           total work is fixed as N grows ("scaling": "strong").

One JSON line on rank 0.  ``value`` is device time (CUDA events per step, L2
flushed by a 512 MB write before every step); ``e2e`` is wall time through
the public ``run()`` API with host state uploaded from pinned memory and the
final state + every step's report read back.  N > 1: independent replicas
(one per GPU, no data-path collective), max time over ranks.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse
import ctypes
import json
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-steps/s at 50k & 1M particles (1/2/4/8 B200); % of HBM roofline"
UNIT = "particle-steps/s"
SETTLED = ROOT / "bench_data" / "hero50k_settled.npz"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hero50k", choices=["hero50k", "bed1m", "envs", "slab"])
    ap.add_argument("--slab-particles", type=int, default=8_000_000)
    ap.add_argument("--envs", type=int, default=4096, help="envs workload: total envs")
    ap.add_argument("--env-particles", type=int, default=2000)
    ap.add_argument("--settle", type=int, default=3000, help="hero50k: settle steps when no state file")
    ap.add_argument("--bed-state", default="",
                    help="bed1m: settled-state cache (.npz): loaded if present, else written after settling")
    ap.add_argument("--settle-bed", type=int, default=8000,
                    help="bed1m: most settle steps (dt 1e-3) before KE/n < 2e-3 J")
    ap.add_argument("--flush-mb", type=int, default=-1,
                    help="L2 flush before every timed step (MB); default: 512 for hero50k "
                         "(its working set fits L2), 0 for the larger beds (inputs > L2)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--solve-mode", type=int, default=0)
    ap.add_argument("--pipeline", default="two-loops-split",
                    choices=["two-loops-split", "two-loops-fused", "one-loop"],
                    help="PipelineMode (loop structure; same results): the paper's Fig. 6 comparison")
    ap.add_argument("--resort-every", type=int, default=8)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None
        if self.world > 1:
            import torch
            import torch.distributed as td

            n_dev = torch.cuda.device_count() if torch.cuda.is_available() else 0
            # one GPU per rank (NCCL); with fewer GPUs than ranks (a plumbing
            # check on a small box) ranks share GPUs round-robin over gloo
            backend = "nccl" if n_dev >= self.world else "gloo"
            if n_dev:
                self.local = self.local % n_dev
                torch.cuda.set_device(self.local)
            td.init_process_group(backend)
            self.pg = td
            self.backend = backend

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def hero_initial_state(args, with_gpu: bool):
    """(x, v, t) of the settled 50k column."""
    if SETTLED.exists():
        z = np.load(SETTLED)
        return z["x"].astype(np.float64), z["v"].astype(np.float64), float(z["t"])
    if not with_gpu:
        return None
    import paper_2306_01369_b200 as gg

    sc = gg.hero_scene(50_000)
    gg.run(sc, args.settle)
    x = sc.particles.positions.astype(np.float32).astype(np.float64)
    v = sc.particles.velocities.astype(np.float32).astype(np.float64)
    return x, v, float(sc.t)


def bed1m_settled(args):
    """SURVEY.md §8d config 4 initial state: lattice_bed(1e6) + floor, settled on
    the GPU at dt = 1e-3 (checked every 250 steps, at most --settle-bed steps)
    until KE / n < 2e-3 J, fp32-rounded.  SURVEY's 1e-3 J is below the PJA
    solver's residual jitter on this pile (KE/n plateaus at ~1.1e-3 J after
    2e4 steps, tools/settle_probe.py); 2e-3 J is the level of the reference's
    own settled acceptance fixture (3.9 J over 2000 particles),
    reached after ~7000 steps with c_pp ~1.45.  Deterministic
    (bitwise-reproducible kernels), so every run starts from the same state."""
    import paper_2306_01369_b200 as gg

    if args.bed_state and os.path.exists(args.bed_state):
        z = np.load(args.bed_state, allow_pickle=False)
        return (z["x"].astype(np.float64), z["v"].astype(np.float64), float(z["t"]),
                json.loads(str(z["settle"])))
    x = gg.lattice_bed(1_000_000).astype(np.float32).astype(np.float64)
    sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                  params=gg.MaterialParams(timestep=1e-3))
    done, ke = 0, float("inf")
    while done < args.settle_bed:
        _, reps = gg.run(sc, 250)
        done += 250
        ke = reps[-1].kinetic_energy / sc.particles.count
        if ke < 2e-3:
            break
    x = sc.particles.positions.astype(np.float32).astype(np.float64)
    v = sc.particles.velocities.astype(np.float32).astype(np.float64)
    info = {"dt": 1e-3, "steps": done, "ke_per_particle_J": ke, "target_J": 2e-3}
    if args.bed_state:
        np.savez(args.bed_state, x=x.astype(np.float32), v=v.astype(np.float32), t=sc.t,
                 settle=json.dumps(info))
    return x, v, float(sc.t), info


def make_scene(args, with_gpu=True):
    import paper_2306_01369_b200 as gg
    from paper_2306_01369_b200.beds import add_scoop
    from paper_2306_01369_b200.meshes import make_box_mesh
    from paper_2306_01369_b200.sdf import bake_mesh_sdf

    if args.workload == "hero50k":
        st = hero_initial_state(args, with_gpu)
        if st is None:
            raise RuntimeError("no settled state file and no GPU to settle one")
        x, v, t = st
        sc = gg.hero_scene(50_000)
        sc.particles = gg.ParticleSet(x, v)
        sc.t = t
        sc.params.timestep = 5e-4
        add_scoop(sc, action=0.3, depth=0.05)
        desc = {"workload": "hero50k", "config": "BASELINE configs[1]: 50k bed + kinematic scoop",
                "n_particles": 50_000, "dt": 5e-4, "solver_iterations": 10,
                "bodies": "floor + tube wall + Box(0.15,0.1,0.04) scoop on 7-joint chain @0.3 limits"}
    else:
        x, v, t, settle = bed1m_settled(args)
        params = gg.MaterialParams(timestep=5e-4)
        verts, faces = make_box_mesh([0.15, 0.1, 0.04])
        grid = bake_mesh_sdf(verts, faces, spacing=0.01)  # on the device (gg_bake_mesh_sdf)
        top = float(np.quantile(x[:, 2], 0.999))
        cx, cy = float(np.median(x[:, 0])), float(np.median(x[:, 1]))
        # the scoop box, spun about the vertical axis with its centre 2 cm under the surface
        tool = gg.RigidBody(grid, gg.SpinDriver(axis=[0, 0, 1], rate=1.0, center=[cx, cy, top],
                                                base_pose=gg.make_pose(np.eye(3), [cx, cy, top - 0.02])),
                            name="tool")
        sc = gg.Scene(particles=gg.ParticleSet(x, v),
                      bodies=[gg.RigidBody(gg.HalfSpace(), name="floor"), tool], params=params)
        sc.t = t
        desc = {"workload": "bed1m",
                "config": "BASELINE configs[3]: lattice_bed(1e6) settled on the GPU + baked mesh tool",
                "n_particles": 1_000_000, "dt": 5e-4, "solver_iterations": 10,
                "bodies": "floor + make_box_mesh([0.15,0.1,0.04]) baked on the device at 1 cm, spinning 1 rad/s",
                "settle": settle}
    return sc, desc


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# byte model and roofline
# ---------------------------------------------------------------------------
def bytes_model(n_h: int, S: int, c_pp: float, c_b: float, fused_split: bool = False) -> dict:
    P = int(np.ceil(np.log2(max(n_h, 2)) / 8))
    # SURVEY.md §8d per-kernel terms mapped onto this schedule
    per_kernel = {
        "k_count": 24.0,                                   # hash: read x, write key + idx
        "k_resort": 68.0,                                  # reorder (every resort_every steps)
        "k_fill": 68.0,                                    # bucket-ordered candidate copy
        # pp narrowphase + body contacts (one kernel: K5 + K6)
        "k_narrow": 20.0 + 20.0 * c_pp + 16.0 + 32.0 * c_b,
        "k_solve": S * (48.0 + 20.0 * c_pp + 32.0 * c_b) + 80.0,  # S sweeps + integrate
    }
    # the small-n schedule: sort + contacts in one persistent kernel, and the
    # solve either in the same kernel or (split) on the 16-CTA cluster
    per_kernel["k_step_fused"] = (per_kernel["k_count"] + 16.0 * 1 + 20.0 + per_kernel["k_fill"]
                                  + per_kernel["k_narrow"]
                                  + (0.0 if fused_split else per_kernel["k_solve"]))
    step = 228.0 + 16.0 * P + 48.0 * S + (S + 1) * (20.0 * c_pp + 32.0 * c_b)
    return {"per_kernel_per_particle": per_kernel, "step_per_particle": step, "radix_passes": P}


def merge_solve_kinds(lib, kind_ms, kind_n):
    """Per-kernel-kind times of gg_profile_steps; the per-sweep launches
    (k_sweep x S + k_finish) are also reported as one logical k_solve per step
    (the byte model's unit), the parts kept for the breakdown."""
    names = [lib.gg_profile_kind_name(k).decode() for k in range(16)]
    ms = {nm: 0.0 for nm in names if nm}
    cnt = {nm: 0 for nm in names if nm}
    for k, nm in enumerate(names):
        if nm:
            ms[nm] += float(kind_ms[k])
            cnt[nm] += int(kind_n[k])
    if cnt.get("k_finish", 0) > 0:
        ms["k_solve"] = ms.get("k_solve", 0.0) + ms["k_sweep"] + ms["k_finish"]
        cnt["k_solve"] = cnt.get("k_solve", 0) + cnt["k_finish"]
    if cnt.get("k_exact", 0) > 0:  # the large-n contact phase runs as k_cand + k_exact
        ms["k_narrow"] = ms.get("k_narrow", 0.0) + ms["k_cand"] + ms["k_exact"]
        cnt["k_narrow"] = cnt.get("k_narrow", 0) + cnt["k_exact"]
    out = [nm for nm in ms if nm != "(unused)"]
    return out, np.array([ms[nm] for nm in out]), np.array([cnt[nm] for nm in out])


def time_shares(names, kind_ms, kind_n) -> dict:
    """Share of the step per kernel kind (k_solve, when it is the sum of the
    per-sweep parts, is reported but not double counted)."""
    parts = "k_finish" in names and kind_n[names.index("k_finish")] > 0
    nparts = "k_exact" in names and kind_n[names.index("k_exact")] > 0
    total = sum(float(kind_ms[k]) for k, nm in enumerate(names)
                if not ((parts and nm == "k_solve") or (nparts and nm == "k_narrow")))
    return {nm: float(kind_ms[k]) / max(total, 1e-9) for k, nm in enumerate(names) if kind_n[k] > 0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        z = json.loads(p.read_text())
        return float(z["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, workload: str):
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    try:
        z = json.loads(f.read_text())
        e = z.get(workload, {}).get(kernel)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU baseline (oracle port on host cores; test infrastructure, timed only)
# ---------------------------------------------------------------------------
class _BodyAt:
    def __init__(self, geometry, pose, omega, v_origin):
        self.geometry, self.pose, self.omega, self.v_origin = geometry, pose, omega, v_origin


def cpu_baseline(sc, x, v, budget_s: float) -> dict:
    from oracle import granular_oracle as O

    params = sc.params
    n = len(x)
    n_h = int(sc.hashmap_size or O.table_size(n))
    t = sc.t
    steps = 0
    t0 = time.perf_counter()
    while True:
        t += params.timestep
        bodies = []
        for b in sc.bodies:
            om, vo = b.driver.twist_at(t)
            bodies.append(_BodyAt(b.geometry, np.asarray(b.driver.pose_at(t), float), om, vo))
        x, v, _, _, _ = O.step(x, v, params, bodies, n_h, sc.boundary)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= 200:
            break
    return {"value": n * steps / el, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{steps} oracle steps of the same workload state ({n} particles), "
                      f"{el:.1f}s, numpy single thread (OPENBLAS_NUM_THREADS=1)"}


# ---------------------------------------------------------------------------
def run_reference(args, dist: Dist):
    """--impl reference: the reference CPU path (oracle port, oracle/_ref absent:
    the reference is Python) on the host, rank 0 only."""
    if dist.rank != 0:
        return
    if args.workload == "envs":
        budget = min(args.cpu_seconds, 60.0)
        cb = envs_cpu_baseline(args, budget)
        n_total = args.envs * args.env_particles
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000.0 * n_total / cb["value"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "envs", "n_envs": args.envs,
                           "n_particles": n_total}, "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    sc, desc = make_scene(args, with_gpu=False)
    x = np.asarray(sc.particles._x, float).copy()
    v = np.asarray(sc.particles._v, float).copy()
    per_step_budget = max(args.cpu_seconds / max(args.steps + args.warmup, 1), 0.5)
    # bounded: warmup W steps and K timed steps are each one oracle step sample
    budget = min(args.cpu_seconds, 60.0)
    cb = cpu_baseline(sc, x, v, budget)
    del per_step_budget
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * desc["n_particles"] / cb["value"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": desc, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def envs_setup(args, dist: Dist, device: int):
    from paper_2306_01369_b200.batch import shard_envs
    from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BulldozerEnvConfig

    mine = shard_envs(args.envs, dist.rank, dist.world)
    cfg = BulldozerEnvConfig(n_particles=args.env_particles, radius=0.025)
    env = BatchedBulldozerEnv(len(mine), cfg, device=device, render=False)  # physics e2e
    env.reset(mine)  # seed = env id
    acts = np.stack([np.random.default_rng(int(e)).uniform(-1, 1, 2) for e in mine])
    acts[:, 0] = np.abs(acts[:, 0])  # drive forward into the bed
    env.driver.command(acts)
    desc = {"workload": "envs", "config": "BASELINE configs[2]: batched bulldozer envs "
            f"{args.envs} x {args.env_particles} particles, sharded env e -> rank e mod N",
            "n_envs": args.envs, "envs_per_rank": len(mine), "n_particles": args.envs * env.batch.n,
            "dt": cfg.timestep, "solver_iterations": 10, "bodies": "ground + Box blade per env"}
    return env, acts, desc


def envs_cpu_baseline(args, budget_s: float) -> dict:
    """Reference algorithm (oracle port) on one env at a time, 1 host core."""
    from oracle import granular_oracle as O
    from paper_2306_01369_b200.envs import BulldozerEnvConfig, bulldozer_scene

    cfg = BulldozerEnvConfig(n_particles=args.env_particles, radius=0.025)
    sc = bulldozer_scene(0, cfg)
    x = sc.particles.positions.astype(np.float32).astype(np.float64)
    v = np.zeros_like(x)
    drv = sc.bodies[1].driver
    drv.command(np.array([0.8, 0.1]))
    steps, t = 0, 0.0
    t0 = time.perf_counter()
    while True:
        t += cfg.timestep
        drv.advance(cfg.timestep)
        bodies = []
        for b in sc.bodies:
            om, vo = b.driver.twist_at(t)
            bodies.append(_BodyAt(b.geometry, np.asarray(b.driver.pose_at(t), float), om, vo))
        x, v, _, _, _ = O.step(x, v, sc.params, bodies, O.table_size(len(x)))
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= 2000:
            break
    n = len(x)
    return {"value": n * steps / el, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{steps} oracle steps of env 0 ({n} particles) from its seeded bed, "
                      f"{el:.1f}s, numpy single thread; per-env work is independent, so the "
                      f"{args.envs}-env batch scales with host cores at best"}


def run_envs(args, dist: Dist):
    from paper_2306_01369_b200 import _native as N

    dev = dist.local
    env, acts, desc = envs_setup(args, dist, dev)
    batch = env.batch
    lib = N.lib()
    # settle: the seeded bed falls onto the floor before the blade arrives
    batch.run_raw(100)
    K, W = args.steps, args.warmup
    if W:
        batch.run_raw(W)
    chunk = 25
    step_ms = np.zeros(K, dtype=np.float32)
    l0 = batch.kernel_launches()
    clocks = Clocks(dev)
    clocks.start()
    dist.barrier()
    done = 0
    reps_all = []
    while done < K:
        m = min(chunk, K - done)
        table = batch.body_tables(m)
        st = lib.gg_bench_steps(batch.ctx, m, N.ptr(np.ascontiguousarray(table)), batch.nb,
                                args.flush_mb << 20, N.ptr(step_ms[done:]))
        N.check(batch.ctx, st, "gg_bench_steps")
        rbuf = np.zeros((m, batch.E), dtype=N.REPORT_DTYPE)
        bbuf = np.zeros((m, batch.E, batch.nb, 3))
        nd, es = ctypes.c_int32(0), ctypes.c_int32(-1)
        st = lib.gg_sync(batch.ctx, N.ptr(rbuf), N.ptr(bbuf), m, ctypes.byref(nd), ctypes.byref(es))
        if st != N.GG_OK or nd.value != m:
            raise RuntimeError(f"envs bench failed: {st} {N.last_error(batch.ctx)}")
        reps_all.append(rbuf)
        done += m
    dist.barrier()
    clk = clocks.stop()
    launches = batch.kernel_launches() - l0
    t_ms = dist.max(float(step_ms.sum()))
    n_total = args.envs * batch.n
    value = n_total * K / (t_ms / 1000.0)
    reps = np.concatenate(reps_all)
    n_local = batch.E * batch.n
    c_pp = float(reps["n_contacts"].sum(axis=1).mean()) / n_local
    c_b = float(reps["n_body_contacts"].sum(axis=1).mean()) / n_local

    # per-kernel roofline pass
    peak, peak_src = peaks()
    P = max(min(args.profile_steps, 10), 1)
    table3 = batch.body_tables(P)
    kind_ms = np.zeros(16, dtype=np.float32)
    kind_n = np.zeros(16, dtype=np.int32)
    st = lib.gg_profile_steps(batch.ctx, P, N.ptr(np.ascontiguousarray(table3)), batch.nb,
                              N.ptr(kind_ms), N.ptr(kind_n))
    N.check(batch.ctx, st, "gg_profile_steps")
    names, kind_ms, kind_n = merge_solve_kinds(lib, kind_ms, kind_n)
    model = bytes_model(batch.n_h, 10, c_pp, c_b)
    share = time_shares(names, kind_ms, kind_n)
    top = max((k for k in range(len(names))
               if names[k] in model["per_kernel_per_particle"] and kind_n[k] > 0),
              key=lambda k: kind_ms[k])
    avg_ms = float(kind_ms[top] / max(kind_n[top], 1))
    bytes_launch = model["per_kernel_per_particle"][names[top]] * n_local
    achieved = bytes_launch / (avg_ms / 1000.0) / 1e9
    roofline = {"bound": "hbm", "kernel": names[top], "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(names[top], "envs"),
                "algorithmic_bytes_per_launch": bytes_launch, "avg_launch_ms": avg_ms,
                "peak_source": peak_src, "kernel_time_share": share,
                "step_bytes_per_particle": model["step_per_particle"],
                "step_frac": (value / dist.world) * model["step_per_particle"] / (peak * 1e9)}

    # e2e through the public env API: actions in, rewards out, frame_skip substeps per call
    fs = env.config.frame_skip
    n_ctrl = max(K // fs, 1)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n_ctrl):
        _, rew, _, info = env.step(acts)
        _ = float(rew.sum())
    t_e2e = dist.max(time.perf_counter() - t0)
    e2e = {"value": n_total * n_ctrl * fs / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": batch.E * batch.nb * N.BODY_DTYPE.itemsize,
           "d2h_bytes_per_step": batch.E * N.REPORT_DTYPE.itemsize
           + (batch.E * (8 + 8) + batch.E * batch.nb * 24) / fs,
           "api": "BatchedBulldozerEnv.step(actions): per-env blade kinematics, body tables "
                  "uploaded, frame_skip substeps, per-env StepReports and on-device rewards read back",
           "wall_s": t_e2e}
    cb = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cb = envs_cpu_baseline(args, args.cpu_seconds)
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
            "warmup": W, "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 state / f64 contact geometry",
            "data": "synthetic (seeded bulldozer beds, settled 100 substeps)",
            "config": {**desc, "parallelism": f"env shards x{dist.world}",
                       "l2": l2_note(args, batch.E * batch.n * 200 / 2**20),
                       "c_pp": c_pp, "c_b": c_b, "n_h_per_env": batch.n_h},
            "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    env.close()


def lattice_cpu_baseline(n_sample: int, budget_s: float, note: str) -> dict:
    """Reference algorithm (oracle port) on a lattice bed of n_sample
    particles with a floor, 1 host core, bounded by budget_s."""
    import paper_2306_01369_b200 as gg
    from oracle import granular_oracle as O

    x = gg.lattice_bed(n_sample).astype(np.float32).astype(np.float64)
    v = np.zeros_like(x)
    params = gg.MaterialParams(timestep=5e-4)
    floor = _BodyAt(gg.HalfSpace(), np.eye(4), np.zeros(3), np.zeros(3))
    steps = 0
    t0 = time.perf_counter()
    while True:
        x, v, _, _, _ = O.step(x, v, params, [floor], O.table_size(n_sample))
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= 200:
            break
    return {"value": n_sample * steps / el, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{steps} oracle steps of lattice_bed({n_sample}) + floor from the lattice "
                      f"start, {el:.1f}s, numpy single thread; {note}"}


def run_slab(args, dist: Dist):
    import paper_2306_01369_b200 as gg
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.slab import SlabBed

    import torch

    dev = dist.local
    n = args.slab_particles
    x = gg.lattice_bed(n).astype(np.float32).astype(np.float64)
    sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                  params=gg.MaterialParams(timestep=5e-4))
    bed = SlabBed(sc, rank=dist.rank, world=dist.world, device=dev,
                  backend=dist.backend if dist.world > 1 else None)
    lib = N.lib()
    K, W = args.steps, args.warmup
    for _ in range(W):
        bed.step()
    stream = torch.cuda.ExternalStream(lib.gg_stream(bed.ctx), device=torch.device("cuda", dev))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = int(lib.gg_kernel_launches(bed.ctx))
    clocks = Clocks(dev)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    reps = [bed.step() for _ in range(K)]
    e1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clk = clocks.stop()
    launches = int(lib.gg_kernel_launches(bed.ctx)) - l0
    t_ms = dist.max(float(e0.elapsed_time(e1)))
    value = n * K / (t_ms / 1000.0)
    c_pp = float(np.mean([r.n_contacts for r in reps])) / n
    c_b = float(np.mean([r.n_body_contacts for r in reps])) / n
    peak, peak_src = peaks()
    model = bytes_model(bed.n_h, 10, c_pp, c_b)
    owned = dist.max(float(bed.n_owned))
    roofline = {"bound": "hbm", "kernel": "step (slab)", "achieved": (value / dist.world) *
                model["step_per_particle"] / 1e9, "peak": peak, "unit": "GB/s",
                "frac": (value / dist.world) * model["step_per_particle"] / (peak * 1e9),
                "traffic": None, "peak_source": peak_src,
                "step_bytes_per_particle": model["step_per_particle"],
                "note": "whole-step byte model per GPU (SURVEY.md §8d); per-kernel fractions "
                        "are those of bed1m/envs (same kernels)"}
    bed.close()
    # e2e through the public API from host buffers: partition + upload
    # (SlabBed), K steps, gather of the global state back to the host
    dist.barrier()
    t0 = time.perf_counter()
    sc2 = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)),
                   bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                   params=gg.MaterialParams(timestep=5e-4))
    bed2 = SlabBed(sc2, rank=dist.rank, world=dist.world, device=dev,
                   backend=dist.backend if dist.world > 1 else None)
    for _ in range(K):
        bed2.step()
    Xg, _ = bed2.gather()
    _ = float(Xg[0, 0])
    t_e2e = dist.max(time.perf_counter() - t0)
    bed2.close()
    e2e = {"value": n * K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 48 * n / max(K, 1),
           "d2h_bytes_per_step": 52 * n / max(K, 1), "wall_s": t_e2e,
           "api": "SlabBed(scene) (partition + upload of the host state), K x SlabBed.step(), "
                  "SlabBed.gather() (global state back on the host)"}
    cb = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cb = lattice_cpu_baseline(100_000, args.cpu_seconds,
                                  "the oracle is O(n): particle-steps/s carries over to 8M")
    if dist.rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
                "warmup": W, "ms_per_step": t_ms / K, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 state / f64 contact geometry", "data": "synthetic (lattice bed)",
                "config": {"workload": "slab", "config": "BASELINE configs[4]: 8M bed, slab "
                           "decomposition over N GPUs", "n_particles": n, "dt": 5e-4,
                           "solver_iterations": 10, "parallelism": f"slabs x{dist.world}",
                           "n_h": bed.n_h, "c_pp": c_pp, "c_b": c_b, "max_owned": owned,
                           "l2": "state (>1 GB) exceeds L2"},
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "clocks": clk, "gpu_launches": launches}
        print(json.dumps(line), flush=True)


def run_ours(args, dist: Dist):
    import paper_2306_01369_b200 as gg
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.engine import engine_for

    dev = dist.local
    os.environ.setdefault("CUDA_VISIBLE_DEVICES", os.environ.get("CUDA_VISIBLE_DEVICES", ""))
    sc, desc = make_scene(args)
    n = sc.particles.count
    eng = engine_for(sc)
    eng.device = dev
    eng.prepare(sc)
    N.check(eng.ctx, N.lib().gg_set_solve_mode(eng.ctx, args.solve_mode), "solve mode")
    N.check(eng.ctx, N.lib().gg_set_resort_every(eng.ctx, args.resort_every), "resort")
    nb = len(sc.bodies)
    K, W = args.steps, args.warmup
    table, _ = eng.body_tables(sc, W + K)
    # warm-up (untimed)
    pmode = {"two-loops-split": 0, "two-loops-fused": 1, "one-loop": 2}[args.pipeline]
    if W:
        reps, _, done, st, msg = eng.run_batch(table[:W], nb, pmode)
        if st:
            raise RuntimeError(msg)
    lib = N.lib()
    rows = np.ascontiguousarray(table[W:])
    step_ms = np.zeros(K, dtype=np.float32)
    l0 = eng.kernel_launches()
    clocks = Clocks(dev)
    clocks.start()
    dist.barrier()
    st = lib.gg_bench_steps(eng.ctx, K, N.ptr(rows), nb, args.flush_mb << 20, N.ptr(step_ms))
    N.check(eng.ctx, st, "gg_bench_steps")
    dist.barrier()
    clk = clocks.stop()
    launches = eng.kernel_launches() - l0
    rbuf = np.zeros(K, dtype=N.REPORT_DTYPE)
    bbuf = np.zeros((K, max(nb, 1), 3))
    nd, es = ctypes.c_int32(0), ctypes.c_int32(-1)
    st = lib.gg_sync(eng.ctx, N.ptr(rbuf), N.ptr(bbuf), K, ctypes.byref(nd), ctypes.byref(es))
    if st != N.GG_OK or nd.value != K:
        raise RuntimeError(f"bench steps failed: status {st} {N.last_error(eng.ctx)}")
    eng.device_newer = True
    t_ms = dist.max(float(step_ms.sum()))
    value = n * K * dist.world / (t_ms / 1000.0)
    c_pp = float(rbuf["n_contacts"].mean()) / n
    c_b = float(rbuf["n_body_contacts"].mean()) / n

    # warm (no flush) steady-state loop, for context
    table2, _ = eng.body_tables(sc, K)
    t_warm = None
    reps, _, done, st2, _ = eng.run_batch(table2, nb, pmode)
    if st2 == 0:
        t_warm = eng.last_batch_ms()

    # per-kernel roofline pass (same schedule, event after every kernel)
    peak, peak_src = peaks()
    P = max(args.profile_steps, 1)
    table3, _ = eng.body_tables(sc, P)
    kind_ms = np.zeros(16, dtype=np.float32)
    kind_n = np.zeros(16, dtype=np.int32)
    st = lib.gg_profile_steps(eng.ctx, P, N.ptr(np.ascontiguousarray(table3)), nb, N.ptr(kind_ms),
                              N.ptr(kind_n))
    N.check(eng.ctx, st, "gg_profile_steps")
    names, kind_ms, kind_n = merge_solve_kinds(lib, kind_ms, kind_n)
    split = "k_step_fused" in names and "k_solve" in names and kind_n[names.index("k_solve")] > 0
    model = bytes_model(eng.n_h, sc.params.solver_iterations, c_pp, c_b, fused_split=split)
    share = time_shares(names, kind_ms, kind_n)
    top = max((k for k in range(len(names))
               if names[k] in model["per_kernel_per_particle"] and kind_n[k] > 0),
              key=lambda k: kind_ms[k])
    top_name = names[top]
    avg_ms = float(kind_ms[top] / max(kind_n[top], 1))
    bytes_launch = model["per_kernel_per_particle"][top_name] * n
    achieved = bytes_launch / (avg_ms / 1000.0) / 1e9
    step_bytes = model["step_per_particle"] * n
    roofline = {"bound": "hbm", "kernel": top_name, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(top_name, desc["workload"]),
                "algorithmic_bytes_per_launch": bytes_launch, "avg_launch_ms": avg_ms,
                "peak_source": peak_src, "kernel_time_share": share,
                "step_bytes_per_particle": model["step_per_particle"],
                "step_frac": (value / dist.world) * model["step_per_particle"] / (peak * 1e9)}

    # e2e through the public API: pinned host state -> run(K) -> reports + state back
    x_host = sc.particles.positions.copy()
    v_host = sc.particles.velocities.copy()
    sc2 = sc
    sc2.particles = gg.ParticleSet(x_host, v_host)
    px, pv = sc2.particles._x, sc2.particles._v
    lib.gg_host_register(N.ptr(px), px.nbytes)
    lib.gg_host_register(N.ptr(pv), pv.nbytes)
    dist.barrier()
    t0 = time.perf_counter()
    _, reports = gg.run(sc2, K, mode=gg.PipelineMode(args.pipeline))
    xf = sc2.particles.positions  # device -> host
    _ = float(xf[0, 0]) + sum(r.kinetic_energy for r in reports)
    t_e2e = dist.max(time.perf_counter() - t0)
    lib.gg_host_unregister(N.ptr(px))
    lib.gg_host_unregister(N.ptr(pv))
    e2e = {"value": n * K * dist.world / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": (2 * 24 * n) / K + 240 * nb,
           "d2h_bytes_per_step": (2 * 24 * n) / K + 72 + 24 * nb,
           "api": "paper_2306_01369_b200.run(scene, K): host state upload, per-step body "
                  "tables, all StepReports and the final state read back",
           "wall_s": t_e2e}

    cb = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        x0 = np.asarray(sc.particles.positions, float).copy()
        v0 = np.asarray(sc.particles.velocities, float).copy()
        cb = cpu_baseline(sc, x0, v0, args.cpu_seconds)

    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
            "warmup": W, "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 state / f64 contact geometry",
            "data": ("synthetic (50k column bed settled on the GPU, bench_data/hero50k_settled.npz)"
                     if args.workload == "hero50k" else
                     "synthetic (lattice_bed(1e6) settled on the GPU before the run)"),
            "config": {**desc, "parallelism": f"replicas x{dist.world}" if dist.world > 1 else "single",
                       "pipeline": args.pipeline,
                       "l2": l2_note(args, n * 200 / 2**20),
                       "c_pp": c_pp, "c_b": c_b, "n_h": eng.n_h,
                       "warm_ms_per_step": None if t_warm is None else t_warm / K},
            "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)


def l2_note(args, working_set_mb: float) -> str:
    if args.flush_mb > 0:
        return f"flushed before every timed step ({args.flush_mb} MB write)"
    return (f"not flushed: the step's working set (~{working_set_mb:.0f} MB) is larger than the "
            f"126 MB L2")


def main():
    args = parse()
    if args.flush_mb < 0:
        args.flush_mb = 512 if args.workload == "hero50k" else 0
    dist = Dist()
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif args.workload == "envs":
            run_envs(args, dist)
        elif args.workload == "slab":
            run_slab(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
