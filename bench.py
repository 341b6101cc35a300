#!/usr/bin/env python
"""bench.py — particle-steps/s of the GranularGym timestep on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload bed1m|hero50k|envs|slab]
    python bench.py --impl reference ...        # the reference CPU path (oracle port)

Workloads (BASELINE.json configs):
  bed1m    DEFAULT, config 4 and the north_star workload (a 1M-particle bed with
           a scoop): lattice_bed(1e6) + floor settled on the GPU, then an
           excavator bucket (make_bucket_mesh, 2.4 x 1.2 x 1.2 m, baked to an SDF
           grid) driving into the pile's flank at 1 m/s; dt = 5e-4, 10 PJA
           sweeps.  Initial state and baked grid: bench_data/bed1m_settled.npz,
           bench_data/bucket1m_grid.npz (tools/make_bed1m.py), shared by both
           arms.  N > 1: the SAME bed slab-decomposed over the N ranks
           (SlabBed: migration + ghost halo + per-sweep w halo), "scaling":
           "strong"; --replicas runs N independent copies instead.
  hero50k  config 2: 50k settled column bed (floor + tube wall) with the
           ExcavationEnv Box scoop on its 7-joint chain, joints at 0.3 x limits.
           Initial state: bench_data/hero50k_settled.npz.
  envs     config 3: 4096 BulldozerEnv scenes x 2000 particles (r = 0.025),
           sharded env e -> rank e mod N with no communication ("strong").
  slab     config 5: lattice_bed(8e6) on a floor, slab-decomposed over N ranks.

--gpus N without torchrun re-launches itself under torch.distributed.run
with N processes (one per GPU, NCCL, NCCL_DEBUG=INFO).  One JSON line on
rank 0.  ``value`` is device time (CUDA events per step); ``e2e`` is wall time
through the public ``run()`` API with host state uploaded from pinned memory
and the final state + every step's report read back.
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
BED1M = ROOT / "bench_data" / "bed1m_settled.npz"
BUCKET1M = ROOT / "bench_data" / "bucket1m_grid.npz"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bed1m", choices=["bed1m", "hero50k", "envs", "slab"])
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent copies of the scene per GPU instead of one slab-decomposed bed")
    ap.add_argument("--slab-particles", type=int, default=8_000_000)
    ap.add_argument("--halo", choices=["auto", "host", "p2p"], default="auto",
                    help="N > 1 single-bed exchange: peer-memory mailboxes (p2p; auto under NCCL) "
                         "or torch.distributed point-to-point (host)")
    ap.add_argument("--envs", type=int, default=4096, help="envs workload: total envs")
    ap.add_argument("--env-particles", type=int, default=2000)
    ap.add_argument("--settle", type=int, default=3000, help="hero50k: settle steps when no state file")
    ap.add_argument("--flush-mb", type=int, default=-1,
                    help="L2 flush before every timed step (MB); default: 512 for hero50k "
                         "(its working set fits L2), 0 for the larger beds (inputs > L2)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="our arm's cpu_baseline leg: CPU time budget (s)")
    ap.add_argument("--ref-seconds", type=float, default=90.0,
                    help="--impl reference: CPU time budget of the W + K sampled steps (s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--solve-mode", type=int, default=0)
    ap.add_argument("--pipeline", default="two-loops-split",
                    choices=["two-loops-split", "two-loops-fused", "one-loop"],
                    help="PipelineMode (loop structure; same results): the paper's Fig. 6 comparison")
    ap.add_argument("--resort-every", type=int, default=32)
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


def bed1m_state():
    """Config-4 initial state (tools/make_bed1m.py): the settled 1M pile with
    the bucket 1 m into its flank; positions float32, velocities float16,
    both upcast to float64 (the same input for both arms)."""
    if not BED1M.exists() or not BUCKET1M.exists():
        raise RuntimeError(f"{BED1M} / {BUCKET1M} missing: run tools/make_bed1m.py on a GPU")
    z = np.load(BED1M, allow_pickle=False)
    x = z["x"].astype(np.float64)
    v = z["v"].astype(np.float64)
    return x, v, float(z["t"]), json.loads(str(z["settle"])), json.loads(str(z["dig"]))


def bucket1m_grid():
    import paper_2306_01369_b200 as gg

    g = np.load(BUCKET1M, allow_pickle=False)
    return gg.SdfGrid(g["origin"], g["spacing"], g["dims"], g["values"], bytes(g["mesh_hash"]))


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
        from paper_2306_01369_b200.beds import DigDriver

        x, v, t, settle, dig = bed1m_state()
        params = gg.MaterialParams(timestep=5e-4)
        bucket = gg.RigidBody(bucket1m_grid(), DigDriver(**dig), name="bucket")
        sc = gg.Scene(particles=gg.ParticleSet(x, v),
                      bodies=[gg.RigidBody(gg.HalfSpace(), name="floor"), bucket], params=params)
        sc.t = t
        desc = {"workload": "bed1m",
                "config": "BASELINE configs[3] (north_star): 1M-particle excavation bed + mesh/SDF tool",
                "n_particles": 1_000_000, "dt": 5e-4, "solver_iterations": 10,
                "bodies": "floor + excavator bucket (make_bucket_mesh, 2.4 x 1.2 x 1.2 m, 15 cm walls, "
                          "baked on the device at 5 cm) driving into the pile flank at 1 m/s",
                "initial_state": "bench_data/bed1m_settled.npz: lattice_bed(1e6) settled on the GPU "
                                 f"({settle['steps']} steps at dt 1e-3, KE/n {settle['ke_per_particle_J']:.2g} J), "
                                 "then 1 s of the bucket's pass"}
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


ORACLE_RATE = 1.3e5  # oracle particle-steps/s on one host core (measured on the GPU box, round 1)


def bodies_at(sc, t: float) -> list:
    out = []
    for b in sc.bodies:
        om, vo = b.driver.twist_at(t)
        out.append(_BodyAt(b.geometry, np.asarray(b.driver.pose_at(t), float), om, vo))
    return out


def workload_sample(sc, x, v, n_sample: int):
    """A bounded sample of the workload state: the n_sample particles nearest
    the tool (the last body; the bed centre when there is only a floor), in
    user order — the part of the bed where the tool works."""
    n = len(x)
    if n_sample >= n:
        return x, v, "the whole state"
    if len(sc.bodies) > 1:
        c = np.asarray(sc.bodies[-1].driver.pose_at(sc.t), float)[:3, 3]
        where = "nearest the tool"
    else:
        c = np.median(x, axis=0)
        where = "nearest the bed centre"
    idx = np.sort(np.argsort(((x - c) ** 2).sum(axis=1), kind="stable")[:n_sample])
    return x[idx].copy(), v[idx].copy(), f"the {n_sample} particles {where}"


def oracle_run(sc, x, v, warmup: int, steps: int, budget_s: float):
    """W untimed + up to K timed oracle steps (stops early at budget_s).
    Returns (timed steps, seconds)."""
    from oracle import granular_oracle as O

    params = sc.params
    n_h = int(sc.hashmap_size or O.table_size(len(x)))
    t = sc.t
    for _ in range(warmup):
        t += params.timestep
        x, v, _, _, _ = O.step(x, v, params, bodies_at(sc, t), n_h, sc.boundary)
    done = 0
    t0 = time.perf_counter()
    while done < steps:
        t += params.timestep
        x, v, _, _, _ = O.step(x, v, params, bodies_at(sc, t), n_h, sc.boundary)
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return done, time.perf_counter() - t0


def cpu_baseline(sc, x, v, budget_s: float, warmup: int = 1, steps: int = 1000) -> dict:
    """The reference algorithm (oracle port, numpy, 1 thread) on a bounded
    sample of the same workload state, sized so the steps fit budget_s."""
    n_s = int(min(len(x), max(2000, ORACLE_RATE * budget_s / max(warmup + min(steps, 20), 1))))
    xs, vs, what = workload_sample(sc, x, v, n_s)
    done, el = oracle_run(sc, xs, vs, warmup, steps, budget_s)
    return {"value": len(xs) * done / el, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(),
            "kind": "port",
            "sample": f"{done} timed oracle steps (after {warmup} untimed) of {what} of the same "
                      f"workload state, {el:.1f} s, numpy single thread (OPENBLAS_NUM_THREADS=1); "
                      f"the reference steps one scene on one core"}


# ---------------------------------------------------------------------------
def run_reference(args, dist: Dist):
    """--impl reference: the reference CPU path (the oracle port: the
    reference is Python, there is no oracle/_ref binary) on the host, rank 0
    only.  W untimed + K timed steps, each one oracle step of a bounded sample
    of the workload sized so the run takes ~--ref-seconds; envs: every host
    core steps its own env."""
    if dist.rank != 0:
        return
    W, K = args.warmup, args.steps
    if args.workload == "envs":
        cb = envs_cpu_baseline(args, W, K, min(args.ref_seconds, 120.0))
        _, _, desc = envs_desc(args)
        scaling = "strong"
    else:
        sc, desc = make_scene(args, with_gpu=False)
        x = np.asarray(sc.particles._x, float).copy()
        v = np.asarray(sc.particles._v, float).copy()
        n_s = int(min(len(x), max(2000, ORACLE_RATE * args.ref_seconds / max(W + K, 1))))
        xs, vs, what = workload_sample(sc, x, v, n_s)
        done, el = oracle_run(sc, xs, vs, W, K, 4.0 * args.ref_seconds)
        cb = {"value": len(xs) * done / el, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(),
              "kind": "port",
              "sample": f"{done} timed steps (after {W} untimed) of {what} of the {desc['workload']} "
                        f"state, {el:.1f} s, numpy single thread (OPENBLAS_NUM_THREADS=1)"}
        scaling = "strong" if (args.gpus > 1 and not args.replicas) else "weak"
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": K, "warmup": W,
            "ms_per_step": 1000.0 * desc["n_particles"] / cb["value"], "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": desc, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def envs_desc(args, n_local: int | None = None):
    from paper_2306_01369_b200.envs import BulldozerEnvConfig

    cfg = BulldozerEnvConfig(n_particles=args.env_particles, radius=0.025)
    desc = {"workload": "envs", "config": "BASELINE configs[2]: batched bulldozer envs "
            f"{args.envs} x {args.env_particles} particles, sharded env e -> rank e mod N",
            "n_envs": args.envs, "n_particles": args.envs * args.env_particles,
            "dt": cfg.timestep, "solver_iterations": 10, "bodies": "ground + Box blade per env"}
    return cfg, n_local, desc


def envs_setup(args, dist: Dist, device: int):
    from paper_2306_01369_b200.batch import shard_envs
    from paper_2306_01369_b200.envs import BatchedBulldozerEnv

    mine = shard_envs(args.envs, dist.rank, dist.world)
    cfg, _, desc = envs_desc(args)
    env = BatchedBulldozerEnv(len(mine), cfg, device=device, render=False)  # physics e2e
    env.reset(mine)  # seed = env id
    acts = np.stack([np.random.default_rng(int(e)).uniform(-1, 1, 2) for e in mine])
    acts[:, 0] = np.abs(acts[:, 0])  # drive forward into the bed
    env.driver.command(acts)
    return env, acts, desc


def _env_worker(a):
    """One host core: env `seed`'s bed stepped by the oracle, W untimed + up
    to K timed steps within budget_s.  Returns (particles, steps, seconds)."""
    seed, env_particles, W, K, budget_s = a
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import granular_oracle as O
    from paper_2306_01369_b200.envs import BulldozerEnvConfig, bulldozer_scene

    cfg = BulldozerEnvConfig(n_particles=env_particles, radius=0.025)
    sc = bulldozer_scene(seed, cfg)
    x = sc.particles.positions.astype(np.float32).astype(np.float64)
    v = np.zeros_like(x)
    drv = sc.bodies[1].driver
    drv.command(np.array([0.8, 0.1]))
    t, done, el = 0.0, 0, 0.0
    for k in range(W + K):
        t0 = time.perf_counter()
        t += cfg.timestep
        drv.advance(cfg.timestep)
        x, v, _, _, _ = O.step(x, v, sc.params, bodies_at(sc, t), O.table_size(len(x)))
        if k >= W:
            el += time.perf_counter() - t0
            done += 1
            if el >= budget_s:
                break
    return len(x), done, el


def envs_cpu_baseline(args, W: int, K: int, budget_s: float) -> dict:
    """The reference algorithm (oracle port) with EVERY host core stepping its
    own env (the envs are independent), W untimed + K timed steps each."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    jobs = [(e, args.env_particles, W, K, budget_s) for e in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_env_worker, jobs)
    value = sum(n * d / el for n, d, el in res if el > 0)
    steps = min(d for _, d, _ in res)
    return {"value": value, "unit": UNIT, "cores": cores, "host_cores": cores, "kind": "port",
            "sample": f"{cores} processes (one per host core), each {steps}+ timed oracle steps "
                      f"(after {W} untimed) of its own {args.env_particles}-particle bulldozer env "
                      f"(seeds 0..{cores - 1}); sum of the per-core rates"}


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
    # (the timed loop above posed the bodies from host tables: hand the host
    # drivers' state back to the device drivers the env uses)
    if env.device_drivers:
        batch.drive_on_device()
    fs = env.config.frame_skip
    n_ctrl = max(K // fs, 1)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n_ctrl):
        _, rew, _, info = env.step(acts)
        _ = float(rew.sum())
    t_e2e = dist.max(time.perf_counter() - t0)
    e2e = {"value": n_total * n_ctrl * fs / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": (batch.E * 16) / fs if env.device_drivers
           else batch.E * batch.nb * N.BODY_DTYPE.itemsize,
           "d2h_bytes_per_step": (batch.E * (N.REPORT_DTYPE.itemsize + batch.nb * 24 + 24 + 8 + 8)) / fs
           if env.device_drivers else batch.E * N.REPORT_DTYPE.itemsize
           + (batch.E * (8 + 8) + batch.E * batch.nb * 24) / fs,
           "api": "BatchedBulldozerEnv.step(actions): actions uploaded, blade TrackSteeringDriver "
                  "and body rows on the device, frame_skip substeps, the last substep's per-env "
                  "StepReports, driver states and on-device rewards read back",
           "wall_s": t_e2e}
    cb = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cb = envs_cpu_baseline(args, 2, 200, args.cpu_seconds)
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
            "warmup": W, "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 state / f64 contact geometry",
            "data": "synthetic (seeded bulldozer beds, settled 100 substeps)",
            "config": desc,
            "run": {"parallelism": f"env shards x{dist.world}", "envs_per_rank": batch.E,
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
    """One bed slab-decomposed over the N ranks (SlabBed): the bed1m workload
    at N > 1 (north_star: the 1M bed with a scoop on 8 GPUs), or config 5
    (--workload slab: lattice_bed(8e6) + floor).  "scaling": "strong"."""
    import paper_2306_01369_b200 as gg
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.slab import SlabBed

    import torch

    dev = dist.local
    if args.workload == "slab":
        n = args.slab_particles
        x = gg.lattice_bed(n).astype(np.float32).astype(np.float64)
        v = np.zeros_like(x)

        def scene():
            return gg.Scene(particles=gg.ParticleSet(x, v), bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                            params=gg.MaterialParams(timestep=5e-4))

        desc = {"workload": "slab", "config": "BASELINE configs[4]: 8M bed, slab decomposition over N GPUs",
                "n_particles": n, "dt": 5e-4, "solver_iterations": 10, "bodies": "floor"}
    else:
        sc0, desc = make_scene(args)
        x = np.asarray(sc0.particles._x, float).copy()
        v = np.asarray(sc0.particles._v, float).copy()
        n = len(x)

        def scene():
            s2, _ = make_scene(args)
            return s2

    bed = SlabBed(scene(), rank=dist.rank, world=dist.world, device=dev,
                  backend=dist.backend if dist.world > 1 else None, halo=args.halo)
    lib = N.lib()
    K, W = args.steps, args.warmup
    bed.run(W)
    stream = torch.cuda.ExternalStream(lib.gg_stream(bed.ctx), device=torch.device("cuda", dev))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = int(lib.gg_kernel_launches(bed.ctx))
    clocks = Clocks(dev)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    reps = bed.run(K)  # (peer-memory transport: K steps back to back on the device)
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
                "note": "whole-step byte model per GPU (SURVEY.md §8d); the kernels are those of "
                        "the one-GPU step (per-kernel fractions in the N = 1 line)"}
    # e2e through the public API from host buffers (pinned, like the
    # one-context line): partition + upload of the global host state into
    # the bed (SlabBed.load), K steps, gather of the global state back to
    # the host (the context and its graphs exist, as for run() there)
    xh = np.ascontiguousarray(x, dtype=np.float64)
    vh = np.ascontiguousarray(v, dtype=np.float64)
    lib.gg_host_register(N.ptr(xh), xh.nbytes)
    lib.gg_host_register(N.ptr(vh), vh.nbytes)
    dist.barrier()
    t0 = time.perf_counter()
    bed.load(xh, vh)
    bed.run(K)
    Xg, _ = bed.gather()
    _ = float(Xg[0, 0])
    t_e2e = dist.max(time.perf_counter() - t0)
    lib.gg_host_unregister(N.ptr(xh))
    lib.gg_host_unregister(N.ptr(vh))
    bed.close()
    e2e = {"value": n * K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 48 * n / max(K, 1),
           "d2h_bytes_per_step": 52 * n / max(K, 1), "wall_s": t_e2e,
           "api": "SlabBed.load(x, v) (partition + upload of the global host state), "
                  "SlabBed.run(K), SlabBed.gather() (global state back on the host)"}
    cb = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        sc_cb = scene()
        cb = cpu_baseline(sc_cb, x, v, args.cpu_seconds)
    if dist.rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
                "warmup": W, "ms_per_step": t_ms / K, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 state / f64 contact geometry", "data": "synthetic",
                "config": desc,
                "run": {"parallelism": f"slabs x{dist.world}", "n_h": bed.n_h, "c_pp": c_pp,
                        "c_b": c_b, "max_owned": owned, "backend": dist.backend, "halo": bed.halo,
                        "l2": "not flushed: the state exceeds L2"},
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
    # contacts with the tool (bodies after the floor and walls), per step
    n_tool = None
    if nb > 1:
        from paper_2306_01369_b200.contact import device_detect

        for body in sc.bodies:
            body.update(sc.t)
        cs, _ = device_detect(sc.particles.positions, sc.params.radius, eng.n_h, sc.bodies,
                              params=sc.params)
        n_tool = int(np.sum((cs.kind == 1) & (cs.other == nb - 1)))

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
        cb = cpu_baseline(sc, x0, v0, args.cpu_seconds, warmup=1, steps=1000)

    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": K,
            "warmup": W, "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 state / f64 contact geometry",
            "data": ("synthetic (50k column bed settled on the GPU, bench_data/hero50k_settled.npz)"
                     if args.workload == "hero50k" else
                     "synthetic (lattice_bed(1e6) settled on the GPU, bench_data/bed1m_settled.npz)"),
            "config": desc,
            "run": {"parallelism": f"replicas x{dist.world}" if dist.world > 1 else "single",
                    "pipeline": args.pipeline, "solve_mode": args.solve_mode,
                    "l2": l2_note(args, n * 200 / 2**20),
                    "c_pp": c_pp, "c_b": c_b, "n_tool_contacts": n_tool, "n_h": eng.n_h,
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


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: run this script under
    torch.distributed.run with N processes on this node (rendezvous on
    127.0.0.1, NCCL_DEBUG=INFO so the communicator's ranks are visible)."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.flush_mb < 0:
        args.flush_mb = 512 if args.workload == "hero50k" else 0
    dist = Dist()
    if args.impl != "reference" and dist.world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={dist.world}")
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif args.workload == "envs":
            run_envs(args, dist)
        elif args.workload == "slab" or (dist.world > 1 and not args.replicas):
            run_slab(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
