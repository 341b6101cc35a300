"""Calibrate the reference arm: the oracle port vs the REAL reference stepper
on the same bounded sample of a bench workload (this container only — the
reference is not on the GPU box, so bench.py's reference arm times the port).

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tools/calibrate_port.py --workload bed1m --n-sample 20000 --steps 5

Both run single-threaded numpy on the same particles (bench.workload_sample,
the particles nearest the tool), the same bodies and the same parameters,
interleaved step for step, from the same start; prints one JSON line with
both rates (particle-steps/s), their ratio and the max |x| difference of the
final states (the two must agree: the port is pinned to the reference).
Test infrastructure: imports oracle/ and the reference, nothing else does.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import granusim  # noqa: E402
from granusim import sdf as rsdf  # noqa: E402
from granusim.scene import MaterialParams, ParticleSet, RigidBody, Scene  # noqa: E402
from granusim.stepper import step as ref_step  # noqa: E402

import bench  # noqa: E402
from oracle import granular_oracle as O  # noqa: E402

assert "/root/reference" in granusim.__file__, granusim.__file__


def ref_geometry(g):
    """Our geometry object -> the reference's class with the same fields."""
    name = type(g).__name__
    if name == "HalfSpace":
        return rsdf.HalfSpace(**{k: getattr(g, k) for k in ("normal", "offset") if hasattr(g, k)})
    if name == "SdfGrid":
        return rsdf.SdfGrid(np.asarray(g.origin), np.asarray(g.spacing), np.asarray(g.dims),
                            np.asarray(g.values), bytes(g.mesh_hash))
    import dataclasses
    cls = getattr(rsdf, name, None)
    if cls is None or not dataclasses.is_dataclass(cls):
        raise TypeError(f"no reference mapping for {name}")
    return cls(**{f.name: getattr(g, f.name) for f in dataclasses.fields(cls) if f.init})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bed1m", choices=["bed1m", "hero50k"])
    ap.add_argument("--n-sample", type=int, default=20000)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    sys.argv = [sys.argv[0], "--workload", a.workload]
    args = bench.parse()
    sc, desc = bench.make_scene(args, with_gpu=False)
    x = np.asarray(sc.particles._x, float).copy()
    v = np.asarray(sc.particles._v, float).copy()
    xs, vs, what = bench.workload_sample(sc, x, v, a.n_sample)
    n_h = int(sc.hashmap_size or O.table_size(len(xs)))

    p = sc.params
    rp = MaterialParams(**{f: getattr(p, f) for f in MaterialParams.__dataclass_fields__})
    rbodies = [RigidBody(ref_geometry(b.geometry), b.driver, name=b.name) for b in sc.bodies]
    rsc = Scene(particles=ParticleSet(xs.copy(), vs.copy()), bodies=rbodies, params=rp,
                hashmap_size=n_h, boundary=sc.boundary)
    rsc.t = sc.t

    xo, vo, t = xs.copy(), vs.copy(), sc.t
    t_ref = t_port = 0.0
    for _ in range(a.steps):
        t0 = time.perf_counter()
        ref_step(rsc)
        t_ref += time.perf_counter() - t0
        t += p.timestep
        t0 = time.perf_counter()
        xo, vo, _, _, _ = O.step(xo, vo, p, bench.bodies_at(sc, t), n_h, sc.boundary)
        t_port += time.perf_counter() - t0
    dx = float(np.abs(np.asarray(rsc.particles.positions) - xo).max())
    n = len(xs)
    print(json.dumps({
        "workload": desc["workload"], "sample": what, "steps": a.steps, "n_h": n_h,
        "reference_rate": n * a.steps / t_ref, "port_rate": n * a.steps / t_port,
        "port_over_reference": t_ref / t_port, "reference_ms_per_step": 1e3 * t_ref / a.steps,
        "port_ms_per_step": 1e3 * t_port / a.steps, "max_abs_dx": dx,
        "threads": os.environ.get("OPENBLAS_NUM_THREADS"),
    }))


if __name__ == "__main__":
    main()
