"""Config-4 inputs shared by both bench arms (run once on a GPU):

  bench_data/bed1m_settled.npz  lattice_bed(1e6) + floor settled on the GPU at
                                dt = 1e-3 until KE/n < 2e-3 J, then the excavator
                                bucket's pass (beds.excavator_dig) run for its
                                first second at dt = 5e-4, so the bench starts
                                with the bucket 1 m into the pile's flank
                                (positions float32, velocities float16, time,
                                the DigDriver arguments)
  bench_data/bucket1m_grid.npz  the excavator bucket (beds.BUCKET1M_*) baked on
                                the device (bit-exact with the reference baker,
                                tests/test_bake.py)

    python tools/make_bed1m.py [out_dir]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2306_01369_b200 as gg  # noqa: E402
from paper_2306_01369_b200.beds import (  # noqa: E402
    BUCKET1M_HALF, BUCKET1M_SPACING, BUCKET1M_WALL, excavator_dig)
from paper_2306_01369_b200.meshes import make_bucket_mesh  # noqa: E402
from paper_2306_01369_b200.sdf import bake_mesh_sdf  # noqa: E402


def main(out_dir: str = "gpurun_out", max_steps: int = 10000):
    out = Path(out_dir)
    out.mkdir(exist_ok=True)
    t0 = time.perf_counter()
    x = gg.lattice_bed(1_000_000).astype(np.float32).astype(np.float64)
    sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                  params=gg.MaterialParams(timestep=1e-3))
    done, ke = 0, float("inf")
    while done < max_steps:
        _, reps = gg.run(sc, 250)
        done += 250
        ke = reps[-1].kinetic_energy / sc.particles.count
        print(f"step {done}: KE/n {ke:.4g} J  c_pp {reps[-1].n_contacts / 1e6:.3f}", flush=True)
        if ke < 2e-3:
            break
    info = {"dt": 1e-3, "steps": done, "ke_per_particle_J": ke, "target_J": 2e-3,
            "generator": "tools/make_bed1m.py"}
    verts, faces = make_bucket_mesh(BUCKET1M_HALF, BUCKET1M_WALL)
    grid = bake_mesh_sdf(verts, faces, BUCKET1M_SPACING)
    # the bucket's first second: it starts outside the flank at the settled time
    lead = 1.0
    xs0 = sc.particles.positions.copy()
    drv = excavator_dig(xs0, sc.t + lead, lead=lead)
    sc.bodies.append(gg.RigidBody(grid, drv, name="bucket"))
    sc.params.timestep = 5e-4
    _, reps = gg.run(sc, int(round(lead / 5e-4)))
    dig = {"start": drv.start.tolist(), "direction": drv.direction.tolist(), "length": drv.length,
           "depth": drv.depth, "duration": drv.duration, "pitch0": drv.pitch0, "pitch1": drv.pitch1,
           "t0": drv.t0, "lift_speed": drv.lift_speed}
    info["dig_lead_s"] = lead
    info["dig_last_step"] = {"n_contacts": reps[-1].n_contacts, "n_body_contacts": reps[-1].n_body_contacts,
                             "kinetic_energy": reps[-1].kinetic_energy}
    print("after the lead:", info["dig_last_step"], flush=True)
    np.savez_compressed(out / "bed1m_settled.npz", x=sc.particles.positions.astype(np.float32),
                        v=sc.particles.velocities.astype(np.float16), t=np.array(sc.t),
                        settle=json.dumps(info), dig=json.dumps(dig))
    np.savez_compressed(out / "bucket1m_grid.npz", values=grid.values, origin=grid.origin,
                        spacing=grid.spacing, dims=np.asarray(grid.dims), mesh_hash=np.frombuffer(grid.mesh_hash, np.uint8))
    print(f"saved in {time.perf_counter() - t0:.1f} s: {info}; grid dims {grid.dims}")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []))
