"""Free-running scoop fixture from the REAL reference (north_star criterion 3).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_scoop.py

Scene (tests/scoop_stats.py): a flat 4000-particle seeded bed settled by the
reference (800 steps at dt = 1e-3), then an open-top bucket (our
make_bucket_mesh, baked by the REFERENCE's bake_mesh_sdf) on a DigDriver
(beds.py; pure numpy, handed to the reference RigidBody duck-typed) makes one
digging pass and lifts: 4000 reference steps at dt = 5e-4.  Every 200 steps
the bulk statistics of tests/scoop_stats.py are recorded.  The settled state
is rounded to float32 before the pass, so both runs start identically.
Output: tests/golden/scoop_run.npz (~2.5 min of CPU).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))

import granusim  # noqa: E402
from granusim.kinematics import StaticDriver, identity_pose  # noqa: E402
from granusim.scene import BoxRegion, MaterialParams, ParticleSet, RigidBody, Scene  # noqa: E402
from granusim.scene import seed_particles_grid  # noqa: E402
from granusim.sdf import HalfSpace, bake_mesh_sdf  # noqa: E402
from granusim.stepper import step  # noqa: E402

import scoop_stats as S  # noqa: E402
from paper_2306_01369_b200.beds import DigDriver  # noqa: E402  (pure numpy)
from paper_2306_01369_b200.meshes import make_bucket_mesh  # noqa: E402  (pure numpy)

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731


def main():
    t_start = time.time()
    seeded = seed_particles_grid(BoxRegion(np.array(S.BED_LO), np.array(S.BED_HI)), S.R,
                                 jitter=S.BED_JITTER, rng=np.random.default_rng(S.BED_SEED))
    assert seeded.count >= S.N, seeded.count
    x = f32(seeded.positions[: S.N])
    floor = RigidBody(HalfSpace(), StaticDriver(identity_pose()), name="floor")
    sc = Scene(particles=ParticleSet(x, np.zeros_like(x)), bodies=[floor],
               params=MaterialParams(timestep=S.SETTLE_DT))
    for _ in range(S.SETTLE_STEPS):
        step(sc)
    xs, vs = f32(sc.particles.positions), f32(sc.particles.velocities)
    ke_settled = 0.5 * sc.params.particle_mass * float((vs ** 2).sum())
    verts, faces = make_bucket_mesh(S.BUCKET_HALF, S.BUCKET_WALL)
    grid = bake_mesh_sdf(verts, faces, S.BUCKET_SPACING)
    path = S.dig_path(xs)
    bucket = RigidBody(grid, DigDriver(**path), name="bucket")
    floor = RigidBody(HalfSpace(), StaticDriver(identity_pose()), name="floor")
    sc = Scene(particles=ParticleSet(xs.copy(), vs.copy()), bodies=[floor, bucket],
               params=MaterialParams(timestep=S.DT))
    lo = np.array([xs[:, 0].min() - 0.5, xs[:, 1].min() - 0.5])
    nx = ny = S.MAP_COLUMNS
    lift_z = float(np.quantile(xs[:, 2], 0.99)) + S.R + 0.1
    rec = {k: [] for k in ("step", "ke", "n_pp", "n_body", "carried", "lifted", "height_map",
                           "bucket_pose")}
    n_pp = n_b = 0
    for k in range(1, S.DIG_STEPS + 1):
        _, rep = step(sc)
        n_pp += rep.n_contacts
        n_b += rep.n_body_contacts
        if k % S.RECORD_EVERY == 0:
            pose = np.asarray(bucket.pose, float)
            st = S.summary(sc.particles.positions, pose, lift_z, lo, nx, ny)
            rec["step"].append(k)
            rec["ke"].append(rep.kinetic_energy)
            rec["n_pp"].append(n_pp / S.RECORD_EVERY)
            rec["n_body"].append(n_b / S.RECORD_EVERY)
            rec["carried"].append(st["carried"])
            rec["lifted"].append(st["lifted"])
            rec["height_map"].append(st["height_map"])
            rec["bucket_pose"].append(pose)
            n_pp = n_b = 0
            print(f"step {k}: carried {st['carried']} lifted {st['lifted']} "
                  f"KE {rep.kinetic_energy:.3g} pp {rec['n_pp'][-1]:.0f} body {rec['n_body'][-1]:.0f}",
                  flush=True)
    out = {k: np.asarray(v) for k, v in rec.items()}
    out.update(x_settled=xs, v_settled=vs, ke_settled=ke_settled, grid_values=grid.values,
               grid_origin=grid.origin, grid_spacing=grid.spacing, grid_dims=grid.dims,
               lo=lo, lift_z=lift_z, x_final=sc.particles.positions.copy(),
               path=np.array([path["start"][0], path["start"][1], path["start"][2], path["length"],
                              path["depth"], path["duration"], path["pitch0"], path["pitch1"],
                              path["lift_speed"]]))
    np.savez_compressed(OUT / "scoop_run.npz", **out)
    print(f"done in {time.time() - t_start:.0f} s")


if __name__ == "__main__":
    main()
