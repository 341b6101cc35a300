"""Hash-table size sweep on the GPU (the paper's n_h = 2 n_p
heuristic; the reference's own CPU test of it is
tests/test_acceptance.py:214-235).  Device ms/step of the same bed for
n_h = f x n_p rounded to a power of two, f in {1/2, 1, 2, 4, 8, 16}.

    python tools/hash_sweep.py [n_particles] [steps]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.engine import engine_for

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
x0 = gg.lattice_bed(n).astype(np.float32).astype(np.float64)
# relax the compressed lattice once, then time every table size from that state
sc = gg.Scene(particles=gg.ParticleSet(x0, np.zeros_like(x0)),
              bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")], params=gg.MaterialParams(timestep=5e-4))
gg.run(sc, 100)
xs, vs = sc.particles.positions.copy(), sc.particles.velocities.copy()
rows = []
for f in (0.5, 1, 2, 4, 8, 16):
    n_h = 1 << int(np.round(np.log2(f * n)))
    sc = gg.Scene(particles=gg.ParticleSet(xs.copy(), vs.copy()),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                  params=gg.MaterialParams(timestep=5e-4), hashmap_size=n_h)
    gg.run(sc, 5)  # warm-up (context, graphs)
    eng = engine_for(sc)
    _, reps = gg.run(sc, steps)
    ms = eng.last_batch_ms() / steps
    cand = np.mean([r.n_candidates for r in reps]) / n
    rows.append((f, n_h, ms, cand))
    print(f"n_h = {f:>4} n_p = {n_h:>9}: {ms:.4f} ms/step, {cand:.1f} candidates/particle", flush=True)
best = min(r[2] for r in rows)
print("relative speed (best = 1):", {r[0]: round(best / r[2], 3) for r in rows})
