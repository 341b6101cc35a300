"""L2 residency probe: the settled bed1m state cut to its n particles of
smallest x (floor only), stepped on the GPU; run under ncu --cache-control
none to read a sweep's DRAM traffic as a function of the per-sweep working
set.  usage: python tools/l2_probe.py N STEPS"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2306_01369_b200 as gg

n, steps = int(sys.argv[1]), int(sys.argv[2])
d = np.load("bench_data/bed1m_settled.npz")
x, v = d["x"].astype(np.float64), d["v"].astype(np.float64)
keep = np.argsort(x[:, 0], kind="stable")[:n]
params = gg.MaterialParams(timestep=5e-4)
sc = gg.Scene(particles=gg.ParticleSet(x[keep], v[keep]), bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
              params=params)
traj, reps = gg.run(sc, steps)
print(n, "c_pp", reps[-1].n_contacts / n)
