"""KE trajectory of the 1M lattice bed settling on the GPU (bench.py bed1m_settled).

    PYTHONPATH=. python tools/settle_probe.py
"""
import time, numpy as np
import paper_2306_01369_b200 as gg
x = gg.lattice_bed(1_000_000).astype(np.float32).astype(np.float64)
sc = gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)), bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
              params=gg.MaterialParams(timestep=1e-3))
t0=time.time(); done=0
while done < 30000:
    _, reps = gg.run(sc, 1000); done += 1000
    r = reps[-1]; p = sc.particles.positions
    print(done, "KE/n %.4g" % (r.kinetic_energy/1e6), "c_pp %.3f" % (r.n_contacts/1e6), "zmax %.2f" % p[:,2].max(), "xext %.2f %.2f" % (p[:,0].min(), p[:,0].max()), "t %.1f" % (time.time()-t0), flush=True)
    if r.kinetic_energy/1e6 < 1e-3: break
