"""Small runs of every schedule for compute-sanitizer (memcheck / racecheck /
synccheck): the fused step (mode 7), per-phase kernels (mode 3), a batched
context (E > 1), a slab step, and the renderer.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.batch import SceneBatch
from paper_2306_01369_b200.engine import engine_for
from paper_2306_01369_b200.render import DepthCamera, render_depth
from paper_2306_01369_b200.slab import SlabBed


def bed(n, seed=0):
    x = gg.lattice_bed(n, seed=seed).astype(np.float32).astype(np.float64)
    tool = gg.RigidBody(gg.Box(np.array([0.2, 0.1, 0.05])),
                        gg.SpinDriver(axis=[0, 0, 1], rate=2.0, center=[0.3, 0.3, 0.3],
                                      base_pose=gg.make_pose(np.eye(3), [0.4, 0.3, 0.25])))
    return gg.Scene(particles=gg.ParticleSet(x, np.zeros_like(x)),
                    bodies=[gg.RigidBody(gg.HalfSpace()), tool], params=gg.MaterialParams(timestep=5e-4))


for mode in (7, 3):
    sc = bed(3000)
    eng = engine_for(sc)
    eng.prepare(sc)
    N.lib().gg_set_solve_mode(eng.ctx, mode)
    gg.run(sc, 3)
    print("mode", mode, "ok")
batch = SceneBatch([bed(700, s) for s in range(3)])
batch.run_raw(3)
print("batch ok")
slab = SlabBed(bed(3000))
slab.run(2)
print("slab ok")
sc = bed(500)
img = render_depth(sc, DepthCamera(kind="perspective", pose=gg.make_pose(np.eye(3), [0.5, 0.5, -2.0]),
                                   width=16, height=12))
print("render ok", float(img.min()))
