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
for pipe in (gg.PipelineMode.TWO_LOOPS_FUSED, gg.PipelineMode.ONE_LOOP):
    sc = bed(2000)
    gg.run(sc, 2, mode=pipe)
    print("pipeline", pipe.value, "ok")
big = bed(40000)  # > fused grid? exercises k_narrow / k_sweep / k_finish when not fused
eng = engine_for(big)
eng.prepare(big)
N.lib().gg_set_solve_mode(eng.ctx, 3)
gg.run(big, 2)
print("per-sweep kernels ok")
from paper_2306_01369_b200.meshes import make_gear_mesh
from paper_2306_01369_b200.sdf import bake_mesh_sdf
g = bake_mesh_sdf(*make_gear_mesh(n_teeth=5, root_radius=0.05, tip_radius=0.08, thickness=0.03, n_layers=2), 0.01)
print("bake ok", g.values.shape)
