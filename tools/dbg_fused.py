import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from helpers import load, scene_from, rel_err
import paper_2306_01369_b200 as gg
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.engine import engine_for

g = load(sys.argv[1] if len(sys.argv) > 1 else "primitives_3000")
for mode in (3, 4):
    for K in (16, 64):
        sc = scene_from(g)
        eng = engine_for(sc)
        eng.max_contacts = K
        eng.prepare(sc)
        N.lib().gg_set_solve_mode(eng.ctx, mode)
        _, rep = gg.step(sc, step_index=0)
        print(f"mode {mode} K0 {K} -> K {eng.max_contacts}: rel_x {rel_err(sc.particles.positions, g['x1']):.2e} "
              f"rel_v {rel_err(sc.particles.velocities, g['v1']):.2e} n_pp {rep.n_contacts} ref {int(g['rep_n_contacts'])} "
              f"body {rep.n_body_contacts} ref {int(g['rep_n_body_contacts'])}")
