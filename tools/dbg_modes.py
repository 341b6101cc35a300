"""Compare launch modes (state after 7 steps) on the golden cases; print diffs."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2306_01369_b200 as gg
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.engine import engine_for
from helpers import load, scene_from

for name in ["grid_tool", "primitives_3000", "lattice_5000"]:
    g = load(name)
    out = {}
    for mode in (4, 4, 1, 2, 3, 6, 7):
        sc = scene_from(g)
        eng = engine_for(sc)
        eng.max_contacts = 64
        eng.prepare(sc)
        N.lib().gg_set_solve_mode(eng.ctx, mode)
        N.lib().gg_set_resort_every(eng.ctx, 3)
        reps = gg.run(sc, 7)[1]
        xv = (sc.particles.positions.copy(), sc.particles.velocities.copy(), [r.n_contacts for r in reps])
        key = mode if mode not in out else f"{mode}b"
        out[key] = xv
    for m in out:
        dx = np.abs(out[m][0] - out[4][0]).max()
        dv = np.abs(out[m][1] - out[4][1]).max()
        print(name, m, "dx", dx, "dv", dv, "contacts", out[m][2] == out[4][2])
