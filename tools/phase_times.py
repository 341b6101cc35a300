"""Per-phase breakdown of the fused single-kernel step (GPU)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.engine import engine_for


class A:
    workload = sys.argv[1] if len(sys.argv) > 1 else "hero50k"
    settle = 3000


sc, desc = bench.make_scene(A)
eng = engine_for(sc)
eng.prepare(sc)
lib = N.lib()
lib.gg_set_solve_mode(eng.ctx, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
lib.gg_phase_timer(eng.ctx, 1, None, 0)
nb = len(sc.bodies)
for resort in (False, True):
    table, _ = eng.body_tables(sc, 20)
    eng.run_batch(table, nb, 0)
    if resort:
        lib.gg_set_resort_every(eng.ctx, 1)
    table, _ = eng.body_tables(sc, 1)
    eng.run_batch(table, nb, 0)
    st = np.zeros(64, dtype=np.uint64)
    lib.gg_phase_timer(eng.ctx, 1, N.ptr(st), 64)
    sub = st[48:56].astype(np.int64)
    if (sub > 0).all():  # contact-kernel sub-phases of block 0, thread 0 (library built with -DGG_CSTAMP=1)
        print("  contacts sub-phases (us): bucket lists, candidates, (phase B start), exact test, body count, records, counters:",
              np.round(np.diff(sub) / 1000.0, 2).tolist())
    st[48:] = 0
    k = int(np.nonzero(st)[0].max()) + 1
    d = np.diff(st[:k].astype(np.int64)) / 1000.0
    print(f"resort={resort} total {(int(st[k-1]) - int(st[0])) / 1000:.1f} us; phases (us):", np.round(d, 2).tolist())
