"""Debug: per-kernel path (ONE_LOOP) with/without integrate-time counting."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")

def run(out):
    import paper_2306_01369_b200 as gg
    from helpers import load, scene_from
    g = load("lattice_500")
    sc = scene_from(g)
    reps = []
    for _ in range(5):
        _, r = gg.step(sc, gg.PipelineMode.ONE_LOOP)
        reps.append((r.n_contacts, r.n_candidates, r.n_body_contacts))
    np.savez(out, x=sc.particles.positions, reps=np.array(reps))

if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1]); sys.exit()
    for name, lib in [("cn", None), ("nocn", "build_variants/a_nocn.so")]:
        env = dict(os.environ)
        if lib: env["GG_LIB"] = os.path.abspath(lib)
        subprocess.run([sys.executable, __file__, f"/tmp/cn_{name}.npz"], env=env, check=True)
    a, b = np.load("/tmp/cn_cn.npz"), np.load("/tmp/cn_nocn.npz")
    print("reps cn", a["reps"].tolist()); print("reps nocn", b["reps"].tolist())
    print("x equal", np.array_equal(a["x"], b["x"]))
