"""Debug: batched envs (E x 2000) under the default library vs GG_LIB variant;
compares final states bitwise and after row sorting."""
import os, sys, json, subprocess
import numpy as np

def run(out):
    sys.path.insert(0, os.getcwd())
    from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BulldozerEnvConfig
    from paper_2306_01369_b200.batch import TrackSteeringBatch
    cfg = BulldozerEnvConfig(n_particles=2000, radius=0.025)
    E, T = int(os.environ.get("E", 256)), int(os.environ.get("T", 80))
    env = BatchedBulldozerEnv(E, cfg)
    env.reset(np.arange(E))
    env.batch.driven = None
    acts = np.random.default_rng(0).uniform(-1, 1, size=(E, 2))
    env.driver.command(acts)
    reps, _ = env.batch.run_raw(T)
    xb, vb = env.batch.state()
    np.savez(out, x=xb, v=vb, nc=reps["n_contacts"])

if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1]); sys.exit()
    for name, lib in [("rm", None), ("old", "build_variants/b_old.so")]:
        env = dict(os.environ)
        if lib: env["GG_LIB"] = os.path.abspath(lib)
        subprocess.run([sys.executable, __file__, f"/tmp/dbg_{name}.npz"], env=env, check=True)
    a, b = np.load("/tmp/dbg_rm.npz"), np.load("/tmp/dbg_old.npz")
    print("nc equal", np.array_equal(a["nc"], b["nc"]))
    for k in ("x", "v"):
        d = np.abs(a[k] - b[k])
        print(k, "bitwise", np.array_equal(a[k], b[k]), "maxdiff", d.max(), "envs differing", int((d.reshape(d.shape[0], -1).max(1) > 0).sum()))
        e = int(np.argmax(d.reshape(d.shape[0], -1).max(1)))
        print("  worst env", e, "rows differing", int((d[e].max(1) > 0).sum()), "sorted-equal", np.array_equal(np.sort(a[k][e], 0), np.sort(b[k][e], 0)))
