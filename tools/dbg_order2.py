import os, sys, subprocess
import numpy as np
sys.path.insert(0, os.getcwd())

def run(out, pre, E, T, rs):
    import paper_2306_01369_b200 as gg
    from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BulldozerEnvConfig
    if pre:
        gg.spatial_hash(np.zeros((1, 3), np.int64), 64)
    cfg = BulldozerEnvConfig(n_particles=2000, radius=0.025)
    env = BatchedBulldozerEnv(E, cfg)
    env.reset(np.arange(E))
    env.batch.driven = None
    if rs: gg._native.lib().gg_set_resort_every(env.batch.ctx, rs)
    x0, v0 = env.batch.state()
    env.driver.command(np.random.default_rng(0).uniform(-1, 1, size=(E, 2)))
    reps, _ = env.batch.run_raw(T)
    xb, vb = env.batch.state()
    import time; time.sleep(0.5)
    xb2, _ = env.batch.state()
    print("pre", pre, "second read equal", np.array_equal(xb, xb2))
    np.savez(out, x0=x0, xb=xb, vb=vb, **{f: reps[f] for f in reps.dtype.names})

if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1], sys.argv[2] == "1", int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])); sys.exit()
    for E, T, rs in ((256, 2, 0), (256, 3, 1), (256, 3, 100), (256, 8, 100), (128, 8, 0), (100, 8, 0)):
        for pre in ("0", "1"):
            subprocess.run([sys.executable, __file__, f"/tmp/o{pre}.npz", pre, str(E), str(T), str(rs)], check=True)
        a, b = np.load("/tmp/o0.npz"), np.load("/tmp/o1.npz")
        diff = [k for k in a.files if not np.array_equal(a[k], b[k])]
        print(E, T, rs, "differs:", diff)
        if "xb" in diff:
            d = np.abs(a["xb"] - b["xb"]).reshape(E, -1).max(1)
            print("   envs differing", np.nonzero(d)[0][:20], d.max())
            print("   sorted equal", all(np.array_equal(np.sort(a["xb"][e], 0), np.sort(b["xb"][e], 0)) for e in range(E)))
