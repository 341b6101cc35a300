"""initcheck target: utility context first, then a small batched bulldozer run."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BulldozerEnvConfig
gg.spatial_hash(np.zeros((1, 3), np.int64), 64)
cfg = BulldozerEnvConfig(n_particles=2000, radius=0.025)
E, T = int(os.environ.get("E", 32)), int(os.environ.get("T", 3))
env = BatchedBulldozerEnv(E, cfg)
env.reset(np.arange(E))
env.batch.driven = None
env.driver.command(np.random.default_rng(0).uniform(-1, 1, size=(E, 2)))
reps, _ = env.batch.run_raw(T)
print("ok", env.batch.state()[0].sum())
