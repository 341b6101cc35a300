import sys, time, cProfile, pstats
sys.path.insert(0, ".")
import numpy as np
from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BulldozerEnvConfig
cfg = BulldozerEnvConfig(n_particles=2000, radius=0.025)
env = BatchedBulldozerEnv(4096, cfg, render=False)
env.reset(seeds=list(range(4096)))
acts = np.tile([0.5, 0.1], (4096, 1))
for _ in range(3): env.step(acts)
t = time.perf_counter()
for _ in range(5): env.step(acts)
print("per env.step ms", (time.perf_counter() - t) / 5 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(5): env.step(acts)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
