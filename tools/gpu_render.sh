mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BulldozerEnvConfig
env = BatchedBulldozerEnv(4096, BulldozerEnvConfig(n_particles=2000, radius=0.025))
env.reset()
acts = np.tile([0.8, 0.1], (4096, 1))
env.step(acts)
for mode in (0, 1, 0):
    N.lib().gg_set_render_mode(mode)
    env._observe()
    t0 = time.perf_counter(); obs = env._observe(); t1 = time.perf_counter()
    print("render mode", mode, "4096 envs x (36x36 + 72x36):", round((t1 - t0) * 1e3, 1), "ms")
N.lib().gg_set_render_mode(0)
t0 = time.perf_counter()
for _ in range(5):
    env.step(acts)
print("env.step (10 substeps + render + reward), 4096 envs:", round((time.perf_counter() - t0) / 5 * 1e3, 1), "ms")
env.render = False
t0 = time.perf_counter()
for _ in range(5):
    env.step(acts)
print("env.step without render:", round((time.perf_counter() - t0) / 5 * 1e3, 1), "ms")
PY
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/q_hero.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/q_hero.json')); print('hero', d['ms_per_step'], d['value'])"
