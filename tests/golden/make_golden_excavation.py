"""Golden fixtures for the batched excavation env, from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_excavation.py

ExcavationEnv(n_particles=300) (envs.py:233-348: 7-joint chain + Box scoop,
the paper's hero scene layout) for seeds 0 and 1: the seeded bed, the state
rounded to float32, then one control step with a fixed 7-joint action: the
scoop pose/twist at every substep, the state after the first substep and
after the whole step, and the observation (ego + sky depth, end pose).
Saved as tests/golden/excavation_env.npz.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

import granusim
from granusim.envs import ExcavationEnv
from granusim.stepper import step

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731

SEEDS = [0, 1]
ACTIONS = np.array([[0.8, -0.5, 0.3, 0.9, -1.0, 0.4, 0.2],
                    [-0.6, 0.7, -0.2, 0.5, 0.3, -0.9, 1.0]])


def main():
    out = {"seeds": np.array(SEEDS), "actions": ACTIONS}
    keys = ["x0", "x1", "v1", "xT", "vT", "scoop_pose", "scoop_omega", "scoop_v", "ego", "sky",
            "end_pose", "q"]
    acc = {k: [] for k in keys}
    for e, seed in enumerate(SEEDS):
        env = ExcavationEnv(n_particles=300)
        env.reset(seed)
        sc = env.scene
        acc["x0"].append(sc.particles.positions.copy())
        sc.particles.positions[:] = f32(sc.particles.positions)
        sc.particles.velocities[:] = f32(sc.particles.velocities)
        a = np.clip(ACTIONS[e], -1.0, 1.0)
        limits = np.array([l.velocity_limit for l in env.chain.links])
        P, W, V = [], [], []
        for k in range(env.frame_skip):
            env.chain.advance(a * limits, sc.params.timestep)
            step(sc)
            scoop = sc.bodies[1]
            P.append(np.asarray(scoop.pose, float).copy())
            W.append(np.asarray(scoop.omega, float).copy())
            V.append(np.asarray(scoop.v_origin, float).copy())
            if k == 0:
                acc["x1"].append(sc.particles.positions.copy())
                acc["v1"].append(sc.particles.velocities.copy())
        acc["xT"].append(sc.particles.positions.copy())
        acc["vT"].append(sc.particles.velocities.copy())
        acc["scoop_pose"].append(P)
        acc["scoop_omega"].append(W)
        acc["scoop_v"].append(V)
        sc.particles.positions[:] = f32(sc.particles.positions)  # render the float32 state
        obs = env._observe()
        acc["ego"].append(obs.ego)
        acc["sky"].append(obs.sky)
        acc["end_pose"].append(obs.pose)
        acc["q"].append(env.chain.q.copy())
    for k in keys:
        out[k] = np.array(acc[k])
    np.savez_compressed(OUT / "excavation_env.npz", **out)
    print({k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
