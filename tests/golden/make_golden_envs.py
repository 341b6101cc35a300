"""Golden fixtures for the batched bulldozer env, from the REAL reference.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_envs.py

For seeds 0..2 of ``BulldozerEnv(BulldozerEnvConfig(n_particles=400))``
(envs.py:102-230): the seeded bed, then the state rounded to float32 (the
device's resident precision) and stepped by the reference with a fixed
action per env: blade poses/twists of every substep, the state after the
first substep and after the whole control step (frame_skip substeps), and
the reward.  Saved as ``tests/golden/bulldozer_env.npz``.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

import granusim
from granusim.envs import BulldozerEnv, BulldozerEnvConfig, bulldozer_reward
from granusim.stepper import step

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731

SEEDS = [0, 1, 2]
ACTIONS = np.array([[1.0, 0.2], [0.5, -0.5], [-0.3, 1.0]])


def main():
    cfg = BulldozerEnvConfig(n_particles=400)
    out = {"seeds": np.array(SEEDS), "actions": ACTIONS, "frame_skip": cfg.frame_skip}
    x0s, x1s, v1s, xTs, vTs, poses, omegas, vels, rews, ncs = [], [], [], [], [], [], [], [], [], []
    for e, seed in enumerate(SEEDS):
        env = BulldozerEnv(cfg)
        env.reset(seed)
        sc = env.scene
        x0s.append(sc.particles.positions.copy())
        sc.particles.positions[:] = f32(sc.particles.positions)
        sc.particles.velocities[:] = f32(sc.particles.velocities)
        env.driver.command(ACTIONS[e])
        P, W, V, nc = [], [], [], []
        for k in range(cfg.frame_skip):
            env.driver.advance(sc.params.timestep)
            _, rep = step(sc)
            blade = sc.bodies[1]
            P.append(np.asarray(blade.pose, float).copy())
            W.append(np.asarray(blade.omega, float).copy())
            V.append(np.asarray(blade.v_origin, float).copy())
            nc.append(rep.n_contacts)
            if k == 0:
                x1s.append(sc.particles.positions.copy())
                v1s.append(sc.particles.velocities.copy())
        xTs.append(sc.particles.positions.copy())
        vTs.append(sc.particles.velocities.copy())
        poses.append(P)
        omegas.append(W)
        vels.append(V)
        ncs.append(nc)
        rews.append(bulldozer_reward(sc.particles.positions, env.goal))
    out.update(x0=np.array(x0s), x1=np.array(x1s), v1=np.array(v1s), xT=np.array(xTs),
               vT=np.array(vTs), blade_pose=np.array(poses), blade_omega=np.array(omegas),
               blade_v=np.array(vels), reward=np.array(rews), n_contacts=np.array(ncs))
    np.savez_compressed(OUT / "bulldozer_env.npz", **out)
    print({k: np.shape(v) for k, v in out.items()}, rews)


if __name__ == "__main__":
    main()
