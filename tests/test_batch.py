"""Batched independent environments.

CPU: the env builder and the array drivers against the reference's own
outputs (tests/golden/bulldozer_env.npz, made by make_golden_envs.py), batch
validation and env sharding.
GPU: a batch of E envs evolves exactly as E single-scene contexts (bitwise
state, exact counters), each env matches the reference / oracle, and the
on-device reward equals the host reward.
"""

import numpy as np
import pytest

from helpers import rel_err

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.batch import SceneBatch, StaticBatch, TrackSteeringBatch, shard_envs
from paper_2306_01369_b200.beds import lattice_scene
from paper_2306_01369_b200.envs import (
    BatchedBulldozerEnv,
    BulldozerEnvConfig,
    GoalBox,
    blade_base_pose,
    bulldozer_reward,
    bulldozer_scene,
)
from oracle import granular_oracle as O

from helpers import GOLDEN

TOL = 1e-5


def golden():
    with np.load(GOLDEN / "bulldozer_env.npz") as z:
        return {k: z[k] for k in z.files}


# ---------------------------------------------------------------------------
# CPU
# ---------------------------------------------------------------------------
def test_bulldozer_scene_matches_reference_seeding():
    g = golden()
    cfg = BulldozerEnvConfig(n_particles=400)
    for e, seed in enumerate(g["seeds"]):
        sc = bulldozer_scene(int(seed), cfg)
        assert np.array_equal(sc.particles.positions, g["x0"][e])
        assert [type(b.geometry).__name__ for b in sc.bodies] == ["HalfSpace", "Box"]


def test_track_steering_batch_matches_reference_driver():
    g = golden()
    cfg = BulldozerEnvConfig(n_particles=400)
    E = len(g["seeds"])
    drv = TrackSteeringBatch(np.full(E, -2.0), np.zeros(E), np.zeros(E), z=0.0,
                             base_pose=blade_base_pose(cfg))
    drv.command(g["actions"])
    P, W, V = drv.rollout(int(g["frame_skip"]), cfg.timestep, None)
    np.testing.assert_allclose(np.transpose(P, (1, 0, 2, 3)), g["blade_pose"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(np.transpose(W, (1, 0, 2)), g["blade_omega"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(np.transpose(V, (1, 0, 2)), g["blade_v"], rtol=0, atol=1e-14)


def test_track_steering_batch_equals_single_driver():
    from paper_2306_01369_b200.kinematics import TrackSteeringDriver, TrackSteeringState

    rng = np.random.default_rng(3)
    E = 5
    x, y, th = rng.normal(size=E), rng.normal(size=E), rng.normal(size=E)
    base = gg.make_pose(gg.so3_exp(np.array([0.1, 0.2, 0.3])), np.array([0.4, -0.1, 0.2]))
    acts = rng.uniform(-1.5, 1.5, size=(E, 2))
    b = TrackSteeringBatch(x, y, th, z=0.3, scale_v=1.3, scale_omega=0.7, base_pose=base)
    b.command(acts)
    P, W, V = b.rollout(4, 2e-3, None)
    for e in range(E):
        d = TrackSteeringDriver(state=TrackSteeringState(x[e], y[e], th[e]), z=0.3, scale_v=1.3,
                                scale_omega=0.7, base_pose=base)
        d.command(acts[e])
        for k in range(4):
            d.advance(2e-3)
            np.testing.assert_allclose(P[k, e], d.pose_at(0.0), rtol=0, atol=1e-13)
            om, vo = d.twist_at(0.0)
            np.testing.assert_allclose(W[k, e], om, rtol=0, atol=1e-13)
            np.testing.assert_allclose(V[k, e], vo, rtol=0, atol=1e-13)


def test_host_reward_matches_reference_formula():
    g = golden()
    goal = GoalBox(BulldozerEnvConfig().goal_min, BulldozerEnvConfig().goal_max)
    for e in range(len(g["seeds"])):
        assert bulldozer_reward(g["xT"][e], goal) == pytest.approx(g["reward"][e], rel=0, abs=1e-12)
    with pytest.raises(ValueError):
        bulldozer_reward(np.zeros((0, 3)), goal)
    with pytest.raises(ValueError):
        GoalBox([0, 0, 0], [1, 0, 1])


def test_shard_envs_partitions():
    for world in (1, 2, 3, 8):
        parts = [shard_envs(4096, r, world) for r in range(world)]
        allv = np.sort(np.concatenate(parts))
        assert np.array_equal(allv, np.arange(4096))
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_scene_batch_validation_before_device():
    a = lattice_scene(100)
    b = lattice_scene(120)
    with pytest.raises(ValueError, match="particles"):
        SceneBatch([a, b])
    c = lattice_scene(100, friction=0.3)
    with pytest.raises(ValueError, match="params"):
        SceneBatch([a, c])
    d = lattice_scene(100)
    d.hashmap_size = 64
    with pytest.raises(ValueError, match="hash table"):
        SceneBatch([a, d])
    with pytest.raises(ValueError):
        SceneBatch([])
    with pytest.raises(ValueError, match="envs"):
        SceneBatch([a, lattice_scene(100)], body_drivers={0: StaticBatch(3)})


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
def _mixed_scenes(E, n=700):
    """E different beds of n particles: lattices of different seeds and
    densities, with a floor and a moving box."""
    out = []
    for e in range(E):
        sc = lattice_scene(n, seed=e, timestep=5e-4)
        sc.particles.positions = sc.particles.positions + np.array([0.013 * e, -0.007 * e, 0.0])
        sc.particles.velocities = np.random.default_rng(e).normal(scale=0.2, size=(n, 3))
        drv = gg.SpinDriver(axis=np.array([0.0, 0.0, 1.0]), rate=2.0 + e,
                            center=np.array([0.3, 0.3, 0.0]),
                            base_pose=gg.make_pose(np.eye(3), np.array([0.45, 0.3, 0.2])))
        sc.bodies.append(gg.RigidBody(gg.Box(np.array([0.15, 0.1, 0.04])), driver=drv, name="tool"))
        out.append(sc)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 3])
def test_batch_equals_single_contexts_bitwise(mode):
    from paper_2306_01369_b200 import _native as N

    E, T = 6, 12
    scenes = _mixed_scenes(E)
    singles = _mixed_scenes(E)
    batch = SceneBatch(scenes)
    N.check(batch.ctx, N.lib().gg_set_solve_mode(batch.ctx, mode), "mode")
    reps, bm = batch.run_raw(T)
    xb, vb = batch.state()
    for e in range(E):
        sc = singles[e]
        _, rs = gg.run(sc, T)
        assert np.array_equal(sc.particles.positions, xb[e]), e
        assert np.array_equal(sc.particles.velocities, vb[e]), e
        for k in (0, T - 1):
            r = rs[k]
            assert reps[k, e]["n_contacts"] == r.n_contacts
            assert reps[k, e]["n_candidates"] == r.n_candidates
            assert reps[k, e]["n_body_contacts"] == r.n_body_contacts
            assert reps[k, e]["max_penetration"] == r.max_penetration
            assert reps[k, e]["max_cone_violation"] == r.max_cone_violation
            assert reps[k, e]["kinetic_energy"] == pytest.approx(r.kinetic_energy, rel=1e-9)
            np.testing.assert_allclose(bm[k, e], r.body_momentum, rtol=0, atol=1e-9)
    assert reps["n_contacts"].min() > 0
    batch.close()


@pytest.mark.gpu
def test_batch_single_step_matches_oracle_per_env():
    E = 4
    scenes = _mixed_scenes(E, n=1500)
    x0 = [np.asarray(sc.particles.positions, np.float32).astype(np.float64) for sc in scenes]
    v0 = [np.asarray(sc.particles.velocities, np.float32).astype(np.float64) for sc in scenes]
    batch = SceneBatch(scenes)
    reps, _ = batch.run_raw(1)
    xb, vb = batch.state()
    for e in range(E):
        sc = scenes[e]
        bodies = []
        for b in sc.bodies:
            b.update(sc.params.timestep)
            bodies.append(b)
        x1, v1, orep, _, _ = O.step(x0[e], v0[e], sc.params, bodies, gg.default_table_size(1500))
        assert int(reps[0, e]["n_contacts"]) == orep["n_contacts"]
        assert int(reps[0, e]["n_candidates"]) == orep["n_candidates"]
        assert int(reps[0, e]["n_body_contacts"]) == orep["n_body_contacts"]
        assert rel_err(xb[e], x1) <= TOL and rel_err(vb[e], v1) <= TOL


@pytest.mark.gpu
def test_batched_bulldozer_env_matches_reference():
    """One control step (frame_skip substeps) of 3 envs vs the reference:
    first substep teacher-forced to 1e-5; the whole control step and the
    reward as bulk statistics."""
    g = golden()
    cfg = BulldozerEnvConfig(n_particles=400)
    env = BatchedBulldozerEnv(len(g["seeds"]), cfg)
    env.reset(g["seeds"])
    env.driver.command(g["actions"])
    reps, _ = env.batch.run_raw(1)
    xb, vb = env.batch.state()
    for e in range(len(g["seeds"])):
        assert rel_err(xb[e], g["x1"][e]) <= TOL
        assert rel_err(vb[e], g["v1"][e]) <= TOL
        assert int(reps[0, e]["n_contacts"]) == int(g["n_contacts"][e, 0])
    # remaining substeps of the control step
    reps, _ = env.batch.run_raw(int(g["frame_skip"]) - 1)
    xb, _ = env.batch.state()
    rew, ins = env.goal_stats()
    for e in range(len(g["seeds"])):
        assert rel_err(xb[e], g["xT"][e]) <= 1e-3
        assert rew[e] == pytest.approx(bulldozer_reward(xb[e], env.goal), rel=1e-12, abs=1e-12)
        assert abs(rew[e] - g["reward"][e]) <= 1e-3 * abs(g["reward"][e])
    assert ins.shape == (3,)
    env.close()


@pytest.mark.gpu
def test_batched_bulldozer_env_api():
    env = BatchedBulldozerEnv(8, BulldozerEnvConfig(n_particles=300))
    obs = env.reset()
    assert obs.pose.shape == (8, 3) and obs.ego.shape == (8, 36, 36) and obs.sky.shape == (8, 36, 72)
    obs, rew, done, info = env.step(np.tile([1.0, 0.0], (8, 1)))
    assert obs.pose.shape == (8, 3) and rew.shape == (8,) and done.shape == (8,)
    assert np.all(obs.pose[:, 0] > -2.0)  # vehicles drove forward
    assert np.all(obs.sky < env.config.far)  # the ground is under the whole sky view
    assert np.all(obs.ego > 0)
    assert np.all(info["t"] == pytest.approx(10 * 2e-3))
    with pytest.raises(ValueError):
        env.step(np.zeros((8, 3)))
    with pytest.raises(ValueError):
        env.step(np.full((8, 2), np.nan))
    env.close()


class _Replay(gg.StaticDriver):
    """Replays recorded per-step poses/twists (step k at t = (k+1) dt)."""

    def __init__(self, P, W, V, dt):
        super().__init__()
        self.P, self.W, self.V, self.dt = P, W, V, dt

    def _k(self, t):
        return int(round(t / self.dt)) - 1

    def pose_at(self, t):
        return self.P[self._k(t)]

    def twist_at(self, t):
        k = self._k(t)
        return self.W[k].copy(), self.V[k].copy()


@pytest.mark.gpu
def test_large_batch_sampled_envs_match_singles():
    """256 envs x 2000 particles (the config-3 env size) in one context:
    sampled envs' counters and states equal single-context runs fed the same
    blade poses."""
    # a utility context first (as when the parity tests run before this one):
    # it moves the batch's allocations, which exposed an out-of-bounds write
    # of the per-sweep commit kernel into the neighbouring buffer
    gg.spatial_hash(np.zeros((1, 3), np.int64), 64)
    cfg = BulldozerEnvConfig(n_particles=2000, radius=0.025)
    E, T = 256, 80  # the bed reaches the floor after ~60 substeps
    env = BatchedBulldozerEnv(E, cfg)
    env.reset(np.arange(E))
    # host-posed blades (the replayed singles get the same poses bit for bit;
    # the device drivers' sin/cos may differ in the last bit, tested apart)
    env.batch.driven = None
    acts = np.random.default_rng(0).uniform(-1, 1, size=(E, 2))
    env.driver.command(acts)
    twin = TrackSteeringBatch(np.full(E, -2.0), np.zeros(E), np.zeros(E), z=0.0,
                              base_pose=blade_base_pose(cfg))
    twin.command(acts)
    P, W, V = twin.rollout(T, cfg.timestep, None)
    reps, _ = env.batch.run_raw(T)
    xb, vb = env.batch.state()
    assert reps["n_contacts"][-1].min() > 0 and reps["n_body_contacts"][-1].min() > 0
    for e in (0, 77, 255):
        sc = bulldozer_scene(e, cfg)
        sc.bodies[1].driver = _Replay(P[:, e], W[:, e], V[:, e], cfg.timestep)
        for k in range(T):
            _, r = gg.step(sc)
            assert int(reps[k, e]["n_contacts"]) == r.n_contacts
            assert int(reps[k, e]["n_body_contacts"]) == r.n_body_contacts
        assert np.array_equal(sc.particles.positions, xb[e])
        assert np.array_equal(sc.particles.velocities, vb[e])
    assert env.batch.kernel_launches() > 0
    env.close()


def _shard_worker(rank, world, port, out):
    import os

    import torch.distributed as td

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_envs(64, rank, world)
    cfg = BulldozerEnvConfig(n_particles=300)
    sums = [float(bulldozer_scene(int(e), cfg).particles.positions.sum()) for e in mine]
    parts = [None] * world
    td.all_gather_object(parts, (mine.tolist(), sums))
    out[rank] = parts
    td.destroy_process_group()


def test_env_sharding_gloo_world2():
    """The multi-GPU env path has no collective on the data path: every rank
    builds exactly its shard (env e -> rank e mod N) and the union over ranks
    is the whole batch, each env seeded as on one rank."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.spawn(_shard_worker, args=(2, port, out), nprocs=2, join=True)
    parts = out[0]
    ids = sorted(i for p in parts for i in p[0])
    assert ids == list(range(64))
    cfg = BulldozerEnvConfig(n_particles=300)
    for p in parts:
        for e, sm in zip(p[0], p[1]):
            assert sm == float(bulldozer_scene(e, cfg).particles.positions.sum())


# ---------------------------------------------------------------------------
# Excavation env (the 7-joint arm + Box scoop, envs.py:233-348)
# ---------------------------------------------------------------------------
def golden_exc():
    with np.load(GOLDEN / "excavation_env.npz") as z:
        return {k: z[k] for k in z.files}


def test_excavation_scene_matches_reference_seeding():
    from paper_2306_01369_b200.envs import excavation_scene

    g = golden_exc()
    for e, seed in enumerate(g["seeds"]):
        sc = excavation_scene(int(seed))
        assert np.array_equal(sc.particles.positions, g["x0"][e])
        assert [type(b.geometry).__name__ for b in sc.bodies] == ["HalfSpace", "Box"]


def test_chain_batch_matches_reference_chain():
    from paper_2306_01369_b200.batch import ChainBatch
    from paper_2306_01369_b200.envs import excavation_links

    g = golden_exc()
    E = len(g["seeds"])
    chain = ChainBatch(excavation_links(), E, link_index=6)
    chain.command(np.clip(g["actions"], -1, 1) * chain.limits)
    P, W, V = chain.rollout(10, 2e-3, None)
    np.testing.assert_allclose(np.transpose(P, (1, 0, 2, 3)), g["scoop_pose"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.transpose(W, (1, 0, 2)), g["scoop_omega"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.transpose(V, (1, 0, 2)), g["scoop_v"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(chain.q, g["q"], rtol=0, atol=1e-15)


@pytest.mark.gpu
def test_batched_excavation_env_matches_reference():
    from paper_2306_01369_b200.envs import BatchedExcavationEnv

    g = golden_exc()
    E = len(g["seeds"])
    env = BatchedExcavationEnv(E)
    env.reset(g["seeds"])
    env.chain.command(np.clip(g["actions"], -1, 1) * env.chain.limits)
    env.batch.run_raw(1)
    xb, vb = env.batch.state()
    for e in range(E):
        assert rel_err(xb[e], g["x1"][e]) <= TOL and rel_err(vb[e], g["v1"][e]) <= TOL
    env.batch.run_raw(9)
    obs = env._observe()
    xb, _ = env.batch.state()
    for e in range(E):
        assert rel_err(xb[e], g["xT"][e]) <= 1e-3
        np.testing.assert_allclose(obs.pose[e], g["end_pose"][e], rtol=0, atol=1e-9)
        for img, ref in ((obs.ego[e], g["ego"][e]), (obs.sky[e], g["sky"][e])):
            bad = np.abs(img.astype(np.float64) - ref) > 2e-4
            assert bad.mean() <= 0.01
    obs, rew, done, info = env.step(np.zeros((E, 7)))
    assert np.all(rew == 0) and obs.ego.shape == (E, 36, 36)
    env.close()


def test_closed_form_body_aabb_matches_corners():
    """SceneBatch._fill's world AABB (centre R c + t, half extents |R| h) is the
    min / max of the 8 transformed contact-box corners up to rounding (CPU)."""
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.batch import SceneBatch, _BodySlot, so3_exp_batch

    T, E = 3, 50
    rng = np.random.default_rng(3)
    lo = rng.uniform(-1, 0, (E, 3))
    hi = lo + rng.uniform(0.1, 1, (E, 3))
    corners = np.stack([[np.where([i & 4, i & 2, i & 1], hi[e], lo[e]) for i in range(8)]
                        for e in range(E)])
    slot = _BodySlot(kind=np.ones(E, np.int32), shape=np.zeros((E, 4)), grid_id=np.zeros(E, np.int32),
                     corners=corners)
    P = np.zeros((T, E, 4, 4))
    P[..., :3, :3] = so3_exp_batch(rng.normal(size=(T * E, 3))).reshape(T, E, 3, 3)
    P[..., :3, 3] = rng.normal(size=(T, E, 3))
    P[..., 3, 3] = 1.0
    col = np.zeros((T, E), dtype=N.BODY_DTYPE)
    SceneBatch._fill(col, slot, P, np.zeros((T, E, 3)), np.zeros((T, E, 3)))
    world = np.einsum("eci,teji->tecj", corners, P[..., :3, :3]) + P[..., None, :3, 3]
    assert np.abs(col["aabb_lo"] - world.min(axis=2)).max() <= 1e-14
    assert np.abs(col["aabb_hi"] - world.max(axis=2)).max() <= 1e-14
    assert (col["bounded"] == 1).all()


@pytest.mark.gpu
@pytest.mark.parametrize("env_kind", ["bulldozer", "excavation"])
def test_device_drivers_match_host_tables(env_kind):
    """The device-resident drivers (gg_drive_track / gg_drive_chain) pose the
    bodies like the host batch drivers: the same batch run once with host
    body tables and once with device-generated rows gives the same state
    (to the last bits of sin/cos), and the drivers' states agree."""
    from paper_2306_01369_b200.envs import BatchedBulldozerEnv, BatchedExcavationEnv

    E = 6
    outs = []
    for device in (False, True):
        env = BatchedBulldozerEnv(E, render=False) if env_kind == "bulldozer" else BatchedExcavationEnv(E)
        env.reset(np.arange(E))
        if not device:
            env.batch.driven = None
            env.device_drivers = False
        rng = np.random.default_rng(1)
        for _ in range(3):
            a = rng.uniform(-1, 1, (E, 2 if env_kind == "bulldozer" else 7))
            if env_kind == "bulldozer":
                env.driver.command(a)
            else:
                env.chain.command(np.clip(a, -1, 1) * env.chain.limits)
            env.batch.run_raw(10)
        x, v = env.batch.state()
        drv = env.driver if env_kind == "bulldozer" else env.chain
        st = np.stack([drv.x, drv.y, drv.theta], 1) if env_kind == "bulldozer" else drv.q
        outs.append((x, v, st))
        env.close()
    (x0, v0, s0), (x1, v1, s1) = outs
    np.testing.assert_allclose(s1, s0, rtol=0, atol=1e-12)
    for e in range(E):
        assert rel_err(x1[e], x0[e]) <= TOL and rel_err(v1[e], v0[e]) <= 1e-3
