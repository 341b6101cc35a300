"""Host-side API: drivers, batched body tables, trajectory IO (CPU only)."""

import numpy as np
import pytest

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.beds import JointTrajectoryDriver, excavation_chain
from paper_2306_01369_b200.engine import Engine, default_table_size
from paper_2306_01369_b200.kinematics import SpinDriver, StaticDriver, make_pose, so3_exp


def _rows_per_step(scene, n):
    eng = Engine()
    table = np.zeros((n, len(scene.bodies)), dtype=N.BODY_DTYPE)
    t = scene.t
    for k in range(n):
        t += scene.params.timestep
        for b, body in enumerate(scene.bodies):
            body.update(t)
            eng.body_row(body, scene.params.radius, table[k, b])
    return table


def _scene():
    chain = excavation_chain((0.3, -0.2, 0.1))
    bodies = [
        gg.RigidBody(gg.HalfSpace(), StaticDriver(make_pose(so3_exp([0.1, 0.0, 0.0]), [0, 0, 0.2]))),
        gg.RigidBody(gg.Box([0.15, 0.1, 0.04]), JointTrajectoryDriver(chain, 6, qd=0.3 * np.ones(7))),
        gg.RigidBody(gg.Sphere(0.2), SpinDriver(axis=[0, 1, 1], rate=1.5, center=[0.1, 0, 0],
                                                base_pose=make_pose(np.eye(3), [0.5, 0.5, 0.5]))),
    ]
    x = np.zeros((4, 3))
    return gg.Scene(particles=gg.ParticleSet(x, x), bodies=bodies, params=gg.MaterialParams(), t=0.3)


def test_batched_body_tables_match_per_step():
    n = 12
    ref = _rows_per_step(_scene(), n)
    sc = _scene()
    table, ts = Engine().body_tables(sc, n)
    assert np.isclose(sc.t, 0.3 + n * 1e-3)
    for f in ("kind", "bounded", "grid_id"):
        assert np.array_equal(table[f], ref[f])
    for f in ("shape", "rot", "trans", "omega", "v_origin", "aabb_lo", "aabb_hi"):
        assert np.allclose(table[f], ref[f], rtol=0, atol=1e-12), f


def test_joint_trajectory_matches_chain_fk():
    chain = excavation_chain()
    qd = 0.3 * np.ones(7)
    drv = JointTrajectoryDriver(chain, 6, qd=qd)
    for t in (0.0, 0.37, 1.2):
        chain.q = qd * t
        chain.qd = qd
        poses, twists = chain.fk()
        assert np.allclose(drv.pose_at(t), poses[6], atol=1e-12)
        w, v = drv.twist_at(t)
        assert np.allclose(w, twists[6][0], atol=1e-12) and np.allclose(v, twists[6][1], atol=1e-12)


def test_default_table_size_kats():
    assert default_table_size(100) == 256
    assert default_table_size(1024) == 2048
    assert default_table_size(1) == 2
    assert default_table_size(0) == 1


def test_trajectory_roundtrip(tmp_path):
    traj = gg.Trajectory(dt=1e-3, stride=2, positions=[np.arange(6, dtype=np.float32).reshape(2, 3)] * 3,
                         velocities=[np.ones((2, 3), np.float32)] * 3)
    p = str(tmp_path / "t.traj")
    gg.save_trajectory(p, traj)
    back = gg.load_trajectory(p)
    assert back.dt == traj.dt and back.stride == 2 and len(back.positions) == 3
    assert all(np.array_equal(a, b) for a, b in zip(back.positions, traj.positions))
    with pytest.raises(ValueError, match="trajectory"):
        (tmp_path / "bad").write_bytes(b"JUNK" * 10)
        gg.load_trajectory(str(tmp_path / "bad"))


def test_validation_errors():
    with pytest.raises(gg.ValidationError):
        gg.MaterialParams(radius=0.0)
    with pytest.raises(gg.ValidationError):
        gg.ParticleSet(np.zeros((2, 3)), np.zeros((3, 3)))
    with pytest.raises(gg.ValidationError):
        gg.CyclicBoundary(1.0, 0.0)
    with pytest.raises(ValueError):
        gg.run(gg.Scene(particles=gg.ParticleSet(np.zeros((1, 3)), np.zeros((1, 3))), bodies=[],
                        params=gg.MaterialParams()), -1)


def test_step_report_fields_match_reference_names():
    names = {f for f in gg.StepReport.__dataclass_fields__}
    assert names == {"wall_time", "n_contacts", "n_candidates", "candidate_hit_rate",
                     "max_penetration", "kinetic_energy", "n_body_contacts",
                     "n_coincident_skipped", "n_degenerate_skipped", "max_cone_violation",
                     "min_normal_impulse", "body_momentum", "step_index"}


def test_gsdf_cache_matches_reference_format(tmp_path):
    """GSDF v1 grid cache (sdf.py:432-465): a file written by the reference
    loads, and saving it again reproduces the reference's bytes."""
    from helpers import GOLDEN
    from paper_2306_01369_b200.sdf import load_grid, save_grid

    src = GOLDEN / "box.gsdf"
    g = load_grid(str(src))
    assert tuple(g.values.shape) == tuple(int(d) for d in g.dims)
    out = tmp_path / "again.gsdf"
    save_grid(str(out), g)
    assert out.read_bytes() == src.read_bytes()
    bad = tmp_path / "bad.gsdf"
    bad.write_bytes(b"NOPE" + src.read_bytes()[4:])
    import pytest

    with pytest.raises(ValueError):
        load_grid(str(bad))
