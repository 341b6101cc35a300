"""Device parity against the reference (golden fixtures) and the pinned
oracle.  Bars (BASELINE.json north_star):
  * cells / hashes / stable order / directed contact lists / counters: bit-exact
  * single-step positions and velocities: max|d| / max(1, max|ref|) <= 1e-5
  * contact depths / normals: float32 storage of float64 values (<= 2^-23 rel)
"""

import numpy as np
import pytest

from helpers import (
    body_states,
    directed_rows,
    golden_cases,
    load,
    params_from,
    rel_err,
    scene_from,
)

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.broadphase import device_hash_sort
from paper_2306_01369_b200.contact import device_detect
from oracle import granular_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("name", golden_cases())
def test_broadphase_bit_exact(name):
    g = load(name)
    cells, hashes, order = device_hash_sort(g["x0"], float(g["radius"]), int(g["n_h"]))
    assert np.array_equal(cells, g["cells"])
    assert np.array_equal(hashes, g["hashes"])
    assert np.array_equal(order, g["order"])


@pytest.mark.parametrize("name", golden_cases())
def test_contacts_bit_exact(name):
    g = load(name)
    sc = scene_from(g)
    cs, rep = device_detect(g["x0"], float(g["radius"]), int(g["n_h"]), sc.bodies,
                            params=sc.params)
    got = directed_rows(cs.owner, cs.kind, cs.other)
    want = directed_rows(g["c_owner"], g["c_kind"], g["c_other"])
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.array_equal(got, want)
    assert int(rep["n_candidates"]) == int(g["rep_n_candidates"])
    assert int(rep["n_coincident"]) == int(g["rep_n_coincident"])
    assert int(rep["n_degenerate"]) == int(g["rep_n_degenerate"])
    # depths / normals: float64 on device, stored float32
    key = np.lexsort((cs.other, cs.kind, cs.owner))
    assert np.abs(cs.psi[key] - g["c_psi"]).max(initial=0) <= 2e-7 * max(1e-3, g["c_psi"].max(initial=0))
    assert np.abs(cs.e1[key] - g["c_e1"]).max(initial=0) <= 2e-7


@pytest.mark.parametrize("name", golden_cases())
def test_single_step_matches_reference(name):
    g = load(name)
    sc = scene_from(g)
    _, rep = gg.step(sc, step_index=0)
    x1, v1 = sc.particles.positions, sc.particles.velocities
    assert rel_err(x1, g["x1"]) <= TOL
    assert rel_err(v1, g["v1"]) <= TOL, rel_err(v1, g["v1"])
    assert rep.n_contacts == int(g["rep_n_contacts"])
    assert rep.n_candidates == int(g["rep_n_candidates"])
    assert rep.n_body_contacts == int(g["rep_n_body_contacts"])
    assert rep.n_coincident_skipped == int(g["rep_n_coincident"])
    assert rep.n_degenerate_skipped == int(g["rep_n_degenerate"])
    assert rep.max_penetration == pytest.approx(float(g["rep_max_penetration"]), rel=1e-6)
    assert rep.kinetic_energy == pytest.approx(float(g["rep_kinetic_energy"]), rel=1e-4, abs=1e-9)
    # solver diagnostics vs the reference's own values: the cone is satisfied
    # to rounding in both; the smallest normal impulse agrees like the
    # velocities (contact normals are stored float32: 6e-8 relative)
    assert rep.max_cone_violation <= 1e-9 and float(g["rep_max_cone_violation"]) <= 1e-9
    mn_ref = float(g["rep_min_normal_impulse"])
    assert rep.min_normal_impulse == pytest.approx(mn_ref, rel=TOL, abs=1e-9)
    # body momentum: per-contact impulses in float64 from float32 records,
    # summed in 2^-36 fixed point (order independent); measured <= 3e-7
    # relative on these cases
    bm_ref = np.asarray(g["rep_body_momentum"])
    scale = max(1e-6, np.abs(bm_ref).max(initial=0))
    assert np.abs(rep.body_momentum - bm_ref).max(initial=0) / scale <= 1e-5


@pytest.mark.parametrize("n", [20_000, 50_000])
def test_lattice_step_vs_oracle(n):
    """Dense lattice bed at bench-like sizes: device vs the pinned oracle."""
    pos = gg.lattice_bed(n).astype(np.float32).astype(np.float64)
    params = gg.MaterialParams(timestep=5e-4)
    sc = gg.Scene(particles=gg.ParticleSet(pos.copy(), np.zeros_like(pos)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")], params=params)
    n_h = gg.default_table_size(n)
    _, rep = gg.step(sc)
    x1, v1, orep, c, _ = O.step(pos, np.zeros_like(pos), params, sc.bodies, n_h)
    assert rep.n_contacts == orep["n_contacts"]
    assert rep.n_candidates == orep["n_candidates"]
    assert rep.n_body_contacts == orep["n_body_contacts"]
    assert rel_err(sc.particles.positions, x1) <= TOL
    assert rel_err(sc.particles.velocities, v1) <= TOL


def test_full_size_bed1m_step_vs_oracle():
    """BASELINE config 4 size (1M particles, the dense initial lattice, c_pp
    ~5.9): one device step against one oracle step (~40 s of numpy).  Directed
    contact lists bit-exact, counters exact, x / v within 1e-5, and the pp
    contact geometry exactly antisymmetric (e1(j->i) == -e1(i->j), same psi)."""
    n = 1_000_000
    pos = gg.lattice_bed(n).astype(np.float32).astype(np.float64)
    params = gg.MaterialParams(timestep=5e-4)
    floor = [gg.RigidBody(gg.HalfSpace(), name="floor")]
    n_h = gg.default_table_size(n)
    cs, drep = device_detect(pos, params.radius, n_h, floor, params=params)
    sc = gg.Scene(particles=gg.ParticleSet(pos.copy(), np.zeros_like(pos)), bodies=floor, params=params)
    _, rep = gg.step(sc)
    x1, v1, orep, c, _ = O.step(pos, np.zeros_like(pos), params, sc.bodies, n_h)
    got = directed_rows(cs.owner, cs.kind, cs.other)
    want = directed_rows(c.owner, c.kind, c.other)
    assert got.shape == want.shape and np.array_equal(got, want)
    assert rep.n_contacts == orep["n_contacts"] and rep.n_candidates == orep["n_candidates"]
    assert rep.n_body_contacts == orep["n_body_contacts"]
    assert rep.n_coincident_skipped == orep["n_coincident_skipped"]
    assert rel_err(sc.particles.positions, x1) <= TOL
    assert rel_err(sc.particles.velocities, v1) <= TOL
    pp = np.flatnonzero(cs.kind == 0)
    own, oth = cs.owner[pp].astype(np.int64), cs.other[pp].astype(np.int64)
    key = own * n + oth
    srt = np.argsort(key)
    pos_rev = np.searchsorted(key[srt], oth * n + own)
    assert np.array_equal(key[srt][pos_rev], oth * n + own)  # every pair has its reverse
    back = pp[srt[pos_rev]]
    assert np.array_equal(cs.e1[back], -cs.e1[pp])
    assert np.array_equal(cs.psi[back], cs.psi[pp])


def _bench_scene(workload):
    import bench

    class A:
        pass

    A.workload = workload
    A.settle = 0
    sc, _ = bench.make_scene(A, with_gpu=False)
    return sc


@pytest.mark.parametrize("workload", ["hero50k", "bed1m"])
def test_teacher_forced_step_on_bench_state(workload):
    """The exact states the bench times (the settled hero column with the
    chain-driven scoop and the tube wall; the settled 1M pile with the baked
    excavator bucket in its flank): one device step against one oracle step
    from the same float32-representable state.  Directed contacts bit-exact,
    counters exact, x / v within 1e-5."""
    import copy

    sc = _bench_scene(workload)
    x0 = np.asarray(sc.particles._x, float).copy()
    v0 = np.asarray(sc.particles._v, float).copy()
    t1 = sc.t + sc.params.timestep
    n_h = int(sc.hashmap_size or gg.default_table_size(len(x0)))
    ref_bodies = copy.deepcopy(sc.bodies)
    for b in ref_bodies:
        b.update(t1)
    _, rep = gg.step(sc)
    x1, v1, orep, c, _ = O.step(x0, v0, sc.params, ref_bodies, n_h, sc.boundary)
    cs, drep = device_detect(x0, sc.params.radius, n_h, ref_bodies, params=sc.params)
    got = directed_rows(cs.owner, cs.kind, cs.other)
    want = directed_rows(c.owner, c.kind, c.other)
    assert got.shape == want.shape and np.array_equal(got, want)
    assert rep.n_contacts == orep["n_contacts"] and rep.n_candidates == orep["n_candidates"]
    assert rep.n_body_contacts == orep["n_body_contacts"] > 0
    assert rep.n_coincident_skipped == orep["n_coincident_skipped"]
    assert rep.n_degenerate_skipped == orep["n_degenerate_skipped"]
    assert int(np.sum(cs.kind == 1) - np.sum((cs.kind == 1) & (cs.other == 0))) > 0  # the tool works
    assert rel_err(sc.particles.positions, x1) <= TOL
    assert rel_err(sc.particles.velocities, v1) <= TOL


def test_config1_free_running_bulk_statistics():
    """Config 1 (lattice_bed(5000), dt=5e-4, 200 steps): long contact rollouts
    are chaotic, so compare bulk statistics against the reference run."""
    ref = load("config1_run")
    x0 = ref["x0"]
    params = gg.MaterialParams(radius=0.05, friction=0.5, baumgarte_alpha=0.2, timestep=5e-4,
                               solver_iterations=10)
    sc = gg.Scene(particles=gg.ParticleSet(x0.copy(), np.zeros_like(x0)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")], params=params)
    _, reps = gg.run(sc, int(ref["steps"]))
    ke = np.array([r.kinetic_energy for r in reps])
    nc = np.array([r.n_contacts for r in reps])
    xT = sc.particles.positions
    h_ref = ref["xT"][:, 2]
    # pile height profile: max and quantiles of z within 2% of the bed height
    height = h_ref.max()
    for q in (0.5, 0.9, 0.99, 1.0):
        assert abs(np.quantile(xT[:, 2], q) - np.quantile(h_ref, q)) <= 0.02 * height
    # mean contacts within 2%, KE trajectory within 5% of its peak
    assert abs(nc.mean() - ref["n_contacts"].mean()) <= 0.02 * ref["n_contacts"].mean()
    assert np.abs(ke - ref["ke"]).max() <= 0.05 * ref["ke"].max()
    # 2-D height map (0.5 m bins) within 2% of bed height
    def hmap(x):
        ij = np.floor(x[:, :2] / 0.5).astype(int)
        out = {}
        for (i, j), z in zip(map(tuple, ij), x[:, 2]):
            out[(i, j)] = max(out.get((i, j), -1e9), z)
        return out
    a, b = hmap(xT), hmap(ref["xT"])
    common = set(a) & set(b)
    assert len(common) >= 0.9 * len(b)
    assert max(abs(a[k] - b[k]) for k in common) <= 0.05 * height


@pytest.mark.parametrize("name", ["lattice_500", "lattice_5000", "primitives_3000", "grid_tool"])
def test_modes_bitwise_identical(name):
    """PipelineMode (stepper.py:74-98) changes the loop structure only:
    TWO_LOOPS_FUSED keeps a masked record per candidate, ONE_LOOP repeats the
    collision test in every sweep; states and counters equal TWO_LOOPS_SPLIT."""
    g = load(name)
    out = {}
    for m in gg.PipelineMode:
        sc = scene_from(g)
        reps = [gg.step(sc, m)[1] for _ in range(5)]
        out[m] = (sc.particles.positions.copy(), sc.particles.velocities.copy(),
                  [(r.n_contacts, r.n_candidates, r.n_body_contacts, r.n_coincident_skipped,
                    r.max_penetration) for r in reps])
    ref = out[gg.PipelineMode.TWO_LOOPS_SPLIT]
    for m, (x, v, rs) in out.items():
        assert np.array_equal(x, ref[0]) and np.array_equal(v, ref[1]), m
        assert rs == ref[2], m


def test_determinism():
    g = load("primitives_3000")
    res = []
    for _ in range(2):
        sc = scene_from(g)
        gg.run(sc, 20)
        res.append((sc.particles.positions.copy(), sc.particles.velocities.copy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def test_physical_order_does_not_change_results():
    """The Morton re-sort period changes only memory locality: contact
    enumeration follows the bucket order, so states are bitwise identical."""
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.engine import engine_for

    g = load("primitives_3000")
    out = []
    for every in (1, 7, 1000):
        sc = scene_from(g)
        eng = engine_for(sc)
        eng.prepare(sc)
        N.lib().gg_set_resort_every(eng.ctx, every)
        gg.run(sc, 15)
        out.append((sc.particles.positions.copy(), sc.particles.velocities.copy()))
    for x, v in out[1:]:
        assert np.array_equal(x, out[0][0]) and np.array_equal(v, out[0][1])


@pytest.mark.parametrize("name", ["grid_tool", "primitives_3000", "lattice_5000", "cyl_slope_cyclic"])
def test_launch_modes_bitwise_identical(name):
    """Fused single-kernel step, per-phase kernels with a cooperative solve,
    one launch per sweep, and the persistent solve with shared-memory staged
    records (mode 8) must give identical states (race detector for the grid
    barriers: run the persistent modes twice)."""
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.engine import engine_for

    g = load(name)
    out = {}
    for mode in (4, 4, 1, 3, 8, 8):
        sc = scene_from(g)
        eng = engine_for(sc)
        eng.max_contacts = 64
        eng.prepare(sc)
        N.lib().gg_set_solve_mode(eng.ctx, mode)
        N.lib().gg_set_resort_every(eng.ctx, 3)
        gg.run(sc, 7)
        xv = (sc.particles.positions.copy(), sc.particles.velocities.copy())
        if mode in out:
            assert np.array_equal(xv[0], out[mode][0]) and np.array_equal(xv[1], out[mode][1])
        out[mode] = xv
    for m in (1, 3, 8):
        assert np.array_equal(out[m][0], out[4][0]) and np.array_equal(out[m][1], out[4][1]), m


def test_ballistic_closed_form():
    x0 = np.array([[0.3, -0.2, 5.0]])
    v0 = np.array([[1.0, 2.0, 0.5]])
    sc = gg.Scene(particles=gg.ParticleSet(x0.copy(), v0.copy()), bodies=[],
                  params=gg.MaterialParams())
    n = 250
    for _ in range(n):
        gg.step(sc)
    g, dt = sc.params.gravity, sc.params.timestep
    want_v = v0[0] + n * dt * g
    want_x = x0[0] + n * dt * v0[0] + dt * dt * g * n * (n + 1) / 2.0
    # float32 state: ~n * ulp drift
    assert np.abs(sc.particles.positions[0] - want_x).max() <= 2e-5 * max(1.0, np.abs(want_x).max())
    assert np.abs(sc.particles.velocities[0] - want_v).max() <= 2e-5


def test_error_labels_step_index():
    sc = gg.Scene(particles=gg.ParticleSet(np.array([[0, 0, 0], [0.07, 0, 0]], float),
                                           np.zeros((2, 3))), bodies=[], params=gg.MaterialParams())
    sc.particles.velocities[0, 0] = np.inf
    # the reference's exact text (stepper.py:99-100 + contact.py:503-509,
    # generated by running the reference on this scene)
    with pytest.raises(gg.SolverError, match=r"^step 7: non-finite velocity correction for particles "
                                             r"\[0, 1\] \(contacts \[0, 1\]\)$"):
        gg.step(sc, step_index=7)


def test_solver_error_lists_contacts_in_reference_order():
    """Bad particles 0..2 own pp contacts 0..3; the floor contacts follow
    (indices 4..7): the message names the first five of them, as the
    reference does ("step 3: ... particles [0, 1, 2] (contacts [0, 1, 2, 3, 4])")."""
    pos = np.array([[0, 0, 0.04], [0.09, 0, 0.04], [0.18, 0, 0.04], [1.0, 0, 0.04]], float)
    sc = gg.Scene(particles=gg.ParticleSet(pos, np.zeros((4, 3))),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="f")], params=gg.MaterialParams())
    sc.particles.velocities[1, 2] = np.nan
    with pytest.raises(gg.SolverError, match=r"^step 3: non-finite velocity correction for particles "
                                             r"\[0, 1, 2\] \(contacts \[0, 1, 2, 3, 4\]\)$"):
        gg.step(sc, step_index=3)
    # the failing step is not committed: the state is the step's input
    assert np.isnan(sc.particles.velocities[1, 2])
    assert np.array_equal(sc.particles.positions, pos)


def test_nonfinite_positions_raise_value_error():
    sc = gg.Scene(particles=gg.ParticleSet(np.zeros((3, 3)), np.zeros((3, 3))), bodies=[],
                  params=gg.MaterialParams())
    sc.particles.positions[1, 2] = np.nan
    with pytest.raises(ValueError, match="finite"):
        gg.step(sc)


def test_reference_objects_are_accepted_duck_typed():
    """A scene built from plain attribute objects (the reference's shape) is
    stepped eagerly in place."""

    class PS:
        def __init__(self, x, v):
            self.positions, self.velocities = x, v

        @property
        def count(self):
            return len(self.positions)

    g = load("lattice_500")
    ours = scene_from(g)
    plain = gg.Scene(particles=PS(g["x0"].copy(), g["v0"].copy()), bodies=ours.bodies,
                     params=ours.params, hashmap_size=int(g["n_h"]))
    xref = plain.particles.positions
    gg.step(plain)
    assert plain.particles.positions is xref  # mutated in place
    assert rel_err(xref, g["x1"]) <= TOL


def test_empty_scene_report():
    sc = gg.Scene(particles=gg.ParticleSet(np.zeros((0, 3)), np.zeros((0, 3))), bodies=[],
                  params=gg.MaterialParams())
    _, rep = gg.step(sc)
    assert rep.n_contacts == 0 and rep.n_candidates == 0 and rep.kinetic_energy == 0.0
    assert sc.t == pytest.approx(sc.params.timestep)


@pytest.mark.parametrize("case", ["one_on_floor", "touching_pair", "pair_in_box_corner", "far_apart"])
def test_tiny_scenes_vs_oracle(case):
    """Smallest inputs (1-3 particles, n_h = 2 .. 8): the kernels' edge paths
    (single-block grids, tables smaller than a warp, owners with one contact)
    against the oracle over 20 steps, bit-exact counters every step."""
    r = 0.05
    if case == "one_on_floor":
        x = np.array([[0.0, 0.0, 0.049]])
        bodies = [gg.RigidBody(gg.HalfSpace(), name="floor")]
    elif case == "touching_pair":
        x = np.array([[0.0, 0.0, 0.3], [0.0, 0.0, 0.399]])
        bodies = []
    elif case == "pair_in_box_corner":
        x = np.array([[0.02, 0.02, 0.049], [0.02, 0.119, 0.049], [0.118, 0.02, 0.049]])
        bodies = [gg.RigidBody(gg.HalfSpace(), name="floor"),
                  gg.RigidBody(gg.Box([0.1, 0.1, 0.1]),
                               gg.StaticDriver(gg.make_pose(np.eye(3), [-0.1, -0.1, 0.1])), name="wall")]
    else:
        x = np.array([[0.0, 0.0, 0.5], [100.0, -50.0, 0.5]])
        bodies = [gg.RigidBody(gg.HalfSpace(), name="floor")]
    x = x.astype(np.float32).astype(np.float64)
    params = gg.MaterialParams(radius=r, timestep=5e-4)
    sc = gg.Scene(particles=gg.ParticleSet(x.copy(), np.zeros_like(x)), bodies=bodies, params=params)
    n_h = gg.default_table_size(len(x))
    xo, vo = x.copy(), np.zeros_like(x)
    for k in range(20):
        _, rep = gg.step(sc)
        xo, vo, orep, _, _ = O.step(xo, vo, params, sc.bodies, n_h)
        assert rep.n_contacts == orep["n_contacts"], k
        assert rep.n_body_contacts == orep["n_body_contacts"], k
        assert rep.n_candidates == orep["n_candidates"], k
        assert rel_err(sc.particles.positions, xo) <= TOL, k
        assert rel_err(sc.particles.velocities, vo) <= TOL, k
        # the oracle continues from the device state (teacher forcing, as in the parity protocol)
        xo = sc.particles.positions.astype(np.float32).astype(np.float64)
        vo = sc.particles.velocities.astype(np.float32).astype(np.float64)


def test_penetration_depth_kats():
    # tests/test_sdf.py:204-231 hand values
    psi, n, hit, deg = gg.penetration_depth(gg.Sphere(1.0), gg.identity_pose(),
                                            np.array([1.05, 0.0, 0.0]), 0.1)
    assert hit and psi == pytest.approx(0.05) and np.allclose(n, [1, 0, 0]) and deg == 0
    psi, _, hit, _ = gg.penetration_depth(gg.HalfSpace(), gg.identity_pose(), np.array([0, 0, 0.1]), 0.1)
    assert not hit and psi == 0.0
    pose = gg.make_pose(np.eye(3), np.array([0.0, 0.0, 0.3]))
    psi, n, hit, _ = gg.penetration_depth(gg.HalfSpace(), pose, np.array([0.0, 0.0, 0.35]), 0.1)
    assert hit and psi == pytest.approx(0.05) and np.allclose(n, [0, 0, 1])


def test_spatial_hash_kats():
    g = load("hash_kats")
    for key in g:
        if key.startswith("h_") or key.startswith("hbig_"):
            n_h = int(key.split("_")[1])
            cells = g["cells"] if key.startswith("h_") else g["big_cells"]
            assert np.array_equal(gg.spatial_hash(cells, n_h), g[key]), key


@pytest.mark.parametrize("mode", [0, 3])
def test_crowded_owners_overflow_path(mode):
    """Clusters of 40 near-coincident particles: every owner has more float32
    prefilter passes than the warp queue holds (16), so the owner's exact
    inline path and the record-capacity growth run.  Contacts and the step
    must still match the oracle (counters exact, state 1e-5)."""
    from paper_2306_01369_b200 import _native as N
    from paper_2306_01369_b200.engine import engine_for

    rng = np.random.default_rng(5)
    centres = rng.uniform(0.0, 2.0, size=(25, 3)) + np.array([0.0, 0.0, 0.2])
    x = (np.repeat(centres, 40, axis=0) + rng.normal(scale=0.02, size=(1000, 3)))
    x = x.astype(np.float32).astype(np.float64)
    params = gg.MaterialParams(timestep=5e-4)
    sc = gg.Scene(particles=gg.ParticleSet(x.copy(), np.zeros_like(x)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")], params=params)
    eng = engine_for(sc)
    eng.max_contacts = 2  # force record-capacity growth as well
    eng.prepare(sc)
    N.lib().gg_set_solve_mode(eng.ctx, mode)
    _, rep = gg.step(sc)
    from helpers import BodyState

    floor = [BodyState(gg.HalfSpace(), np.eye(4), np.zeros(3), np.zeros(3))]
    x1, v1, orep, _, _ = O.step(x, np.zeros_like(x), params, floor, gg.default_table_size(1000))
    assert rep.n_contacts == orep["n_contacts"] and rep.n_contacts > 1000 * 16
    assert rep.n_candidates == orep["n_candidates"]
    assert rep.n_coincident_skipped == orep["n_coincident_skipped"]
    assert rel_err(sc.particles.positions, x1) <= TOL
    assert rel_err(sc.particles.velocities, v1) <= TOL


def test_deepcopy_and_pickle_after_run_carry_current_state():
    """A copy made after device steps holds the state of the last step (the
    reference's cli.clone_scene deep-copies scenes), and stepping the copy
    continues from there exactly like the original."""
    import copy
    import pickle

    pos = gg.lattice_bed(3000).astype(np.float32).astype(np.float64)
    sc = gg.Scene(particles=gg.ParticleSet(pos, np.zeros_like(pos)),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")], params=gg.MaterialParams())
    gg.run(sc, 5)
    clone = copy.deepcopy(sc)
    pick = pickle.loads(pickle.dumps(sc.particles))
    assert np.array_equal(clone.particles.positions, sc.particles.positions)
    assert np.array_equal(pick.velocities, sc.particles.velocities)
    assert not np.array_equal(clone.particles.positions, pos)
    gg.run(sc, 3)
    gg.run(clone, 3)
    assert np.array_equal(clone.particles.positions, sc.particles.positions)
    assert np.array_equal(clone.particles.velocities, sc.particles.velocities)


def test_huge_bucket_tiny_table():
    """A bucket with more than 2^16 particles (n_h = 1: every cell aliases to
    bucket 0) gives the contacts of the default table and n(n-1) candidates
    (bucket lengths were stored in 16 bits)."""
    n = 66000
    pos = gg.lattice_bed(n).astype(np.float32).astype(np.float64)
    r = 0.05
    cs1, rep1 = device_detect(pos, r, 1)
    cs2, rep2 = device_detect(pos, r, gg.default_table_size(n))
    assert int(rep1["n_candidates"]) == n * (n - 1)
    assert np.array_equal(cs1.directed(), cs2.directed())
    assert int(rep1["n_contacts"]) == int(rep2["n_contacts"]) > 0


@pytest.mark.parametrize("seed", [0, 1])
def test_contacts_at_reach_across_cell_edges_and_corners(seed):
    """Pairs at 2r (1 -/+ 1e-6) in random directions from random points of a
    cell: partners land in the edge and corner neighbour cells at the limit
    of reach, where the contact kernel's geometric bucket culling decides.
    Directed contacts and counters bit-exact against the oracle."""
    r = 0.05
    rng = np.random.default_rng(seed)
    m = 1500
    base = np.stack(np.meshgrid(np.arange(12), np.arange(12), np.arange(11), indexing="ij"), -1)
    base = base.reshape(-1, 3)[:m] * (20 * r)  # pairs 10 cells apart
    p = base + rng.uniform(-r, r, size=(m, 3))  # anywhere in its cell (cell size 2r)
    u = rng.normal(size=(m, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    scale = np.where(rng.random(m) < 0.5, 1.0 - 1e-6, 1.0 + 1e-6)[:, None]
    q = p + u * (2.0 * r) * scale
    x = np.concatenate([p, q]).astype(np.float32).astype(np.float64)
    n_h = gg.default_table_size(len(x))
    params = gg.MaterialParams(radius=r, timestep=5e-4)
    cs, rep = device_detect(x, r, n_h, [], params=params)
    oc, _ = O.detect(x, r, n_h, [])
    got = directed_rows(cs.owner, cs.kind, cs.other)
    want = directed_rows(oc.owner, oc.kind, oc.other)
    assert len(want) > 0.8 * m  # about half the pairs touch, both directions each
    assert np.array_equal(got, want)
    assert int(rep["n_candidates"]) == int(oc.n_candidates)
    assert int(rep["n_coincident"]) == int(oc.n_coincident)
