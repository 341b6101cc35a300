"""The reference's L1 entry points on the device:
candidate_pairs, query_candidates, narrowphase_candidates / CandidateContacts,
narrowphase_contacts / ContactSet / Contact, solve_contacts_pja,
project_friction_cone, position_cells.

Two kinds of checks:
  * against tests/golden/l1_api.npz, made by running the real reference
    (tests/golden/make_golden_l1.py) on float64 inputs: candidate lists,
    contact sets (order included) and every integer field bit-exact, float64
    geometry and impulses to float64 rounding (the device uses CUDA's hypot
    and a fixed-point body-momentum sum, so the last bits may differ);
  * the reference's own unit tests for these functions restated against this
    package (tests/test_broadphase.py:87-180, tests/test_contact.py:37-249 of
    the reference).
"""

import numpy as np
import pytest

from helpers import load

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.broadphase import EMPTY, build_hashmap, candidate_pairs, query_candidates
from paper_2306_01369_b200.contact import (
    Contact,
    ContactSet,
    SolverError,
    make_contact_frame,
    narrowphase_candidates,
    narrowphase_contacts,
    detect_contacts,
    project_friction_cone,
    solve_contacts_pja,
)
from paper_2306_01369_b200.kinematics import ScriptedDriver, StaticDriver, identity_pose, make_pose, so3_exp
from paper_2306_01369_b200.scene import MaterialParams, RigidBody
from paper_2306_01369_b200.sdf import Box, HalfSpace

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------
# golden fixture (real reference, float64 inputs)
# ---------------------------------------------------------------------------
def _golden_bodies(g):
    """Bodies frozen at the recorded poses/twists (make_golden_l1.bodies)."""
    from helpers import FixedTwistDriver

    slope_n = np.array([0.1, 0.0, 1.0]) / np.linalg.norm([0.1, 0.0, 1.0])
    geoms = [HalfSpace(), HalfSpace(normal=slope_n), Box(np.array([0.12, 0.06, 0.05]))]
    out = []
    for b, geom in enumerate(geoms):
        body = RigidBody(geom, FixedTwistDriver(g["body_poses"][b], g["body_omega"][b], g["body_vel"][b]),
                         name=f"b{b}")
        body.update(0.01)
        out.append(body)
    return out


@pytest.fixture(scope="module")
def G():
    return load("l1_api")


def test_build_hashmap_and_candidates_bit_exact(G):
    r, n_h = float(G["radius"]), int(G["n_h"])
    hm = build_hashmap(G["pos"], r, n_h)
    assert np.array_equal(hm.cells, G["cells"])
    assert np.array_equal(hm.hashes, G["hashes"])
    assert np.array_equal(hm.table, G["table"])
    assert np.array_equal(hm.next, G["next"])
    ci, cj = candidate_pairs(hm)
    assert np.array_equal(ci, G["ci"]) and np.array_equal(cj, G["cj"])
    hm64 = build_hashmap(G["pos"], r, 64)  # heavy aliasing: de-duplicated buckets
    assert np.array_equal(hm64.table, G["table64"]) and np.array_equal(hm64.next, G["next64"])
    ci, cj = candidate_pairs(hm64)
    assert np.array_equal(ci, G["ci64"]) and np.array_equal(cj, G["cj64"])


def test_narrowphase_candidates_matches_reference(G):
    bodies = _golden_bodies(G)
    cand = narrowphase_candidates(G["pos"], float(G["radius"]), G["ci"], G["cj"], bodies)
    for f in ("owner", "kind", "other", "colliding"):
        assert np.array_equal(getattr(cand, f), G[f"cand_{f}"]), f
    assert [cand.n_pp_candidates, cand.n_coincident, cand.n_degenerate] == G["cand_counts"].tolist()
    for f in ("e1", "psi", "vj"):
        np.testing.assert_allclose(getattr(cand, f), G[f"cand_{f}"], rtol=0, atol=1e-15, err_msg=f)


def test_narrowphase_contacts_order_and_values(G):
    bodies = _golden_bodies(G)
    hm = build_hashmap(G["pos"], float(G["radius"]), int(G["n_h"]))
    cs = narrowphase_contacts(G["pos"], float(G["radius"]), hm, bodies)
    for f in ("owner", "kind", "other"):  # the reference's ContactSet order, exactly
        assert np.array_equal(getattr(cs, f), G[f"cs_{f}"]), f
    assert [cs.n_pp_candidates, cs.n_coincident, cs.n_degenerate] == G["cs_counts"].tolist()
    for f in ("e1", "e2", "e3", "psi", "vj"):
        np.testing.assert_allclose(getattr(cs, f), G[f"cs_{f}"], rtol=0, atol=1e-15, err_msg=f)
    # body contacts carry the surface velocity of the moving bodies
    assert np.abs(cs.vj[cs.kind == 1]).max() > 0.1
    c = cs[5]
    assert isinstance(c, Contact) and c.i == int(G["cs_owner"][5]) and c.j == int(G["cs_other"][5])
    assert np.allclose(c.frame @ c.e1, [1, 0, 0], atol=1e-12)
    assert len(list(iter(cs))) == len(cs)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max())))


@pytest.mark.parametrize("variant", ["plain", "mask", "gamma"])
def test_solve_contacts_pja_matches_reference(G, variant):
    bodies = _golden_bodies(G)
    r = float(G["radius"])
    hm = build_hashmap(G["pos"], r, int(G["n_h"]))
    if variant == "mask":
        cs = narrowphase_candidates(G["pos"], r, G["ci"], G["cj"], bodies)
        params = MaterialParams(friction=0.4)
        buf = solve_contacts_pja(cs, G["vel"], params, n_bodies=3, inline_narrowphase_mask=True)
        sfx = "_mask"
    else:
        cs = narrowphase_contacts(G["pos"], r, hm, bodies)
        params = (MaterialParams(friction=0.4) if variant == "plain"
                  else MaterialParams(friction=0.3, gamma=0.8, solver_iterations=6))
        buf = solve_contacts_pja(cs, G["vel"], params, n_bodies=3)
        sfx = "" if variant == "plain" else "_gamma"
    # float64 arithmetic in numpy's order; 10 Jacobi sweeps of a deeply
    # overlapping blob amplify last-bit differences (CUDA hypot) ~1e3x
    assert _rel(buf.delta_v, G["dv" + sfx]) <= 1e-11
    assert _rel(buf.body_momentum, G["bm" + sfx]) <= 1e-9
    d = G["diag" + sfx]
    assert buf.max_cone_violation == pytest.approx(d[0], rel=1e-9, abs=1e-12)
    assert buf.min_normal_impulse == pytest.approx(d[1], rel=1e-9, abs=1e-15)
    assert buf.n_contacts == int(d[2])


def test_solve_refresh_candidates_equals_plain(G):
    """ONE_LOOP cost profile (refresh every sweep) gives the same result."""
    bodies = _golden_bodies(G)
    r = float(G["radius"])
    cand = narrowphase_candidates(G["pos"], r, G["ci"], G["cj"], bodies)
    params = MaterialParams(friction=0.4)
    calls = []

    def refresh():
        calls.append(1)
        return narrowphase_candidates(G["pos"], r, G["ci"], G["cj"], bodies)

    a = solve_contacts_pja(cand, G["vel"], params, n_bodies=3, inline_narrowphase_mask=True)
    b = solve_contacts_pja(cand, G["vel"], params, n_bodies=3, inline_narrowphase_mask=True,
                           refresh_candidates=refresh)
    assert len(calls) == params.solver_iterations - 1
    assert np.array_equal(a.delta_v, b.delta_v)
    assert np.array_equal(a.body_momentum, b.body_momentum)


def test_project_friction_cone_matches_reference(G):
    out = project_friction_cone(G["cone_b"], 0.5, G["cone_psi"], 0.2, 1e-3)
    np.testing.assert_allclose(out, G["cone"], rtol=1e-15, atol=1e-15)


def test_query_candidates_vs_chain_walk(G):
    hm = build_hashmap(G["pos"], float(G["radius"]), 64)
    ci, cj = candidate_pairs(hm)
    for i in (0, 17, 311, 599):
        got = query_candidates(hm, G["pos"], i)
        assert sorted(got) == sorted(cj[ci == i].tolist())


# ---------------------------------------------------------------------------
# reference unit tests restated (tests/test_broadphase.py, tests/test_contact.py)
# ---------------------------------------------------------------------------
def _solve(positions, velocities, params, bodies=(), **kw):
    positions = np.asarray(positions, dtype=np.float64)
    m = build_hashmap(positions, params.radius, gg.default_table_size(len(positions)))
    ci, cj = candidate_pairs(m)
    cand = narrowphase_candidates(positions, params.radius, ci, cj, list(bodies))
    return solve_contacts_pja(ContactSet(cand), np.asarray(velocities, float), params,
                              n_bodies=len(bodies), **kw)


def _static_halfspace(normal=(0, 0, 1)):
    return RigidBody(HalfSpace(normal=np.asarray(normal, float)), StaticDriver(identity_pose()),
                     name="floor")


def _brute_pairs(pos, r):
    d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1)
    i, j = np.nonzero(np.triu(d2 <= (2 * r) ** 2, 1))
    return set(zip(i.tolist(), j.tolist()))


class TestBroadphaseReference:
    def test_two_in_one_cell(self):
        pos = np.array([[0.01, 0.0, 0.0], [0.02, 0.0, 0.0]])
        m = build_hashmap(pos, 0.05, 8)
        h = gg.spatial_hash(gg.position_cells(pos, 0.05)[0], 8)
        assert sorted(m.chain(h)) == [0, 1]

    def test_partition_invariant(self):
        rng = np.random.default_rng(11)
        pos = rng.uniform(-1, 1, size=(300, 3))
        m = build_hashmap(pos, 0.05, 128)
        seen = []
        for h in range(128):
            seen.extend(m.chain(h))
        assert sorted(seen) == list(range(300))

    def test_chain_multisets_match_serial_insertion(self):
        rng = np.random.default_rng(3)
        pos = rng.uniform(-2, 2, size=(500, 3))
        n_h = 256
        m = build_hashmap(pos, 0.05, n_h)
        cells = gg.position_cells(pos, 0.05)
        table = np.full(n_h, EMPTY, dtype=np.int64)
        nxt = np.full(len(pos), EMPTY, dtype=np.int64)
        for i in range(len(pos)):  # the literal head-insertion loop
            h = gg.spatial_hash(cells[i], n_h)
            nxt[i] = table[h]
            table[h] = i
        assert np.array_equal(m.table, table) and np.array_equal(m.next, nxt)

    def test_insertion_order_changes_chains_not_sets(self):
        rng = np.random.default_rng(5)
        pos = rng.uniform(-1, 1, size=(100, 3))
        m1 = build_hashmap(pos, 0.05, 64)
        m2 = build_hashmap(pos, 0.05, 64, insertion_order=rng.permutation(100))
        for h in range(64):
            assert sorted(m1.chain(h)) == sorted(m2.chain(h))

    def test_touching_pair_found_both_ways(self):
        r = 0.05
        pos = np.array([[0.0, 0.0, 0.0], [1.9 * r, 0.0, 0.0]])
        m = build_hashmap(pos, r, 16)
        assert 1 in query_candidates(m, pos, 0)
        assert 0 in query_candidates(m, pos, 1)

    def test_superset_of_brute_force(self):
        rng = np.random.default_rng(17)
        pos = rng.uniform(0, 1, size=(500, 3))
        r = 0.03
        m = build_hashmap(pos, r, gg.default_table_size(500))
        ci, cj = candidate_pairs(m)
        cand = set(zip(ci.tolist(), cj.tolist()))
        for i, j in _brute_pairs(pos, r):
            assert (i, j) in cand and (j, i) in cand

    def test_candidate_pairs_match_query_per_particle(self):
        rng = np.random.default_rng(23)
        pos = rng.uniform(0, 0.5, size=(200, 3))
        m = build_hashmap(pos, 0.04, 128)
        ci, cj = candidate_pairs(m)
        for i in range(200):
            assert set(cj[ci == i].tolist()) == set(query_candidates(m, pos, i))

    def test_empty_hashmap(self):
        m = build_hashmap(np.zeros((0, 3)), 0.05, 16)
        ci, cj = candidate_pairs(m)
        assert len(ci) == len(cj) == 0


class TestContactReference:
    def test_separated_pair_no_contact(self):
        r = 0.05
        pos = np.array([[0, 0, 0], [2.1 * r, 0, 0]], float)
        assert len(detect_contacts(pos, r, build_hashmap(pos, r, 16))) == 0

    def test_overlapping_pair_both_owners(self):
        r = 0.05
        pos = np.array([[0, 0, 0], [1.8 * r, 0, 0]], float)
        contacts = detect_contacts(pos, r, build_hashmap(pos, r, 16))
        assert len(contacts) == 2
        by_owner = {c.i: c for c in contacts}
        assert by_owner[0].psi == pytest.approx(0.2 * r)
        assert np.allclose(by_owner[0].e1, -by_owner[1].e1)
        assert np.allclose(by_owner[1].e1, [1, 0, 0])

    def test_settled_column_equals_brute_force(self):
        rng = np.random.default_rng(9)
        r = 0.05
        pos = rng.uniform(0, 0.8, size=(500, 3))
        got = detect_contacts(pos, r, build_hashmap(pos, r, gg.default_table_size(500))).pair_set()
        d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1)
        i, j = np.nonzero(np.triu(d2 < (2 * r) ** 2, 1))
        assert got == set(zip(i.tolist(), j.tolist()))

    def test_coincident_centers_skipped(self):
        r = 0.05
        pos = np.array([[0.2, 0.2, 0.2], [0.2, 0.2, 0.2]], float)
        ci, cj = candidate_pairs(build_hashmap(pos, r, 16))
        cand = narrowphase_candidates(pos, r, ci, cj, [])
        assert cand.n_coincident == 2
        assert not cand.colliding.any()

    def test_make_contact_frame(self):
        for n in ([1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0], [0, 0, -1.0], [0.3, -0.4, 0.5]):
            e2, e3 = make_contact_frame(np.array(n))
            e1 = np.asarray(n) / np.linalg.norm(n)
            g = np.stack([e1, e2, e3])
            assert np.abs(g @ g.T - np.eye(3)).max() < 1e-9
            assert np.allclose(np.cross(e1, e2), e3, atol=1e-9)
        with pytest.raises(ValueError):
            make_contact_frame(np.zeros(3))

    # TestConeProjection (reference tests/test_contact.py:116-147)
    def test_cone_outside_rescaled(self):
        out = project_friction_cone(np.array([1.0, 3.0, 4.0]), 0.5, 0.0, 0.2, 1e-3)
        assert np.allclose(out, [1.0, 0.3, 0.4], atol=1e-12)

    def test_cone_inside_unchanged(self):
        out = project_friction_cone(np.array([1.0, 0.1, 0.0]), 0.5, 0.0, 0.2, 1e-3)
        assert np.allclose(out, [1.0, 0.1, 0.0], atol=1e-12)

    def test_cone_negative_normal_collapses(self):
        out = project_friction_cone(np.array([-2.0, 1.0, 0.0]), 0.5, 0.0, 0.2, 1e-3)
        assert np.allclose(out, [0.0, 0.0, 0.0], atol=1e-12)

    def test_cone_stabilization_bias_added(self):
        psi, alpha, dt = 0.01, 0.2, 1e-3
        out = project_friction_cone(np.array([0.0, 0.0, 0.0]), 0.5, psi, alpha, dt)
        assert out[0] == pytest.approx(alpha * psi / dt)

    def test_cone_batch_matches_scalar(self):
        rng = np.random.default_rng(2)
        bs = rng.normal(size=(50, 3))
        psis = rng.uniform(0, 0.01, size=50)
        batch = project_friction_cone(bs, 0.5, psis, 0.2, 1e-3)
        for k in range(50):
            assert np.allclose(batch[k], project_friction_cone(bs[k], 0.5, psis[k], 0.2, 1e-3), atol=1e-14)

    def test_cone_invalid_args(self):
        with pytest.raises(ValueError):
            project_friction_cone(np.zeros(3), -0.1, 0.0, 0.2, 1e-3)
        with pytest.raises(ValueError):
            project_friction_cone(np.zeros(3), 0.5, 0.0, 0.2, 0.0)

    # TestSolver / TestBodyMomentum (reference tests/test_contact.py:150-249)
    def test_no_contacts_zero_delta_v(self):
        pos = np.array([[0, 0, 0], [1.0, 0, 0]], float)
        buf = _solve(pos, np.zeros((2, 3)), MaterialParams())
        assert np.array_equal(buf.delta_v, np.zeros((2, 3)))

    def test_head_on_pair_equal_opposite(self):
        r = 0.05
        params = MaterialParams(friction=0.0, gravity=np.zeros(3))
        pos = np.array([[0, 0, 0], [1.9 * r, 0, 0]], float)
        vel = np.array([[0.3, 0, 0], [-0.3, 0, 0]])
        buf = _solve(pos, vel, params)
        assert np.allclose(buf.delta_v[0], -buf.delta_v[1], atol=1e-9)
        post = vel + buf.delta_v
        assert np.dot(post[1] - post[0], np.array([1.0, 0, 0])) >= -1e-9

    def test_resting_on_halfspace_cancels_gravity(self):
        params = MaterialParams(friction=0.5)
        r = params.radius
        pos = np.array([[0, 0, r * (1.0 - 1e-9)]], float)
        buf = _solve(pos, np.zeros((1, 3)), params, bodies=[_static_halfspace()])
        residual = params.timestep * params.gravity + buf.delta_v[0]
        assert abs(residual[2]) <= 1e-6

    def test_cone_feasibility_random_pile(self):
        rng = np.random.default_rng(21)
        params = MaterialParams(friction=0.4)
        pos = rng.uniform(0, 0.5, size=(120, 3))
        vel = rng.normal(scale=0.5, size=(120, 3))
        buf = _solve(pos, vel, params, bodies=[_static_halfspace()])
        assert buf.max_cone_violation <= 1e-9
        assert buf.min_normal_impulse >= 0.0

    def test_frame_independence(self):
        rng = np.random.default_rng(33)
        pos = rng.uniform(0, 0.4, size=(40, 3))
        vel = rng.normal(scale=0.3, size=(40, 3))
        R = so3_exp(np.array([0.4, -0.2, 0.7]))
        params = MaterialParams(friction=0.3)
        params_rot = MaterialParams(friction=0.3, gravity=R @ params.gravity)
        buf = _solve(pos, vel, params)
        buf_rot = _solve(pos @ R.T, vel @ R.T, params_rot)
        scale = max(np.abs(buf.delta_v).max(), 1e-12)
        assert np.abs(buf_rot.delta_v - buf.delta_v @ R.T).max() / scale <= 1e-6

    def test_pair_symmetry_no_gravity(self):
        r = 0.05
        params = MaterialParams(friction=0.5, gravity=np.zeros(3))
        pos = np.array([[0, 0, 0], [0, 1.7 * r, 0]], float)
        vel = np.array([[0.1, 0.2, -0.1], [-0.1, -0.2, 0.1]])
        buf = _solve(pos, vel, params)
        assert np.abs(buf.delta_v[0] + buf.delta_v[1]).max() <= 1e-9

    def test_nonfinite_velocity_raises_with_reference_text(self):
        r = 0.05
        pos = np.array([[0, 0, 0], [1.5 * r, 0, 0]], float)
        vel = np.array([[np.inf, 0, 0], [0, 0, 0]])
        with pytest.raises(SolverError, match=r"^non-finite velocity correction for particles "
                                              r"\[0, 1\] \(contacts \[0, 1\]\)$"):
            _solve(pos, vel, MaterialParams())

    def test_body_contact_uses_surface_velocity(self):
        params = MaterialParams(friction=0.0)
        r = params.radius
        body = RigidBody(HalfSpace(), ScriptedDriver(lambda t: make_pose(np.eye(3), np.array([0.0, 0.0, 0.5 * t]))),
                         name="lift")
        body.update(0.0)
        pos = np.array([[0, 0, 0.9 * r]], float)
        buf = _solve(pos, np.zeros((1, 3)), params, bodies=[body])
        static_buf = _solve(pos, np.zeros((1, 3)), params, bodies=[_static_halfspace()])
        assert buf.delta_v[0, 2] > static_buf.delta_v[0, 2] + 0.4

    def test_reaction_momentum_reported(self):
        params = MaterialParams(friction=0.0)
        r = params.radius
        pos = np.array([[0, 0, 0.5 * r]], float)
        vel = np.array([[0.0, 0.0, -1.0]])
        buf = _solve(pos, vel, params, bodies=[_static_halfspace()])
        assert buf.body_momentum.shape == (1, 3)
        assert buf.body_momentum[0, 2] == pytest.approx(-params.particle_mass * buf.delta_v[0, 2])
