"""The CPU oracle against the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py from /root/reference).  CPU only."""

import numpy as np
import pytest

from helpers import body_states, boundary_from, directed_rows, golden_cases, load, params_from

from oracle import granular_oracle as O


def test_hash_kats_match_reference():
    g = load("hash_kats")
    for key in g:
        if key.startswith("h_") or key.startswith("hbig_"):
            n_h = int(key.split("_")[1])
            cells = g["cells"] if key.startswith("h_") else g["big_cells"]
            assert np.array_equal(O.cell_hash(cells, n_h), g[key]), key


def test_independent_hash_rule():
    # python-int evaluation with int64 wrap (the reference's own KAT idea,
    # tests/test_broadphase.py:20-30)
    def ref(cell, n_h):
        acc = 0
        for c, p in zip(cell, (73856093, 19349663, 83492791)):
            t = ((int(c) - 100) * p + 2**63) % 2**64 - 2**63
            acc ^= t & 0xFFFFFFFFFFFFFFFF
        acc = (acc + 2**63) % 2**64 - 2**63
        return acc % n_h

    g = load("hash_kats")
    for cell in g["big_cells"][:50]:
        for n_h in (37, 1000, 2**21):
            assert O.cell_hash(cell, n_h) == ref(cell, n_h)


def test_rounding_and_table_size_kats():
    g = load("hash_kats")
    assert np.array_equal(O.cell_coords(g["round_in"][:, None].repeat(3, 1), 0.5), g["round_cells"])
    for n, want in g["table_sizes"]:
        assert O.table_size(int(n)) == want
    # tests/test_broadphase.py:76-83
    assert np.array_equal(O.cell_coords(np.array([[-0.30, -0.01, 0.0]]), 0.05)[0], [-3, 0, 0])


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_step_matches_reference(name):
    g = load(name)
    params = params_from(g)
    x1, v1, rep, c, bp = O.step(g["x0"], g["v0"], params, body_states(g), int(g["n_h"]),
                                boundary_from(g))
    # broadphase: bit-exact
    assert np.array_equal(bp["cells"], g["cells"])
    assert np.array_equal(bp["hashes"], g["hashes"])
    assert np.array_equal(bp["order"], g["order"])
    # contacts: bit-exact directed lists, exact depths/normals
    got = directed_rows(c.owner, c.kind, c.other)
    want = directed_rows(g["c_owner"], g["c_kind"], g["c_other"])
    assert np.array_equal(got, want)
    key = np.lexsort((c.other, c.kind, c.owner))
    assert np.array_equal(c.psi[key], g["c_psi"])
    assert np.array_equal(c.e1[key], g["c_e1"])
    # counters exact
    assert rep["n_contacts"] == g["rep_n_contacts"]
    assert rep["n_candidates"] == g["rep_n_candidates"]
    assert rep["n_body_contacts"] == g["rep_n_body_contacts"]
    assert rep["n_coincident_skipped"] == g["rep_n_coincident"]
    assert rep["n_degenerate_skipped"] == g["rep_n_degenerate"]
    assert rep["max_penetration"] == g["rep_max_penetration"]
    # the solve follows the reference's array program: same results
    assert np.max(np.abs(x1 - g["x1"])) <= 1e-12
    assert np.max(np.abs(v1 - g["v1"])) <= 1e-12
    assert rep["kinetic_energy"] == pytest.approx(float(g["rep_kinetic_energy"]), rel=1e-12)
    assert np.allclose(rep["body_momentum"], g["rep_body_momentum"], rtol=1e-10, atol=1e-12)
    assert rep["min_normal_impulse"] == pytest.approx(float(g["rep_min_normal_impulse"]), abs=1e-12)


def test_config1_first_step_state_matches_run_fixture():
    run = load("config1_run")
    one = load("lattice_5000")
    assert np.array_equal(run["x0"], one["x0"])
