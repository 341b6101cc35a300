"""Golden fixtures for the L1 entry points, made by running the REAL reference.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_l1.py

Cases (float64 inputs, NOT rounded to float32: the L1 functions take the
reference's float64 arrays and compute on them in float64):
  * build_hashmap (cells, hashes, table, next), candidate_pairs (ci, cj),
    narrowphase_candidates (every CandidateContacts field) and
    narrowphase_contacts (ContactSet arrays incl. e2, e3, vj) on a random blob
    with a static floor, a moving tilted half-space and a spinning box;
  * solve_contacts_pja on that ContactSet (delta_v, body momentum,
    diagnostics), on the masked CandidateContacts (inline mask), and with
    gamma != 1;
  * project_friction_cone on a batch with per-row psi.
Output: tests/golden/l1_api.npz.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

import granusim
from granusim.broadphase import build_hashmap, candidate_pairs, default_table_size
from granusim.contact import (
    ContactSet,
    narrowphase_candidates,
    narrowphase_contacts,
    project_friction_cone,
    solve_contacts_pja,
)
from granusim.kinematics import ScriptedDriver, StaticDriver, identity_pose, make_pose, so3_exp
from granusim.scene import MaterialParams, RigidBody
from granusim.sdf import Box, HalfSpace

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__


def bodies():
    floor = RigidBody(HalfSpace(), StaticDriver(identity_pose()), name="floor")
    R = so3_exp(np.array([0.3, -0.2, 0.1]))

    def lift(t):
        return make_pose(R, np.array([0.0, 0.0, 0.03 + 0.5 * t]))

    slope = RigidBody(HalfSpace(normal=np.array([0.1, 0.0, 1.0]) / np.linalg.norm([0.1, 0.0, 1.0])),
                      ScriptedDriver(lift), name="slope")

    def spin(t):
        return make_pose(so3_exp(np.array([0.0, 0.0, 2.0 * t + 0.4])), np.array([0.25, 0.25, 0.12]))

    box = RigidBody(Box(np.array([0.12, 0.06, 0.05])), ScriptedDriver(spin), name="box")
    out = [floor, slope, box]
    for b in out:
        b.update(0.01)
    return out


def main():
    rng = np.random.default_rng(42)
    r = 0.05
    n = 600
    pos = rng.uniform(0.0, 0.8, size=(n, 3))
    pos[:, 2] = rng.uniform(0.0, 0.4, size=n)
    vel = rng.normal(scale=0.5, size=(n, 3))
    n_h = default_table_size(n)
    hm = build_hashmap(pos, r, n_h)
    ci, cj = candidate_pairs(hm)
    bs = bodies()
    cand = narrowphase_candidates(pos, r, ci, cj, bs)
    cs = narrowphase_contacts(pos, r, hm, bs)
    cs2 = ContactSet(cand)
    assert np.array_equal(cs.owner, cs2.owner) and np.array_equal(cs.other, cs2.other)
    params = MaterialParams(friction=0.4)
    buf = solve_contacts_pja(cs, vel, params, n_bodies=len(bs))
    bufm = solve_contacts_pja(cand, vel, params, n_bodies=len(bs), inline_narrowphase_mask=True)
    params_g = MaterialParams(friction=0.3, gamma=0.8, solver_iterations=6)
    bufg = solve_contacts_pja(cs, vel, params_g, n_bodies=len(bs))
    cone_b = rng.normal(size=(64, 3))
    cone_psi = rng.uniform(0, 0.01, size=64)
    cone = project_friction_cone(cone_b, 0.5, cone_psi, 0.2, 1e-3)
    # small hash table with heavy aliasing for the candidate order
    hm64 = build_hashmap(pos, r, 64)
    ci64, cj64 = candidate_pairs(hm64)
    out = dict(
        pos=pos, vel=vel, radius=r, n_h=n_h,
        cells=hm.cells, hashes=hm.hashes, table=hm.table, next=hm.next,
        ci=ci, cj=cj, ci64=ci64, cj64=cj64, table64=hm64.table, next64=hm64.next,
        cand_owner=cand.owner, cand_kind=cand.kind, cand_other=cand.other, cand_e1=cand.e1,
        cand_psi=cand.psi, cand_vj=cand.vj, cand_colliding=cand.colliding,
        cand_counts=np.array([cand.n_pp_candidates, cand.n_coincident, cand.n_degenerate]),
        cs_owner=cs.owner, cs_kind=cs.kind, cs_other=cs.other, cs_e1=cs.e1, cs_e2=cs.e2, cs_e3=cs.e3,
        cs_psi=cs.psi, cs_vj=cs.vj,
        cs_counts=np.array([cs.n_pp_candidates, cs.n_coincident, cs.n_degenerate]),
        dv=buf.delta_v, bm=buf.body_momentum,
        diag=np.array([buf.max_cone_violation, buf.min_normal_impulse, buf.n_contacts]),
        dv_mask=bufm.delta_v, bm_mask=bufm.body_momentum,
        diag_mask=np.array([bufm.max_cone_violation, bufm.min_normal_impulse, bufm.n_contacts]),
        dv_gamma=bufg.delta_v, bm_gamma=bufg.body_momentum,
        diag_gamma=np.array([bufg.max_cone_violation, bufg.min_normal_impulse, bufg.n_contacts]),
        cone_b=cone_b, cone_psi=cone_psi, cone=cone,
        body_poses=np.stack([b.pose for b in bs]), body_omega=np.stack([b.omega for b in bs]),
        body_vel=np.stack([b.v_origin for b in bs]),
    )
    np.savez_compressed(OUT / "l1_api.npz", **out)
    print(f"l1_api: {len(ci)} candidates, {len(cs)} contacts "
          f"({int((cs.kind == 1).sum())} body), max|dv| {np.abs(buf.delta_v).max():.3g}")


if __name__ == "__main__":
    main()
