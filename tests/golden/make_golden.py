"""Generate golden fixtures by running the REAL reference implementation.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every input is rounded to float32 first (the resident precision of the
device state) and handed to the reference as float64, so the device, the
oracle and the reference see bit-identical inputs.  Outputs are saved as
``tests/golden/<case>.npz``; ``tests/golden/cases.json`` lists them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

import granusim
from granusim import sdf as rsdf
from granusim.broadphase import build_hashmap, default_table_size, position_cells, spatial_hash
from granusim.contact import narrowphase_contacts
from granusim.kinematics import ScriptedDriver, StaticDriver, make_pose, so3_exp
from granusim.meshes import make_box_mesh, make_icosphere
from granusim.scene import CyclicBoundary, MaterialParams, ParticleSet, RigidBody, Scene
from granusim.stepper import step

OUT = Path(__file__).resolve().parent
assert "/root/reference" in granusim.__file__, granusim.__file__

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731


def lattice_bed(n, r=0.05, s=0.99, jitter=0.01, seed=0):
    nx = max(int(round(n ** (1.0 / 3.0))), 1)
    nz = int(np.ceil(n / (nx * nx)))
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(nx), np.arange(nz), indexing="ij")
    idx = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3).astype(np.float64)
    rng = np.random.default_rng(seed)
    pts = idx * (2.0 * r * s) + np.array([0.0, 0.0, r * s])
    pts = pts + rng.uniform(-jitter * r, jitter * r, size=pts.shape)
    return pts[:n]


def body_record(b):
    """Geometry + state of a reference body after update(t), as plain arrays."""
    g = b.geometry
    kind = type(g).__name__
    rec = {"kind": kind, "pose": np.asarray(b.pose, float), "omega": np.asarray(b.omega, float),
           "v_origin": np.asarray(b.v_origin, float)}
    if kind == "Sphere":
        rec["radius"] = g.radius
    elif kind == "HalfSpace":
        rec["normal"] = np.asarray(g.normal, float)
        rec["offset"] = g.offset
    elif kind == "Box":
        rec["half_extents"] = np.asarray(g.half_extents, float)
    elif kind == "Cylinder":
        rec["radius"], rec["half_height"] = g.radius, g.half_height
    elif kind == "Tube":
        rec["radius"] = g.radius
    elif kind == "SdfGrid":
        rec.update(origin=g.origin, spacing=g.spacing, dims=g.dims, values=g.values)
    return rec


def pack_bodies(bodies):
    out = {}
    for i, b in enumerate(bodies):
        for k, v in body_record(b).items():
            out[f"body{i}_{k}"] = np.asarray(v)
    out["n_bodies"] = np.array(len(bodies))
    return out


def one_step_case(name, x, v, params, bodies, n_h=None, boundary=None, t0=0.0):
    x = f32(x)
    v = f32(v)
    scene = Scene(particles=ParticleSet(x.copy(), v.copy()), bodies=bodies, params=params,
                  boundary=boundary, t=t0, hashmap_size=n_h)
    nh = n_h or default_table_size(len(x))
    hm = build_hashmap(x, params.radius, nh)
    order = np.argsort(hm.hashes, kind="stable")
    # contacts at the post-update body state the step will see
    t1 = t0 + params.timestep
    for b in bodies:
        b.update(t1)
    cs = narrowphase_contacts(x, params.radius, hm, bodies)
    key = np.lexsort((cs.other, cs.kind, cs.owner))
    for b in bodies:
        b.update(t0)
    _, rep = step(scene, step_index=0)
    data = dict(
        x0=x, v0=v, n_h=np.array(nh), t0=np.array(t0),
        radius=np.array(params.radius), mass=np.array(params.particle_mass),
        friction=np.array(params.friction), alpha=np.array(params.baumgarte_alpha),
        dt=np.array(params.timestep), iters=np.array(params.solver_iterations),
        gravity=np.asarray(params.gravity, float), gamma=np.array(params.gamma),
        has_boundary=np.array(boundary is not None),
        z_min=np.array(boundary.z_min if boundary else 0.0),
        z_max=np.array(boundary.z_max if boundary else 0.0),
        cells=hm.cells, hashes=hm.hashes, order=order,
        c_owner=cs.owner[key], c_kind=cs.kind[key], c_other=cs.other[key],
        c_psi=cs.psi[key], c_e1=cs.e1[key],
        x1=scene.particles.positions, v1=scene.particles.velocities,
        rep_n_contacts=np.array(rep.n_contacts), rep_n_candidates=np.array(rep.n_candidates),
        rep_n_body_contacts=np.array(rep.n_body_contacts),
        rep_n_coincident=np.array(rep.n_coincident_skipped),
        rep_n_degenerate=np.array(rep.n_degenerate_skipped),
        rep_max_penetration=np.array(rep.max_penetration),
        rep_kinetic_energy=np.array(rep.kinetic_energy),
        rep_max_cone_violation=np.array(rep.max_cone_violation),
        rep_min_normal_impulse=np.array(rep.min_normal_impulse),
        rep_body_momentum=np.asarray(rep.body_momentum, float),
    )
    # bodies as they were during the step (t1)
    data.update(pack_bodies(scene.bodies))
    np.savez_compressed(OUT / f"{name}.npz", **data)
    print(f"{name}: n={len(x)} contacts={rep.n_contacts}+{rep.n_body_contacts} "
          f"cand={rep.n_candidates} coinc={rep.n_coincident_skipped}", file=sys.stderr)
    return name


def hash_kats():
    rng = np.random.default_rng(7)
    cells = rng.integers(-500, 500, size=(200, 3))
    big = rng.integers(-3_000_000, 3_000_000, size=(200, 3))
    out = {"cells": cells, "big_cells": big}
    for n_h in (1, 37, 64, 1000, 65536, 2**21, 2**24, 1_000_003):
        out[f"h_{n_h}"] = spatial_hash(cells, n_h)
        out[f"hbig_{n_h}"] = spatial_hash(big, n_h)
    rnd = np.array([0.5, -0.5, 1.5, -1.5, 0.4999, -0.4999, 2.5, 0.05, -0.05, 0.15])
    out["round_in"] = rnd
    out["round_cells"] = position_cells(rnd[:, None].repeat(3, axis=1), 0.5)
    out["table_sizes"] = np.array([[n, default_table_size(n)] for n in (0, 1, 2, 100, 1024, 5000,
                                                                         50_000, 1_000_000)])
    np.savez_compressed(OUT / "hash_kats.npz", **out)
    return "hash_kats"


def config1_run(n=5000, steps=200):
    """Config 1: lattice_bed(5000) + floor, dt=5e-4, 200 steps (free-running)."""
    x = f32(lattice_bed(n))
    params = MaterialParams(radius=0.05, friction=0.5, baumgarte_alpha=0.2, timestep=5e-4,
                            solver_iterations=10)
    scene = Scene(particles=ParticleSet(x.copy(), np.zeros_like(x)),
                  bodies=[RigidBody(rsdf.HalfSpace(), StaticDriver(), name="floor")], params=params)
    ke, nc, zmax = [], [], []
    for k in range(steps):
        _, rep = step(scene, step_index=k)
        ke.append(rep.kinetic_energy)
        nc.append(rep.n_contacts)
        zmax.append(scene.particles.positions[:, 2].max())
    np.savez_compressed(OUT / "config1_run.npz", x0=x, xT=scene.particles.positions,
                        vT=scene.particles.velocities, ke=np.array(ke), n_contacts=np.array(nc),
                        zmax=np.array(zmax), steps=np.array(steps))
    return "config1_run"


def main():
    cases = [hash_kats()]
    r = 0.05
    # 1. small dense lattice on a floor
    p = MaterialParams(timestep=5e-4)
    cases.append(one_step_case("lattice_500", lattice_bed(500), np.zeros((500, 3)), p,
                               [RigidBody(rsdf.HalfSpace(), StaticDriver(), name="floor")]))
    # 2. config-1 bed, first step
    cases.append(one_step_case("lattice_5000", lattice_bed(5000), np.zeros((5000, 3)), p,
                               [RigidBody(rsdf.HalfSpace(), StaticDriver(), name="floor")]))
    # 3. random moving pile against every primitive, moving box scoop
    rng = np.random.default_rng(11)
    n = 3000
    x = rng.uniform([-0.6, -0.6, 0.0], [0.6, 0.6, 0.9], size=(n, 3))
    v = rng.normal(scale=0.3, size=(n, 3))

    def scoop_path(t):
        return make_pose(so3_exp(np.array([0.2 + t, -0.4, 0.3])), np.array([0.1, 0.05 + 0.5 * t, 0.3]))

    bodies = [
        RigidBody(rsdf.HalfSpace(), StaticDriver(), name="floor"),
        RigidBody(rsdf.Box(np.array([0.15, 0.1, 0.04])), ScriptedDriver(scoop_path), name="scoop"),
        RigidBody(rsdf.Sphere(0.12), StaticDriver(make_pose(np.eye(3), np.array([-0.3, 0.25, 0.4]))),
                  name="ball"),
        RigidBody(rsdf.Tube(0.62), StaticDriver(), name="wall"),
    ]
    cases.append(one_step_case("primitives_3000", x, v, MaterialParams(friction=0.4), bodies))
    # 4. tilted half-space, capped cylinder, sphere; cyclic boundary; gamma != 1
    x = rng.uniform([-0.5, -0.5, -0.1], [0.5, 0.5, 0.8], size=(2000, 3))
    v = rng.normal(scale=0.2, size=(2000, 3))
    nrm = np.array([0.1, -0.2, 1.0])
    bodies = [
        RigidBody(rsdf.HalfSpace(normal=nrm, offset=-0.05), StaticDriver(), name="slope"),
        RigidBody(rsdf.Cylinder(0.15, 0.2), StaticDriver(
            make_pose(so3_exp(np.array([0.5, 0.1, 0.0])), np.array([0.2, -0.1, 0.35]))), name="cyl"),
    ]
    cases.append(one_step_case("cyl_slope_cyclic", x, v,
                               MaterialParams(friction=0.6, gamma=0.8, timestep=1e-3), bodies,
                               boundary=CyclicBoundary(z_min=0.0, z_max=1.0)))
    # 5. baked-grid tool (icosphere + box mesh), rotated and translated
    vi, fi = make_icosphere(2, radius=0.3)
    grid = rsdf.bake_mesh_sdf(vi, fi, 0.04)
    vb, fb = make_box_mesh([0.15, 0.1, 0.04])
    gbox = rsdf.bake_mesh_sdf(vb, fb, 0.02)
    x = rng.uniform([-0.5, -0.5, -0.2], [0.5, 0.5, 0.6], size=(2500, 3))
    bodies = [
        RigidBody(grid, StaticDriver(make_pose(so3_exp(np.array([0.3, -0.5, 0.2])),
                                               np.array([0.05, -0.02, 0.1]))), name="ico"),
        RigidBody(gbox, StaticDriver(make_pose(so3_exp(np.array([0.0, 0.4, 0.0])),
                                               np.array([0.2, 0.2, 0.35]))), name="boxgrid"),
        RigidBody(rsdf.HalfSpace(), StaticDriver(make_pose(np.eye(3), np.array([0, 0, -0.15]))),
                  name="floor"),
    ]
    cases.append(one_step_case("grid_tool", x, rng.normal(scale=0.1, size=x.shape),
                               MaterialParams(), bodies))
    # 6. non-power-of-two table, coincident particles, two far clusters (aliasing)
    x = rng.uniform(0.0, 0.6, size=(300, 3))
    x[10] = x[11]
    x[12] = x[11]
    x = np.concatenate([x, x[:50] + np.array([40.0, -30.0, 7.5])])
    cases.append(one_step_case("nonpow2_coincident", x, np.zeros_like(x), MaterialParams(), [],
                               n_h=1000))
    # 7. tiny table: heavy aliasing
    x = rng.uniform(-1, 1, size=(400, 3))
    cases.append(one_step_case("alias_nh64", x, rng.normal(size=x.shape), MaterialParams(), [],
                               n_h=64))
    cases.append(config1_run())
    (OUT / "cases.json").write_text(json.dumps(cases, indent=1))


if __name__ == "__main__":
    main()
