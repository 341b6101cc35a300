"""The drop-in boundary with the REAL reference objects (host side, CPU).

When the reference package is importable (this container:
/root/reference/pkg/src; never on the GPU box, where these tests skip), its
own Scene / RigidBody / geometry / driver / MaterialParams objects go through
the host half of the boundary exactly as ours do: the same parameter struct,
the same per-step gg_body rows (geometry kind and shape, pose, twist, world
AABB of _near_body, contact.py:187-203), the same table size
(broadphase.py:58-60).  The device half is covered by the GPU parity tests.
"""
import os
import sys

import numpy as np
import pytest

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200 import _native as N
from paper_2306_01369_b200.engine import Engine, _params_struct, default_table_size

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    import granusim

    return granusim


def _pair(ref, kind):
    """The same body built from reference objects and from ours."""
    R, O = ref, gg
    if kind == "sphere":
        return R.sdf.Sphere(0.2), O.Sphere(0.2)
    if kind == "halfspace":
        n = np.array([0.1, 0.0, 1.0]) / np.linalg.norm([0.1, 0.0, 1.0])
        return R.sdf.HalfSpace(n, 0.05), O.HalfSpace(n, 0.05)
    if kind == "box":
        return R.sdf.Box(np.array([0.15, 0.1, 0.04])), O.Box(np.array([0.15, 0.1, 0.04]))
    if kind == "cylinder":
        return R.sdf.Cylinder(0.1, 0.3), O.Cylinder(0.1, 0.3)
    return R.sdf.Tube(0.9), O.Tube(0.9)


@pytest.mark.parametrize("kind", ["sphere", "halfspace", "box", "cylinder", "tube"])
def test_reference_bodies_pack_like_ours(ref, kind):
    gr, go = _pair(ref, kind)
    base = gg.make_pose(np.eye(3), np.array([0.4, 0.3, 0.25]))
    dr = ref.kinematics.SpinDriver(axis=np.array([0.2, 0.0, 1.0]), rate=2.0,
                                   center=np.array([0.3, 0.3, 0.3]), base_pose=base)
    do = gg.SpinDriver(axis=np.array([0.2, 0.0, 1.0]), rate=2.0, center=np.array([0.3, 0.3, 0.3]),
                       base_pose=base)
    x = np.random.default_rng(0).uniform(0, 1, size=(50, 3))
    sr = ref.scene.Scene(particles=ref.scene.ParticleSet(x.copy(), np.zeros_like(x)),
                         bodies=[ref.scene.RigidBody(gr, dr)], params=ref.scene.MaterialParams())
    so = gg.Scene(particles=gg.ParticleSet(x.copy(), np.zeros_like(x)), bodies=[gg.RigidBody(go, do)],
                  params=gg.MaterialParams())
    eng = Engine()  # host-side packing only: no device context is created
    tr, ts_r = eng.body_tables(sr, 7)
    to, ts_o = eng.body_tables(so, 7)
    assert np.array_equal(ts_r, ts_o)
    for f in ("kind", "shape", "bounded", "aabb_lo", "aabb_hi"):
        assert np.array_equal(tr[f], to[f]), f
    # poses and twists: the same formulas (Rodrigues, omega x r) evaluated by
    # two implementations; equal to rounding
    for f in ("rot", "trans", "omega", "v_origin"):
        assert np.allclose(tr[f], to[f], rtol=0, atol=1e-12), f
    assert sr.t == pytest.approx(so.t)


def test_reference_params_and_table_size(ref):
    kw = dict(radius=0.04, particle_mass=0.3, friction=0.7, baumgarte_alpha=0.15, timestep=1e-3,
              solver_iterations=7, gravity=np.array([0.5, 0.0, -9.0]), gamma=0.8)
    pr = ref.scene.MaterialParams(**kw)
    po = gg.MaterialParams(**kw)
    br = ref.scene.CyclicBoundary(-1.0, 2.0)
    bo = gg.CyclicBoundary(-1.0, 2.0)
    a, b = _params_struct(pr, br), _params_struct(po, bo)
    for name, _ in N.GGParams._fields_:
        va, vb = getattr(a, name), getattr(b, name)
        if hasattr(va, "__len__"):  # ctypes arrays (gravity)
            va, vb = list(va), list(vb)
        assert va == vb, name
    for n in (1, 5, 4096, 50_000, 1_000_000):
        assert default_table_size(n) == ref.broadphase.default_table_size(n)


def test_module_attribute_dropin(ref):
    """rebinding the reference's step/run names."""
    import granusim.envs
    import granusim.stepper

    saved = (granusim.stepper.step, granusim.stepper.run, granusim.envs.step)
    try:
        granusim.stepper.step = gg.step
        granusim.envs.step = gg.step
        granusim.stepper.run = gg.run
        assert granusim.envs.step is gg.step and granusim.stepper.run is gg.run
    finally:
        granusim.stepper.step, granusim.stepper.run, granusim.envs.step = saved
