"""North-star criterion 3: a free-running scoop run matches the reference in
bulk statistics (pile height profile, mass transported by the scoop).

The reference ran the scene of tests/scoop_stats.py (4000-particle bed, an
open-top bucket baked from our make_bucket_mesh by the REFERENCE's baker, on
a DigDriver: a front-loader pass into the bed, a curl and a lift; 4000 steps
at dt = 5e-4) and recorded the statistics every 200 steps
(tests/golden/make_golden_scoop.py -> tests/golden/scoop_run.npz).  The
device runs the same scene from the same float32 settled state through the
public API (``run``); the bucket is baked on the device and must equal the
reference's grid bit for bit.  Long contact rollouts are chaotic (float32
state vs the reference's float64), so the runs are compared through bulk
statistics with the tolerances stated below.
"""

import numpy as np
import pytest

from helpers import load

import scoop_stats as S

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.beds import DigDriver
from paper_2306_01369_b200.meshes import make_bucket_mesh
from paper_2306_01369_b200.sdf import bake_mesh_sdf

pytestmark = pytest.mark.gpu

# tolerances (stated; north_star: "within a stated tolerance")
TOL_CARRIED = 0.15      # carried particles: |d| <= 15% of the reference's (>= 3 particles)
TOL_HEIGHT_MEAN = 0.02  # height map: mean |d| over the bed columns <= 2% of the bed height
TOL_HEIGHT_P95 = 0.15   # ... and 95% of the columns within 15% of the bed height (one particle layer)
TOL_CONTACTS = 0.03     # mean pp / body contacts per recorded interval: <= 3%
TOL_KE_MEAN = 0.10      # kinetic energy averaged over the run: <= 10%
TOL_KE = 0.25           # ... and per record |d| <= 25% of the run's peak (a chaotic flow)


@pytest.fixture(scope="module")
def runs():
    g = load("scoop_run")
    xs, vs = g["x_settled"], g["v_settled"]
    verts, faces = make_bucket_mesh(S.BUCKET_HALF, S.BUCKET_WALL)
    grid = bake_mesh_sdf(verts, faces, S.BUCKET_SPACING)
    path = S.dig_path(xs)
    bucket = gg.RigidBody(grid, DigDriver(**path), name="bucket")
    sc = gg.Scene(particles=gg.ParticleSet(xs.copy(), vs.copy()),
                  bodies=[gg.RigidBody(gg.HalfSpace(), name="floor"), bucket],
                  params=gg.MaterialParams(timestep=S.DT))
    lo, lift_z = g["lo"], float(g["lift_z"])
    nx, ny = g["height_map"].shape[1:]
    rec = {k: [] for k in ("ke", "n_pp", "n_body", "carried", "lifted", "height_map")}
    for _ in range(S.DIG_STEPS // S.RECORD_EVERY):
        _, reps = gg.run(sc, S.RECORD_EVERY)
        st = S.summary(sc.particles.positions, np.asarray(bucket.pose, float), lift_z, lo, nx, ny)
        rec["ke"].append(reps[-1].kinetic_energy)
        rec["n_pp"].append(np.mean([r.n_contacts for r in reps]))
        rec["n_body"].append(np.mean([r.n_body_contacts for r in reps]))
        rec["carried"].append(st["carried"])
        rec["lifted"].append(st["lifted"])
        rec["height_map"].append(st["height_map"])
    ours = {k: np.asarray(v) for k, v in rec.items()}
    return g, ours, grid


def _report(g, ours):
    print("\ncarried ref ", g["carried"].tolist())
    print("carried ours", ours["carried"].tolist())
    print("lifted ref  ", g["lifted"].tolist())
    print("lifted ours ", ours["lifted"].tolist())
    print("ke ref ", np.round(g["ke"], 1).tolist())
    print("ke ours", np.round(ours["ke"], 1).tolist())


def test_bucket_grid_baked_bit_exact(runs):
    g, _, grid = runs
    assert np.array_equal(np.asarray(grid.dims), g["grid_dims"])
    assert np.array_equal(np.asarray(grid.origin), g["grid_origin"])
    assert np.array_equal(np.asarray(grid.values), g["grid_values"])


def test_mass_transported_by_the_scoop(runs):
    g, ours, _ = runs
    _report(g, ours)
    ref, got = g["carried"].astype(float), ours["carried"].astype(float)
    assert ref[-1] >= 15, "the reference scoop must carry material"
    # every record: the bucket fills while it drives in, then holds its load
    print("carried ref ", ref.tolist(), "\ncarried ours", got.tolist())
    for r, o in zip(ref, got):
        assert abs(o - r) <= max(3.0, TOL_CARRIED * r), (r, o)


def test_pile_height_profile(runs):
    g, ours, _ = runs
    h_bed = float(np.quantile(g["x_settled"][:, 2], 0.99)) + S.R
    for hr, ho in zip(g["height_map"], ours["height_map"]):
        bed = (hr > 0) | (ho > 0)
        d = np.abs(hr - ho)[bed]
        assert d.mean() <= TOL_HEIGHT_MEAN * h_bed, (d.mean(), h_bed)
        p95 = float(np.quantile(d, 0.95))
        print(f"height |d|: mean {d.mean():.4f} p95 {p95:.4f} max {d.max():.4f} (bed {h_bed:.3f} m)")
        assert p95 <= TOL_HEIGHT_P95 * h_bed, (p95, h_bed)


def test_contacts_and_energy(runs):
    g, ours, _ = runs
    for k in ("n_pp", "n_body"):
        rel = np.abs(ours[k] - g[k]) / np.maximum(g[k], 1.0)
        print(k, "max rel diff", rel.max())
        assert rel.max() <= TOL_CONTACTS, (k, rel.max())
    peak = float(g["ke"].max())
    print("KE mean ref %.2f ours %.2f; max |d| %.2f (peak %.1f)" % (
        g["ke"].mean(), ours["ke"].mean(), np.abs(ours["ke"] - g["ke"]).max(), peak))
    assert abs(ours["ke"].mean() - g["ke"].mean()) <= TOL_KE_MEAN * g["ke"].mean()
    assert np.abs(ours["ke"] - g["ke"]).max() <= TOL_KE * peak
