"""Bulk statistics of a free-running scoop run (BASELINE.json north_star
criterion 3: "pile height profile, mass transported by the scoop").

Long contact rollouts are chaotic, so a device run is compared with the
reference through these statistics, not particle by particle.  Shared by the
fixture generator (tests/golden/make_golden_scoop.py, which runs the real
reference) and the GPU test (tests/test_scoop_parity.py); pure numpy.

The scoop is an open-top bucket (meshes.make_bucket_mesh) on a DigDriver
(beds.py).  Definitions:
  * carried   particles whose centre lies in the bucket's cavity, in the
              bucket frame: |x| < ix, |y| < iy, floor_z < z < hz + r (up to
              one radius above the rim) — the mass the scoop holds;
  * lifted    particles whose centre is more than `lift_z` above the floor
              (above the undisturbed bed surface): material raised out of
              the bed;
  * height map  the highest particle top (z + r) per 0.2 m x 0.2 m column
              over the bed's footprint (0 for an empty column);
  * KE, pp contacts, body contacts per recorded step.
"""

from __future__ import annotations

import numpy as np

# scene constants (make_golden_scoop.py and the test build the same scene)
R = 0.05
N = 4000                        # particles (the first N seeded sites)
BUCKET_HALF = (0.35, 0.25, 0.2)
BUCKET_WALL = 0.05
BUCKET_SPACING = 0.025          # SDF grid spacing of the baked bucket
DT = 5e-4
SETTLE_DT = 1e-3
SETTLE_STEPS = 800
DIG_STEPS = 4000                # 2.0 s of digging and lifting at DT
RECORD_EVERY = 200
COLUMN = 0.2
MAP_COLUMNS = 24               # height map: 24 x 24 columns from the bed's corner - 0.5 m


# the bed: seed_particles_grid (scene.py:226-262, jitter 0.3 as ExcavationEnv.reset
# uses, envs.py:270-276) in this box, first N sites, settled by the reference
BED_LO = (0.0, 0.0, 0.05)
BED_HI = (3.64, 3.64, 1.1)
BED_JITTER = 0.3
BED_SEED = 0


def dig_path(x_settled: np.ndarray) -> dict:
    """DigDriver arguments for a front-loader pass along +x: the bucket's
    mouth faces the travel direction (pitch pi/2: its local +z is world +x),
    its centre 0.3 m below the bed surface and its lip 5 cm before the bed's
    -x edge; it drives 0.9 m into the bed in 1.5 s while curling the mouth up
    to 0.3 rad, then lifts at 0.5 m/s."""
    top = float(np.quantile(x_settled[:, 2], 0.99)) + R
    x0 = float(np.quantile(x_settled[:, 0], 0.001)) - R - 0.05 - BUCKET_HALF[2]
    yc = float(np.median(x_settled[:, 1]))
    return dict(start=np.array([x0, yc, top - 0.3]), direction=np.array([1.0, 0.0, 0.0]),
                length=0.9, depth=0.0, duration=1.5, pitch0=0.5 * np.pi, pitch1=0.3, t0=0.0,
                lift_speed=0.5)


def carried(x: np.ndarray, pose: np.ndarray) -> int:
    hx, hy, hz = BUCKET_HALF
    w = BUCKET_WALL
    local = (x - pose[:3, 3]) @ pose[:3, :3]
    inside = ((np.abs(local[:, 0]) < hx - w) & (np.abs(local[:, 1]) < hy - w)
              & (local[:, 2] > -hz + w) & (local[:, 2] < hz + R))
    return int(inside.sum())


def height_map(x: np.ndarray, lo: np.ndarray, nx: int, ny: int) -> np.ndarray:
    ix = np.floor((x[:, 0] - lo[0]) / COLUMN).astype(np.int64)
    iy = np.floor((x[:, 1] - lo[1]) / COLUMN).astype(np.int64)
    ok = (ix >= 0) & (ix < nx) & (iy >= 0) & (iy < ny)
    hm = np.zeros((nx, ny))
    np.maximum.at(hm, (ix[ok], iy[ok]), x[ok, 2] + R)
    return hm


def summary(x: np.ndarray, pose: np.ndarray, lift_z: float, lo: np.ndarray, nx: int, ny: int) -> dict:
    return {"carried": carried(x, pose), "lifted": int((x[:, 2] > lift_z).sum()),
            "height_map": height_map(x, lo, nx, ny)}
