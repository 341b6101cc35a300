// gg_drive.cuh — device-resident body drivers for batched environments
// (SURVEY.md §8f rank 1): the per-step body rows of E envs are generated on
// the device instead of packed on the host and uploaded (4096 envs x 2
// bodies x 10 substeps = 20 MB of gg_body rows per control step).
//
//   fixed   the same row every step (the ground, a static tool)
//   track   TrackSteeringDriver (kinematics.py:179-230) with per-env state
//           (x, y, theta) and a per-env action: every step first advances the
//           state (track_steering_advance: heading before position), then
//           poses the body (Rz(theta) at (x, y, z), times the base pose) with
//           the twist of TrackSteeringDriver.twist_at, and the world AABB of
//           the body's local contact bounds (`_near_body`, contact.py:187-203).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gg_kernels.cuh"

namespace gg {

struct DriveTrack {
  double* x;            // [E] state, advanced on the device
  double* y;
  double* theta;
  const double* action; // [E][2], clipped to [-1, 1] by the host
  double z, scale_v, scale_omega, dt;
  double base[16];      // base pose, row-major 4x4
  double lo[3], hi[3];  // local contact bounds (bounded rows)
  gg_body tmpl;         // kind, grid, shape, bounded
};

// rows[k][e][slot] for k < T: the template row in every step
__global__ void k_drive_fixed(gg_body* __restrict__ rows, const gg_body* __restrict__ fixed, int T,
                              int E, int nb, int slot) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const gg_body b = fixed[e];
  for (int k = 0; k < T; ++k) rows[(static_cast<long long>(k) * E + e) * nb + slot] = b;
}

__global__ void k_drive_track(gg_body* __restrict__ rows, DriveTrack P, int T, int E, int nb, int slot) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double x = P.x[e], y = P.y[e], th = P.theta[e];
  const double a0 = P.action[2 * e], a1 = P.action[2 * e + 1];
  const double* B = P.base;
  for (int k = 0; k < T; ++k) {
    // track_steering_advance: theta + dt*so*a1, then x/y with the new heading
    th = th + P.dt * P.scale_omega * a1;
    double s, c;
    sincos(th, &s, &c);
    x = x + P.dt * P.scale_v * a0 * c;
    y = y + P.dt * P.scale_v * a0 * s;
    // pose = [Rz(theta) | (x, y, z)] @ base
    const double Rz[9] = {c, -s, 0.0, s, c, 0.0, 0.0, 0.0, 1.0};
    const double tz[3] = {x, y, P.z};
    gg_body r = P.tmpl;
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j)
        r.rot[3 * i + j] = Rz[3 * i] * B[j] + Rz[3 * i + 1] * B[4 + j] + Rz[3 * i + 2] * B[8 + j];
      r.trans[i] = Rz[3 * i] * B[3] + Rz[3 * i + 1] * B[7] + Rz[3 * i + 2] * B[11] + tz[i];
    }
    // twist_at: omega = (0, 0, so*a1); v = so-rotation of the offset + vehicle velocity
    const double w = P.scale_omega * a1;
    const double vv = P.scale_v * a0;
    const double ox = r.trans[0] - x, oy = r.trans[1] - y;
    r.omega[0] = 0.0;
    r.omega[1] = 0.0;
    r.omega[2] = w;
    r.v_origin[0] = vv * c - w * oy;  // v_vehicle + omega x (pos - ref)
    r.v_origin[1] = vv * s + w * ox;
    r.v_origin[2] = 0.0;
    if (r.bounded) {  // world AABB of the 8 local corners (corners @ R^T + t)
      for (int a = 0; a < 3; ++a) {
        double mn = 1e300, mx = -1e300;
        for (int q = 0; q < 8; ++q) {
          const double px = (q & 4) ? P.hi[0] : P.lo[0];
          const double py = (q & 2) ? P.hi[1] : P.lo[1];
          const double pz = (q & 1) ? P.hi[2] : P.lo[2];
          const double wv = px * r.rot[3 * a] + py * r.rot[3 * a + 1] + pz * r.rot[3 * a + 2] + r.trans[a];
          mn = wv < mn ? wv : mn;
          mx = wv > mx ? wv : mx;
        }
        r.aabb_lo[a] = mn;
        r.aabb_hi[a] = mx;
      }
    }
    rows[(static_cast<long long>(k) * E + e) * nb + slot] = r;
  }
  P.x[e] = x;
  P.y[e] = y;
  P.theta[e] = th;
}

}  // namespace gg
