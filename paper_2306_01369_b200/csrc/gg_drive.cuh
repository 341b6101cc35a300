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

// KinematicChain + ChainLinkDriver (kinematics.py:237-322) per env, the way
// ExcavationEnv advances it (envs.py:336-341): every step the joint rates
// are the command clipped to the velocity limits, q += dt * qd, then the
// forward kinematics of link `link`: its pose, and its spatial twist turned
// into the body twist (omega, v at the link origin).
constexpr int kChainMax = 16;
struct DriveChain {
  double* q;            // [E][J] joint positions, advanced on the device
  const double* cmd;    // [E][J] commanded joint rates
  int J, link;
  int parent[kChainMax];
  int prismatic[kChainMax];
  double origin[kChainMax][12];  // rows 0..2 of the fixed parent-to-joint 4x4
  double axis[kChainMax][3];
  double limit[kChainMax];
  double base[12];
  double dt;
  double lo[3], hi[3];
  gg_body tmpl;
};

__device__ __forceinline__ void mat34_mul(const double* A, const double* B, double* C) {
  // C = A @ B for 4x4 rigid transforms stored as their first 3 rows
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) C[4 * i + j] = A[4 * i] * B[j] + A[4 * i + 1] * B[4 + j] + A[4 * i + 2] * B[8 + j];
    C[4 * i + 3] = A[4 * i] * B[3] + A[4 * i + 1] * B[7] + A[4 * i + 2] * B[11] + A[4 * i + 3];
  }
}

__global__ void k_drive_chain(gg_body* __restrict__ rows, DriveChain C, int T, int E, int nb, int slot) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int J = C.J;
  double q[kChainMax], qd[kChainMax];
  for (int i = 0; i < J; ++i) {
    q[i] = C.q[static_cast<long long>(e) * J + i];
    const double c = C.cmd[static_cast<long long>(e) * J + i];
    qd[i] = c < -C.limit[i] ? -C.limit[i] : (c > C.limit[i] ? C.limit[i] : c);
  }
  double P[kChainMax][12], W[kChainMax][3], V[kChainMax][3];
  for (int k = 0; k < T; ++k) {
    for (int i = 0; i < J; ++i) q[i] = q[i] + C.dt * qd[i];
    for (int i = 0; i < J; ++i) {
      const double* par = C.parent[i] < 0 ? C.base : P[C.parent[i]];
      double joint[12];
      mat34_mul(par, C.origin[i], joint);
      const double* a = C.axis[i];
      double aw[3];
      for (int r = 0; r < 3; ++r) aw[r] = joint[4 * r] * a[0] + joint[4 * r + 1] * a[1] + joint[4 * r + 2] * a[2];
      double local[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
      double wj[3] = {0, 0, 0}, vj[3];
      if (!C.prismatic[i]) {
        // so3_exp(axis * q) (Rodrigues; first order below 1e-12 rad)
        const double w0 = a[0] * q[i], w1 = a[1] * q[i], w2 = a[2] * q[i];
        const double ang = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        if (ang < 1e-12) {
          local[1] = -w2; local[2] = w1; local[4] = w2; local[6] = -w0; local[8] = -w1; local[9] = w0;
        } else {
          const double k0 = w0 / ang, k1 = w1 / ang, k2 = w2 / ang;
          double sn, cs;
          sincos(ang, &sn, &cs);
          const double K[9] = {0, -k2, k1, k2, 0, -k0, -k1, k0, 0};
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
              double k2rc = 0.0;
              for (int m = 0; m < 3; ++m) k2rc += K[3 * r + m] * K[3 * m + c];
              local[4 * r + c] = (r == c ? 1.0 : 0.0) + sn * K[3 * r + c] + (1.0 - cs) * k2rc;
            }
        }
        for (int r = 0; r < 3; ++r) wj[r] = aw[r] * qd[i];
        const double* t = joint;  // t = column 3
        vj[0] = -(wj[1] * t[11] - wj[2] * t[7]);
        vj[1] = -(wj[2] * t[3] - wj[0] * t[11]);
        vj[2] = -(wj[0] * t[7] - wj[1] * t[3]);
      } else {
        local[3] = a[0] * q[i];
        local[7] = a[1] * q[i];
        local[11] = a[2] * q[i];
        for (int r = 0; r < 3; ++r) vj[r] = aw[r] * qd[i];
      }
      mat34_mul(joint, local, P[i]);
      for (int r = 0; r < 3; ++r) {
        W[i][r] = (C.parent[i] < 0 ? 0.0 : W[C.parent[i]][r]) + wj[r];
        V[i][r] = (C.parent[i] < 0 ? 0.0 : V[C.parent[i]][r]) + vj[r];
      }
    }
    const int L = C.link;
    gg_body r = C.tmpl;
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) r.rot[3 * i + j] = P[L][4 * i + j];
      r.trans[i] = P[L][4 * i + 3];
      r.omega[i] = W[L][i];
    }
    // body twist: v at the link origin = spatial v + omega x p
    r.v_origin[0] = V[L][0] + (W[L][1] * r.trans[2] - W[L][2] * r.trans[1]);
    r.v_origin[1] = V[L][1] + (W[L][2] * r.trans[0] - W[L][0] * r.trans[2]);
    r.v_origin[2] = V[L][2] + (W[L][0] * r.trans[1] - W[L][1] * r.trans[0]);
    if (r.bounded) {
      for (int a = 0; a < 3; ++a) {
        double mn = 1e300, mx = -1e300;
        for (int qq = 0; qq < 8; ++qq) {
          const double px = (qq & 4) ? C.hi[0] : C.lo[0];
          const double py = (qq & 2) ? C.hi[1] : C.lo[1];
          const double pz = (qq & 1) ? C.hi[2] : C.lo[2];
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
  for (int i = 0; i < J; ++i) C.q[static_cast<long long>(e) * J + i] = q[i];
}

}  // namespace gg
