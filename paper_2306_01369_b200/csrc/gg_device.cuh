// gg_device.cuh — device math shared by all kernels: cell rounding, spatial
// hash, signed-distance primitives and the sphere/body penetration test.
//
// Everything that decides WHETHER a contact exists is computed in float64
// with the reference's operation order (the library is built with
// --fmad=false so nvcc never contracts a*b+c behind our back; fused
// multiply-adds appear only where the reference's BLAS uses them, written as
// explicit fma()).  Inputs are float32 positions upcast to float64, which is
// exactly what the CPU oracle is fed, so decisions are bit-identical.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/granusim_b200.h"

namespace gg {

// ---------------------------------------------------------------------------
// Broadphase hash (broadphase.py:22-55)
// ---------------------------------------------------------------------------
constexpr long long kCellOffset = 100;            // broadphase.py:23
constexpr uint32_t kP0 = 73856093u;               // broadphase.py:22
constexpr uint32_t kP1 = 19349663u;
constexpr uint32_t kP2 = 83492791u;

struct HashCfg {
  long long n_h;   // table size
  uint32_t mask;   // n_h - 1 when n_h is a power of two
  int pow2;        // 1: floor-mod == low bits (exact for n_h <= 2^32)
};

// round_half_away(x / (2r)) -> int64 (broadphase.py:33-41).  Division is the
// IEEE-rounded quotient, as numpy computes it.
__device__ __forceinline__ long long cell_coord(double x, double two_r) {
  const double q = __ddiv_rn(x, two_r);
  const double a = floor(__dadd_rn(fabs(q), 0.5));
  return static_cast<long long>(copysign(a, q));
}

// Low 32 bits of (c - 100) * prime: enough for any power-of-two table since
// *, ^ and & commute with reduction mod 2^32.
__device__ __forceinline__ uint32_t hash_term32(long long c, uint32_t prime) {
  return static_cast<uint32_t>(c - kCellOffset) * prime;
}

// Full int64 rule with numpy's floor-mod (non-power-of-two n_h).
__device__ __forceinline__ long long hash_cell64_full(long long c0, long long c1, long long c2,
                                                     long long n_h) {
  const unsigned long long t0 = static_cast<unsigned long long>(c0 - kCellOffset) * 73856093ull;
  const unsigned long long t1 = static_cast<unsigned long long>(c1 - kCellOffset) * 19349663ull;
  const unsigned long long t2 = static_cast<unsigned long long>(c2 - kCellOffset) * 83492791ull;
  const long long h = static_cast<long long>(t0 ^ t1 ^ t2);
  long long m = h % n_h;
  if (m < 0) m += n_h;
  return m;
}

__device__ __forceinline__ uint32_t hash_cell64(long long c0, long long c1, long long c2,
                                                long long n_h) {
  return static_cast<uint32_t>(hash_cell64_full(c0, c1, c2, n_h));
}

__device__ __forceinline__ uint32_t hash_cell(long long c0, long long c1, long long c2,
                                              const HashCfg& H) {
  if (H.pow2)
    return (hash_term32(c0, kP0) ^ hash_term32(c1, kP1) ^ hash_term32(c2, kP2)) & H.mask;
  return hash_cell64(c0, c1, c2, H.n_h);
}

// ---------------------------------------------------------------------------
// small fp64 helpers with numpy's association order
// ---------------------------------------------------------------------------
struct d3 {
  double x, y, z;
};

// np.linalg.norm(axis=1) on 3-vectors sums (x^2 + y^2) + z^2.
__device__ __forceinline__ double norm3(double x, double y, double z) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// NaN-propagating max/min, like np.maximum / np.minimum.
__device__ __forceinline__ double nmax(double a, double b) {
  return (a != a) ? a : ((b != b) ? b : (a > b ? a : b));
}
__device__ __forceinline__ double nmin(double a, double b) {
  return (a != a) ? a : ((b != b) ? b : (a < b ? a : b));
}

// ---------------------------------------------------------------------------
// Gridded SDF (sdf.py:179-241)
// ---------------------------------------------------------------------------
struct DevGrid {
  double origin[3];
  double spacing[3];
  double upper[3];        // origin + (dims - 1) * spacing, host-computed
  int dims[3];
  int pad;
  long long offset;       // into the concatenated value store
};

__device__ __noinline__ double grid_distance(const DevGrid& G, const double* __restrict__ vals,
                                                double px, double py, double pz) {
  const double p[3] = {px, py, pz};
  double cl[3], u[3], f[3];
  long long i0[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    // np.clip(p, origin, upper)
    double c = p[a] < G.origin[a] ? G.origin[a] : p[a];
    c = c > G.upper[a] ? G.upper[a] : c;
    cl[a] = c;
    u[a] = __ddiv_rn(__dsub_rn(c, G.origin[a]), G.spacing[a]);
    long long fl = static_cast<long long>(floor(u[a]));
    const long long lim = G.dims[a] - 2;
    i0[a] = fl < lim ? fl : lim;
    f[a] = __dsub_rn(u[a], static_cast<double>(i0[a]));
  }
  const double outward = norm3(__dsub_rn(px, cl[0]), __dsub_rn(py, cl[1]), __dsub_rn(pz, cl[2]));
  const long long s1 = static_cast<long long>(G.dims[2]);
  const long long s0 = static_cast<long long>(G.dims[1]) * s1;
  const double* v = vals + G.offset;
  auto at = [&](long long ix, long long iy, long long iz) { return v[ix * s0 + iy * s1 + iz]; };
  const long long ix = i0[0], iy = i0[1], iz = i0[2];
  const double fx = f[0], fy = f[1], fz = f[2];
  const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy), gz = __dsub_rn(1.0, fz);
  auto lerp = [](double a, double wa, double b, double wb) {
    return __dadd_rn(__dmul_rn(a, wa), __dmul_rn(b, wb));
  };
  const double c00 = lerp(at(ix, iy, iz), gx, at(ix + 1, iy, iz), fx);
  const double c10 = lerp(at(ix, iy + 1, iz), gx, at(ix + 1, iy + 1, iz), fx);
  const double c01 = lerp(at(ix, iy, iz + 1), gx, at(ix + 1, iy, iz + 1), fx);
  const double c11 = lerp(at(ix, iy + 1, iz + 1), gx, at(ix + 1, iy + 1, iz + 1), fx);
  const double c0 = lerp(c00, gy, c10, fy);
  const double c1 = lerp(c01, gy, c11, fy);
  return __dadd_rn(lerp(c0, gz, c1, fz), outward);
}

// ---------------------------------------------------------------------------
// Primitive distance + gradient in the body frame (sdf.py:44-172)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sdf_distance(const gg_body& B, const DevGrid* __restrict__ grids,
                                               const double* __restrict__ gvals, double x,
                                               double y, double z) {
  switch (B.kind) {
    case GG_GEOM_SPHERE:
      return __dsub_rn(norm3(x, y, z), B.shape[0]);
    case GG_GEOM_HALFSPACE:
      // p @ normal - offset, dot as an FMA chain like the BLAS kernel
      return __dsub_rn(fma(z, B.shape[2], fma(y, B.shape[1], __dmul_rn(x, B.shape[0]))),
                       B.shape[3]);
    case GG_GEOM_BOX: {
      const double qx = __dsub_rn(fabs(x), B.shape[0]);
      const double qy = __dsub_rn(fabs(y), B.shape[1]);
      const double qz = __dsub_rn(fabs(z), B.shape[2]);
      const double outside = norm3(nmax(qx, 0.0), nmax(qy, 0.0), nmax(qz, 0.0));
      const double inside = nmin(nmax(nmax(qx, qy), qz), 0.0);
      return __dadd_rn(outside, inside);
    }
    case GG_GEOM_CYLINDER: {
      const double rho = hypot(x, y);
      const double dr = __dsub_rn(rho, B.shape[0]);
      const double dz = __dsub_rn(fabs(z), B.shape[1]);
      const double a = nmax(dr, 0.0), b = nmax(dz, 0.0);
      return __dadd_rn(nmin(nmax(dr, dz), 0.0),
                       sqrt(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b))));
    }
    case GG_GEOM_TUBE:
      return __dsub_rn(B.shape[0], hypot(x, y));
    case GG_GEOM_GRID:
      return grid_distance(grids[B.grid_id], gvals, x, y, z);
    default:
      return 1e300;
  }
}

__device__ __noinline__ d3 sdf_gradient(const gg_body& B, const DevGrid* __restrict__ grids,
                                           const double* __restrict__ gvals, double x, double y,
                                           double z) {
  d3 g{0.0, 0.0, 0.0};
  switch (B.kind) {
    case GG_GEOM_SPHERE: {
      const double n = norm3(x, y, z);
      if (n > 0.0) g = {__ddiv_rn(x, n), __ddiv_rn(y, n), __ddiv_rn(z, n)};
      break;
    }
    case GG_GEOM_HALFSPACE:
      g = {B.shape[0], B.shape[1], B.shape[2]};
      break;
    case GG_GEOM_BOX: {
      const double q[3] = {__dsub_rn(fabs(x), B.shape[0]), __dsub_rn(fabs(y), B.shape[1]),
                           __dsub_rn(fabs(z), B.shape[2])};
      const double p[3] = {x, y, z};
      const double qp[3] = {nmax(q[0], 0.0), nmax(q[1], 0.0), nmax(q[2], 0.0)};
      const double n = norm3(qp[0], qp[1], qp[2]);
      double s[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) s[a] = p[a] >= 0.0 ? 1.0 : -1.0;
      if (n > 0.0) {
        g = {__dmul_rn(__ddiv_rn(qp[0], n), s[0]), __dmul_rn(__ddiv_rn(qp[1], n), s[1]),
             __dmul_rn(__ddiv_rn(qp[2], n), s[2])};
      } else {
        // least-penetrated axis, first on ties (np.argmax)
        int ax = 0;
        if (q[1] > q[ax]) ax = 1;
        if (q[2] > q[ax]) ax = 2;
        double gg3[3] = {0.0, 0.0, 0.0};
        gg3[ax] = s[ax];
        g = {gg3[0], gg3[1], gg3[2]};
      }
      break;
    }
    case GG_GEOM_CYLINDER: {
      const double rho = hypot(x, y);
      const double sr = rho > 1e-300 ? rho : 1e-300;
      const double rx = __ddiv_rn(x, sr), ry = __ddiv_rn(y, sr);
      const double az = z >= 0.0 ? 1.0 : -1.0;
      const double dr = __dsub_rn(rho, B.shape[0]);
      const double dz = __dsub_rn(fabs(z), B.shape[1]);
      const double mr = nmax(dr, 0.0), mz = nmax(dz, 0.0);
      // radial * max(dr,0) + axial * max(dz,0)
      const double ox = __dadd_rn(__dmul_rn(rx, mr), 0.0 * mz);
      const double oy = __dadd_rn(__dmul_rn(ry, mr), 0.0 * mz);
      const double oz = __dadd_rn(0.0 * mr, __dmul_rn(az, mz));
      const double n = norm3(ox, oy, oz);
      if (n > 0.0) {
        g = {__ddiv_rn(ox, n), __ddiv_rn(oy, n), __ddiv_rn(oz, n)};
      } else if (dr > dz) {
        g = {rx, ry, 0.0};
      } else {
        g = {0.0, 0.0, az};
      }
      break;
    }
    case GG_GEOM_TUBE: {
      double rho = hypot(x, y);
      rho = rho > 1e-300 ? rho : 1e-300;
      g = {-__ddiv_rn(x, rho), -__ddiv_rn(y, rho), 0.0};
      break;
    }
    case GG_GEOM_GRID: {
      // central differences, h = min(spacing) / 2 (sdf.py:230-238)
      const DevGrid& G = grids[B.grid_id];
      double h = G.spacing[0];
      h = G.spacing[1] < h ? G.spacing[1] : h;
      h = G.spacing[2] < h ? G.spacing[2] : h;
      h = h / 2.0;
      const double two_h = 2.0 * h;
      g.x = __ddiv_rn(__dsub_rn(grid_distance(G, gvals, __dadd_rn(x, h), y, z),
                                grid_distance(G, gvals, __dsub_rn(x, h), y, z)),
                      two_h);
      g.y = __ddiv_rn(__dsub_rn(grid_distance(G, gvals, x, __dadd_rn(y, h), z),
                                grid_distance(G, gvals, x, __dsub_rn(y, h), z)),
                      two_h);
      g.z = __ddiv_rn(__dsub_rn(grid_distance(G, gvals, x, y, __dadd_rn(z, h)),
                                grid_distance(G, gvals, x, y, __dsub_rn(z, h))),
                      two_h);
      break;
    }
    default:
      break;
  }
  return g;
}

// ---------------------------------------------------------------------------
// Sphere-vs-posed-body penetration (sdf.py:472-512).
// Returns 1 for a contact (psi, world normal filled), 0 otherwise; *degenerate
// is set when d < r but the gradient norm is <= 1e-9 (counted, not a contact).
// ---------------------------------------------------------------------------
constexpr double kDegenerateGradEps = 1e-9;  // sdf.py:19

__device__ __forceinline__ int penetrate(const gg_body& B, const DevGrid* __restrict__ grids,
                                         const double* __restrict__ gvals, double px, double py,
                                         double pz, double r, double* psi, d3* nrm,
                                         int* degenerate) {
  *degenerate = 0;
  // local = (p - t) @ R; row vector times R -> fma chain over R's rows
  const double dx = __dsub_rn(px, B.trans[0]);
  const double dy = __dsub_rn(py, B.trans[1]);
  const double dz = __dsub_rn(pz, B.trans[2]);
  const double* R = B.rot;
  const double lx = fma(dz, R[6], fma(dy, R[3], __dmul_rn(dx, R[0])));
  const double ly = fma(dz, R[7], fma(dy, R[4], __dmul_rn(dx, R[1])));
  const double lz = fma(dz, R[8], fma(dy, R[5], __dmul_rn(dx, R[2])));
  const double d = sdf_distance(B, grids, gvals, lx, ly, lz);
  if (!(d < r)) return 0;
  const d3 g = sdf_gradient(B, grids, gvals, lx, ly, lz);
  const double gn = norm3(g.x, g.y, g.z);
  if (!(gn > kDegenerateGradEps)) {
    *degenerate = 1;
    return 0;
  }
  const double ux = __ddiv_rn(g.x, gn), uy = __ddiv_rn(g.y, gn), uz = __ddiv_rn(g.z, gn);
  // (g / |g|) @ R^T
  nrm->x = fma(uz, R[2], fma(uy, R[1], __dmul_rn(ux, R[0])));
  nrm->y = fma(uz, R[5], fma(uy, R[4], __dmul_rn(ux, R[3])));
  nrm->z = fma(uz, R[8], fma(uy, R[7], __dmul_rn(ux, R[6])));
  *psi = __dsub_rn(r, d);
  return 1;
}

// RigidBody.velocity_at (scene.py:163-166) at the contact point
// cp = p - n * (r - psi) (contact.py:279).
__device__ __forceinline__ d3 body_surface_velocity(const gg_body& B, double px, double py,
                                                    double pz, const d3& n, double r,
                                                    double psi) {
  const double s = __dsub_rn(r, psi);
  const double cx = __dsub_rn(__dsub_rn(px, __dmul_rn(n.x, s)), B.trans[0]);
  const double cy = __dsub_rn(__dsub_rn(py, __dmul_rn(n.y, s)), B.trans[1]);
  const double cz = __dsub_rn(__dsub_rn(pz, __dmul_rn(n.z, s)), B.trans[2]);
  const double* w = B.omega;
  d3 v;
  v.x = __dadd_rn(B.v_origin[0], __dsub_rn(__dmul_rn(w[1], cz), __dmul_rn(w[2], cy)));
  v.y = __dadd_rn(B.v_origin[1], __dsub_rn(__dmul_rn(w[2], cx), __dmul_rn(w[0], cz)));
  v.z = __dadd_rn(B.v_origin[2], __dsub_rn(__dmul_rn(w[0], cy), __dmul_rn(w[1], cx)));
  return v;
}

}  // namespace gg
