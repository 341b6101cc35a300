// gg_bake.cuh — exact signed distance to a watertight triangle mesh on the
// device: the knots of a baked SdfGrid (bake_mesh_sdf, sdf.py:393-419) or an
// arbitrary point list (MeshDistance.signed_distance, sdf.py:357-391).
//
// One thread per point scans every triangle (tiles of triangle corners staged
// in shared memory, read as warp-uniform broadcasts), keeps the nearest one
// (strict <: the first triangle wins ties, like numpy argmin) and signs the
// distance with the pseudonormal of the nearest feature.  Arithmetic follows
// the reference's numpy expressions operation for operation (einsum dot
// products sum (x + z) + y on the reference host, see tests/golden), with
// --fmad=false and IEEE division / square root, so the baked values are the
// reference's bit for bit.
#pragma once

namespace gg {

constexpr int kBakeTile = 128;  // triangles per shared-memory tile
constexpr int kTriDoubles = 30;

__device__ __forceinline__ double edot(double ax, double ay, double az, double bx, double by,
                                       double bz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(az, bz)), __dmul_rn(ay, by));
}

// np.clip(x, 0, 1) then np.nan_to_num
__device__ __forceinline__ double clip01(double x) {
  if (x != x) return 0.0;
  return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
}
// np.nan_to_num: NaN -> 0, +-inf -> +-DBL_MAX
__device__ __forceinline__ double nan_to_num(double x) {
  if (x != x) return 0.0;
  if (isinf(x)) return x > 0 ? 1.7976931348623157e308 : -1.7976931348623157e308;
  return x;
}

struct BakeArgs {
  const double* tri;  // [T][30]
  long long T;
  const double* pts;  // [n][3] or null: grid knots
  double origin[3], spacing[3];
  long long dims[3];
  long long n;
  double* out;
};

// closest point on triangle (a, b, c) to p: barycentrics, region rules of
// _closest_on_triangles (sdf.py:299-355), later regions winning
__device__ __forceinline__ void closest_bary(const double* a, const double* b, const double* c,
                                             double px, double py, double pz, double w[3]) {
  const double abx = b[0] - a[0], aby = b[1] - a[1], abz = b[2] - a[2];
  const double acx = c[0] - a[0], acy = c[1] - a[1], acz = c[2] - a[2];
  const double apx = px - a[0], apy = py - a[1], apz = pz - a[2];
  const double d1 = edot(abx, aby, abz, apx, apy, apz);
  const double d2 = edot(acx, acy, acz, apx, apy, apz);
  const double bpx = px - b[0], bpy = py - b[1], bpz = pz - b[2];
  const double d3 = edot(abx, aby, abz, bpx, bpy, bpz);
  const double d4 = edot(acx, acy, acz, bpx, bpy, bpz);
  const double cpx = px - c[0], cpy = py - c[1], cpz = pz - c[2];
  const double d5 = edot(abx, aby, abz, cpx, cpy, cpz);
  const double d6 = edot(acx, acy, acz, cpx, cpy, cpz);
  const double vc = __dsub_rn(__dmul_rn(d1, d4), __dmul_rn(d3, d2));
  const double vb = __dsub_rn(__dmul_rn(d5, d2), __dmul_rn(d1, d6));
  const double va = __dsub_rn(__dmul_rn(d3, d6), __dmul_rn(d5, d4));
  if (d1 <= 0.0 && d2 <= 0.0) {  // vertex a
    w[0] = 1.0; w[1] = 0.0; w[2] = 0.0;
  } else if (d3 >= 0.0 && d4 <= d3) {  // vertex b
    w[0] = 0.0; w[1] = 1.0; w[2] = 0.0;
  } else if (d6 >= 0.0 && d5 <= d6) {  // vertex c
    w[0] = 0.0; w[1] = 0.0; w[2] = 1.0;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {  // edge ab
    const double v = clip01(d1 / (d1 - d3));
    w[0] = 1.0 - v; w[1] = v; w[2] = 0.0;
  } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {  // edge ac
    const double v = clip01(d2 / (d2 - d6));
    w[0] = 1.0 - v; w[1] = 0.0; w[2] = v;
  } else if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {  // edge bc
    const double v = clip01((d4 - d3) / ((d4 - d3) + (d5 - d6)));
    w[0] = 0.0; w[1] = 1.0 - v; w[2] = v;
  } else {  // face interior
    const double den = (va + vb) + vc;
    const double v = nan_to_num(vb / den), u = nan_to_num(vc / den);
    w[0] = (1.0 - v) - u; w[1] = v; w[2] = u;
  }
}

__global__ void __launch_bounds__(256) k_bake_sdf(BakeArgs A) {
  __shared__ double st[kBakeTile][9];
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = i < A.n;
  double px = 0.0, py = 0.0, pz = 0.0;
  if (live) {
    if (A.pts) {
      px = A.pts[3 * i]; py = A.pts[3 * i + 1]; pz = A.pts[3 * i + 2];
    } else {  // knot (ix, iy, iz), C order over (x, y, z): knot_points (sdf.py:206-209)
      const long long iz = i % A.dims[2], iy = (i / A.dims[2]) % A.dims[1], ix = i / (A.dims[2] * A.dims[1]);
      px = A.origin[0] + A.spacing[0] * static_cast<double>(ix);
      py = A.origin[1] + A.spacing[1] * static_cast<double>(iy);
      pz = A.origin[2] + A.spacing[2] * static_cast<double>(iz);
    }
  }
  double best = __longlong_as_double(0x7ff0000000000000ll);
  long long bt = 0;
  double bw[3] = {1.0, 0.0, 0.0};
  double bc[3] = {0.0, 0.0, 0.0};
  for (long long t0 = 0; t0 < A.T; t0 += kBakeTile) {
    const int nt = static_cast<int>(A.T - t0 < kBakeTile ? A.T - t0 : kBakeTile);
    __syncthreads();
    for (int q = threadIdx.x; q < nt * 9; q += blockDim.x)
      st[q / 9][q % 9] = A.tri[(t0 + q / 9) * kTriDoubles + q % 9];
    __syncthreads();
    if (!live) continue;
    for (int t = 0; t < nt; ++t) {
      const double* a = st[t];
      double w[3];
      closest_bary(a, a + 3, a + 6, px, py, pz, w);
      // cp = w0 a + w1 b + w2 c, left to right
      const double cx = __dadd_rn(__dadd_rn(__dmul_rn(w[0], a[0]), __dmul_rn(w[1], a[3])), __dmul_rn(w[2], a[6]));
      const double cy = __dadd_rn(__dadd_rn(__dmul_rn(w[0], a[1]), __dmul_rn(w[1], a[4])), __dmul_rn(w[2], a[7]));
      const double cz = __dadd_rn(__dadd_rn(__dmul_rn(w[0], a[2]), __dmul_rn(w[1], a[5])), __dmul_rn(w[2], a[8]));
      const double dx = px - cx, dy = py - cy, dz = pz - cz;
      const double d2 = edot(dx, dy, dz, dx, dy, dz);
      if (d2 < best || t0 + t == 0) {  // first minimum (numpy argmin)
        best = d2;
        bt = t0 + t;
        bw[0] = w[0]; bw[1] = w[1]; bw[2] = w[2];
        bc[0] = cx; bc[1] = cy; bc[2] = cz;
      }
    }
  }
  if (!live) return;
  // pseudonormal of the nearest feature: face, edge (one barycentric ~0;
  // edges v0v1, v1v2, v2v0) or corner (two ~0)
  const double eps = 1e-9;
  const bool z0 = bw[0] < eps, z1 = bw[1] < eps, z2 = bw[2] < eps;
  const int nz = int(z0) + int(z1) + int(z2);
  const double* row = A.tri + bt * kTriDoubles;
  const double* pn = row + 9;
  if (nz == 1) {
    // the reference maps the zero corner k to edge [2, 0, 1][k] (sdf.py:378-382)
    const int zc = z0 ? 0 : (z1 ? 1 : 2);
    pn = row + 12 + 3 * (zc == 0 ? 2 : zc - 1);
  } else if (nz == 2) {
    const int vc = !z0 ? 0 : (!z1 ? 1 : 2);
    pn = row + 21 + 3 * vc;
  }
  const double dx = px - bc[0], dy = py - bc[1], dz = pz - bc[2];
  const double dist = sqrt(best);
  const double s = edot(dx, dy, dz, pn[0], pn[1], pn[2]) >= 0.0 ? 1.0 : -1.0;
  A.out[i] = s * dist;
}

}  // namespace gg
