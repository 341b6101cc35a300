// gg_render.cuh — depth rendering of the particle bed and the bodies
// (render.py: DepthCamera.rays :35-58, ray_spheres_depth :61-82,
// sphere_trace_depth :85-116, render_depth :119-135), SURVEY.md §8(f) row 2:
// the observation step right after physics in env.step (envs.py:180-205).
//
// One block renders 256 pixels of one camera of one env.  The env's particles
// are streamed through shared memory in tiles (float4, the resident state —
// no host copy of the bed); each thread tests its ray against every particle
// of the tile with a float32 pre-filter (the discriminant, conservative
// margin) and the exact float64 near-root for the survivors, then sphere-
// traces the env's bodies (float64 SDFs, the same device functions the
// contact kernel uses).  Depth = min over particles and bodies, capped at far.
#pragma once

#include "gg_kernels.cuh"

namespace gg {

constexpr int kRenderTile = 1024;
constexpr double kTraceEps = 1e-4;  // sphere_trace_depth eps (render.py:89)
constexpr int kTraceSteps = 128;    // sphere_trace_depth max_steps (render.py:90)

struct RenderArgs {
  const gg_camera* cams;   // [E][n_cams] if per_env else [n_cams]
  int n_cams, per_env;
  const gg_body* bodies;   // [E][nb]
  int nb;
  const long long* pix_off;  // [n_cams + 1] pixel offsets of each camera in an env's output
  float* out;              // [E][pix_off[n_cams]]
};

// DepthCamera.rays for pixel p (row-major): origin and unit direction, float64
__device__ __forceinline__ void camera_ray(const gg_camera& C, int p, double o[3], double d[3]) {
  const int W = C.width, H = C.height;
  const int ix = p % W, iy = p / W;
  const double gx = (static_cast<double>(ix) + 0.5) / W - 0.5;
  const double gy = (static_cast<double>(iy) + 0.5) / H - 0.5;
  const double* T = C.pose;  // row-major 4x4
  if (C.kind == 0) {
    const double tan_half = tan(C.fov / 2.0);
    const double aspect = static_cast<double>(W) / static_cast<double>(H);
    double l[3] = {gx * 2.0 * tan_half * aspect, gy * 2.0 * tan_half, 1.0};
    const double nrm = norm3(l[0], l[1], l[2]);
    l[0] /= nrm;
    l[1] /= nrm;
    l[2] /= nrm;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      o[i] = T[4 * i + 3];
      d[i] = fma(l[2], T[4 * i + 2], fma(l[1], T[4 * i + 1], l[0] * T[4 * i + 0]));  // d @ R^T
    }
  } else {
    const double l[3] = {gx * C.extent[0], gy * C.extent[1], 0.0};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      o[i] = fma(l[2], T[4 * i + 2], fma(l[1], T[4 * i + 1], l[0] * T[4 * i + 0])) + T[4 * i + 3];
      d[i] = T[4 * i + 2];  // R[:, 2]
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_render(Dev D, RenderArgs A) {
  __shared__ float4 tile[kRenderTile];
  const int env = blockIdx.z, cam = blockIdx.y;
  const gg_camera& C = A.cams[A.per_env ? env * A.n_cams + cam : cam];
  const int npix = C.width * C.height;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (static_cast<int>(blockIdx.x * blockDim.x) >= npix) return;  // block-uniform
  const bool live = p < npix;
  double o[3] = {0.0, 0.0, 0.0}, d[3] = {0.0, 0.0, 1.0};
  if (live) camera_ray(C, p, o, d);
  const double far = C.far;
  double best = far;
  // ---- particles of this env (ray_spheres_depth) ----------------------------
  const float4* X = D.X[D.ctl->cur] + static_cast<long long>(env) * D.ne;
  const double r2 = D.r * D.r;
  const float of[3] = {static_cast<float>(o[0]), static_cast<float>(o[1]), static_cast<float>(o[2])};
  const float df[3] = {static_cast<float>(d[0]), static_cast<float>(d[1]), static_cast<float>(d[2])};
  const float r2f = static_cast<float>(r2);
  for (int t0 = 0; t0 < D.ne; t0 += kRenderTile) {
    const int m = min(kRenderTile, D.ne - t0);
    __syncthreads();
    for (int q = threadIdx.x; q < m; q += blockDim.x) tile[q] = X[t0 + q];
    __syncthreads();
    if (!live) continue;
    for (int q = 0; q < m; ++q) {
      const float4 c = tile[q];
      const float ox = of[0] - c.x, oy = of[1] - c.y, oz = of[2] - c.z;
      const float bf = ox * df[0] + oy * df[1] + oz * df[2];
      const float cc = ox * ox + oy * oy + oz * oz;
      // float32 discriminant, conservative: its error is far below this margin
      if (bf * bf - (cc - r2f) < -1e-4f * (cc + bf * bf) - 1e-6f) continue;
      if (bf > 0.f && cc > r2f) continue;  // sphere behind the origin: near root < 0
      const double ocx = o[0] - static_cast<double>(c.x);
      const double ocy = o[1] - static_cast<double>(c.y);
      const double ocz = o[2] - static_cast<double>(c.z);
      const double b = ocx * d[0] + ocy * d[1] + ocz * d[2];
      const double cterm = (ocx * ocx + ocy * ocy + ocz * ocz) - r2;
      const double disc = b * b - cterm;
      if (!(disc >= 0.0)) continue;
      const double t = -b - sqrt(disc);
      if (t > 0.0 && t < best) best = t;
    }
  }
  if (!live) return;
  // ---- bodies (sphere_trace_depth) -------------------------------------------
  const gg_body* bodies = A.bodies + static_cast<long long>(env) * A.nb;
  for (int bi = 0; bi < A.nb; ++bi) {
    const gg_body& B = bodies[bi];
    const double* R = B.rot;
    const double ex = o[0] - B.trans[0], ey = o[1] - B.trans[1], ez = o[2] - B.trans[2];
    // (o - t) @ R and d @ R
    const double lo0 = fma(ez, R[6], fma(ey, R[3], ex * R[0]));
    const double lo1 = fma(ez, R[7], fma(ey, R[4], ex * R[1]));
    const double lo2 = fma(ez, R[8], fma(ey, R[5], ex * R[2]));
    const double ld0 = fma(d[2], R[6], fma(d[1], R[3], d[0] * R[0]));
    const double ld1 = fma(d[2], R[7], fma(d[1], R[4], d[0] * R[1]));
    const double ld2 = fma(d[2], R[8], fma(d[1], R[5], d[0] * R[2]));
    double t = 0.0;
    for (int it = 0; it < kTraceSteps; ++it) {
      const double f = sdf_distance(B, D.grids, D.gvals, lo0 + t * ld0, lo1 + t * ld1, lo2 + t * ld2);
      if (f < kTraceEps) {  // arrived: a hit at t
        best = t < best ? t : best;
        break;
      }
      t += (f > kTraceEps ? f : kTraceEps) * 0.9;
      if (!(t < far)) break;
    }
  }
  A.out[static_cast<long long>(env) * A.pix_off[A.n_cams] + A.pix_off[cam] + p] =
      static_cast<float>(best < far ? best : far);
}

}  // namespace gg
