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
  const double* local;     // [pix_off[n_cams]][3] camera-frame ray of every pixel (k_render_local)
};

// DepthCamera.rays (render.py:35-58), split in two: the camera-frame part of
// pixel p depends only on the intrinsics (perspective: the unit direction;
// orthographic: the ray origin on the image plane), computed once per camera
// index; the pose is applied per env.  float64.
__device__ __forceinline__ void camera_local(const gg_camera& C, int p, double l[3]) {
  const int W = C.width, H = C.height;
  const int ix = p % W, iy = p / W;
  const double gx = (static_cast<double>(ix) + 0.5) / W - 0.5;
  const double gy = (static_cast<double>(iy) + 0.5) / H - 0.5;
  if (C.kind == 0) {
    const double tan_half = tan(C.fov / 2.0);
    const double aspect = static_cast<double>(W) / static_cast<double>(H);
    l[0] = gx * 2.0 * tan_half * aspect;
    l[1] = gy * 2.0 * tan_half;
    l[2] = 1.0;
    const double nrm = norm3(l[0], l[1], l[2]);
    l[0] /= nrm;
    l[1] /= nrm;
    l[2] /= nrm;
  } else {
    l[0] = gx * C.extent[0];
    l[1] = gy * C.extent[1];
    l[2] = 0.0;
  }
}

__global__ void k_render_local(const gg_camera* __restrict__ cams, int n_cams,
                               const long long* __restrict__ pix_off, double* __restrict__ local) {
  const int cam = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const gg_camera& C = cams[cam];
  if (cam >= n_cams || p >= C.width * C.height) return;
  camera_local(C, p, local + 3 * (pix_off[cam] + p));
}

// world ray of a pixel from its camera-frame part and the camera pose
__device__ __forceinline__ void camera_ray(const gg_camera& C, const double* l, double o[3],
                                           double d[3]) {
  const double* T = C.pose;  // row-major 4x4
  if (C.kind == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      o[i] = T[4 * i + 3];
      d[i] = fma(l[2], T[4 * i + 2], fma(l[1], T[4 * i + 1], l[0] * T[4 * i + 0]));  // d @ R^T
    }
  } else {
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
  if (live) camera_ray(C, A.local + 3 * (A.pix_off[cam] + p), o, d);
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

// ---------------------------------------------------------------------------
// Splatting (the default): instead of every pixel testing every particle,
// every particle tests only the pixels whose rays can reach it — a
// conservative pixel box from the sphere's angular extent (perspective) or
// its footprint (orthographic), one pixel of margin — with the SAME exact
// float64 ray and near root, and keeps the minimum with a 64-bit atomicMin on
// the depth's bit pattern (positive doubles order like their bits).  The
// image is bitwise that of k_render; the bodies are traced afterwards.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void splat_box(const gg_camera& C, double cx, double cy, double cz,
                                          double r, int* x0, int* x1, int* y0, int* y1) {
  const double* T = C.pose;
  const double ex = cx - T[3], ey = cy - T[7], ez = cz - T[11];
  // camera-frame centre: R^T (c - t), R's columns are the camera axes
  const double px = T[0] * ex + T[4] * ey + T[8] * ez;
  const double py = T[1] * ex + T[5] * ey + T[9] * ez;
  const double pz = T[2] * ex + T[6] * ey + T[10] * ez;
  const int W = C.width, H = C.height;
  *x0 = 0; *x1 = W - 1; *y0 = 0; *y1 = H - 1;
  if (C.kind == 0) {
    if (px * px + py * py + pz * pz <= r * r * (1.0 + 1e-9)) {  // camera inside: no positive near root
      *x0 = 1; *x1 = 0;
      return;
    }
    if (pz - r <= 1e-9 * r) return;  // reaches behind the camera plane: whole image (rare)
    const double tan_half = tan(C.fov / 2.0);
    const double sx = 2.0 * tan_half * static_cast<double>(W) / static_cast<double>(H);
    const double sy = 2.0 * tan_half;
    const double ax = atan2(px, pz), aax = asin(fmin(1.0, r / hypot(px, pz)));
    const double ay = atan2(py, pz), aay = asin(fmin(1.0, r / hypot(py, pz)));
    const double gx0 = tan(ax - aax) / sx, gx1 = tan(ax + aax) / sx;
    const double gy0 = tan(ay - aay) / sy, gy1 = tan(ay + aay) / sy;
    *x0 = max(0, static_cast<int>(floor((gx0 + 0.5) * W - 0.5)) - 1);
    *x1 = min(W - 1, static_cast<int>(ceil((gx1 + 0.5) * W - 0.5)) + 1);
    *y0 = max(0, static_cast<int>(floor((gy0 + 0.5) * H - 0.5)) - 1);
    *y1 = min(H - 1, static_cast<int>(ceil((gy1 + 0.5) * H - 0.5)) + 1);
  } else {
    const double w = C.extent[0], h = C.extent[1];
    *x0 = max(0, static_cast<int>(floor(((px - r) / w + 0.5) * W - 0.5)) - 1);
    *x1 = min(W - 1, static_cast<int>(ceil(((px + r) / w + 0.5) * W - 0.5)) + 1);
    *y0 = max(0, static_cast<int>(floor(((py - r) / h + 0.5) * H - 0.5)) - 1);
    *y1 = min(H - 1, static_cast<int>(ceil(((py + r) / h + 0.5) * H - 0.5)) + 1);
  }
}

__global__ void __launch_bounds__(kBlock) k_render_splat(Dev D, RenderArgs A,
                                                         unsigned long long* __restrict__ zbuf) {
  const int env = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= D.ne) return;
  const float4 cf = D.X[D.ctl->cur][static_cast<long long>(env) * D.ne + q];
  const double cx = cf.x, cy = cf.y, cz = cf.z;
  const double r = D.r, r2 = D.r * D.r;
  const long long base = static_cast<long long>(env) * A.pix_off[A.n_cams];
  for (int cam = 0; cam < A.n_cams; ++cam) {
    const gg_camera& C = A.cams[A.per_env ? env * A.n_cams + cam : cam];
    int x0, x1, y0, y1;
    splat_box(C, cx, cy, cz, r, &x0, &x1, &y0, &y1);
    unsigned long long* z = zbuf + base + A.pix_off[cam];
    for (int iy = y0; iy <= y1; ++iy)
      for (int ix = x0; ix <= x1; ++ix) {
        const int p = iy * C.width + ix;
        double o[3], d[3];
        camera_ray(C, A.local + 3 * (A.pix_off[cam] + p), o, d);
        const double ocx = o[0] - cx, ocy = o[1] - cy, ocz = o[2] - cz;
        const double b = ocx * d[0] + ocy * d[1] + ocz * d[2];
        const double cterm = (ocx * ocx + ocy * ocy + ocz * ocz) - r2;
        const double disc = b * b - cterm;
        if (!(disc >= 0.0)) continue;
        const double t = -b - sqrt(disc);
        if (t > 0.0 && t < C.far) atomicMin(z + p, static_cast<unsigned long long>(__double_as_longlong(t)));
      }
  }
}

// per pixel: the splatted particle depth, then the bodies (sphere tracing)
__global__ void __launch_bounds__(kBlock) k_render_bodies(Dev D, RenderArgs A,
                                                          const unsigned long long* __restrict__ zbuf) {
  const int env = blockIdx.z, cam = blockIdx.y;
  const gg_camera& C = A.cams[A.per_env ? env * A.n_cams + cam : cam];
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= C.width * C.height) return;
  const long long idx = static_cast<long long>(env) * A.pix_off[A.n_cams] + A.pix_off[cam] + p;
  const unsigned long long zb = zbuf[idx];
  const double far = C.far;
  double best = zb == ~0ull ? far : __longlong_as_double(static_cast<long long>(zb));
  double o[3], d[3];
  camera_ray(C, A.local + 3 * (A.pix_off[cam] + p), o, d);
  const gg_body* bodies = A.bodies + static_cast<long long>(env) * A.nb;
  for (int bi = 0; bi < A.nb; ++bi) {
    const gg_body& B = bodies[bi];
    const double* R = B.rot;
    const double ex = o[0] - B.trans[0], ey = o[1] - B.trans[1], ez = o[2] - B.trans[2];
    const double lo0 = fma(ez, R[6], fma(ey, R[3], ex * R[0]));
    const double lo1 = fma(ez, R[7], fma(ey, R[4], ex * R[1]));
    const double lo2 = fma(ez, R[8], fma(ey, R[5], ex * R[2]));
    const double ld0 = fma(d[2], R[6], fma(d[1], R[3], d[0] * R[0]));
    const double ld1 = fma(d[2], R[7], fma(d[1], R[4], d[0] * R[1]));
    const double ld2 = fma(d[2], R[8], fma(d[1], R[5], d[0] * R[2]));
    double t = 0.0;
    for (int it = 0; it < kTraceSteps; ++it) {
      const double f = sdf_distance(B, D.grids, D.gvals, lo0 + t * ld0, lo1 + t * ld1, lo2 + t * ld2);
      if (f < kTraceEps) {
        best = t < best ? t : best;
        break;
      }
      t += (f > kTraceEps ? f : kTraceEps) * 0.9;
      if (!(t < far)) break;
    }
  }
  A.out[idx] = static_cast<float>(best < far ? best : far);
}

}  // namespace gg
