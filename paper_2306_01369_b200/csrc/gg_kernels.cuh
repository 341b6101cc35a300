// gg_kernels.cuh — the per-step kernels of the split pipeline
// (stepper.py:57-135, TWO_LOOPS_SPLIT):
//
//   K1 k_hash_count   cell + hash per particle, bucket occupancy (atomic)
//   K2 k_scan_*       exclusive scan of bucket counts -> bucket starts
//   K3 k_scatter      counting-sort scatter (arrival order within bucket)
//   K4 k_reorder      stable fix-up (ties by user id) + gather x, v to sorted SoA
//   K5 k_narrow       pp narrowphase over 27 de-duplicated buckets + body SDF contacts
//   K7 k_sweep (xS)   projected-Jacobi sweep, owner-computes, atomic-free
//   K8 k_integrate    symplectic Euler + cyclic boundary + NaN check + KE
//   K9 k_finalize     fixed-order reductions -> StepReport, commit
//
// Layout (all in HBM, n = particles):
//   X[2], V[2]  float4   committed state, in the PREVIOUS step's sorted order
//   UID[2]      int32    sorted position -> user particle id
//   Xs, V0      float4   this step's sorted positions / start-of-step velocity
//   W[2]        float4   predicted velocity w = v + dv, ping-ponged per sweep
//   cgeo[K][n]  float4   contact (e1.xyz, psi)   slot-major, coalesced per slot
//   coth[K][n]  int32    other: >=0 sorted particle index, <0 -> body -(b+1)
//   cvb[K][n]   float4   body surface velocity (body contacts only)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gg_device.cuh"

namespace gg {

constexpr int kBlock = 256;
constexpr int kScanTile = 2048;        // elements per scan tile (256 thr x 8)
constexpr int kRegBodies = 4;          // bodies with deterministic in-register momentum
constexpr int kMaxBad = 32;

struct Ctl {
  int cur;        // committed state buffer
  int step;       // steps committed in this batch
  int err;        // first error code (0 = none)
  int err_step;   // batch-relative step of the error
  int cap_needed; // largest per-owner contact count seen (capacity hint)
  int n_bad;      // non-finite particles recorded
  int pad[2];
  int bad_uid[kMaxBad];
};

struct Acc {
  unsigned long long n_pp, n_cand, n_body, n_coinc, n_deg;
  unsigned long long max_psi_bits, max_viol_bits, min_b1_bits;
};

struct Dev {
  int n, K, nb, S, nblocks;
  HashCfg H;
  double r, two_r, contact_d2, coinc_d2, mass, mu, alpha, dt, gamma;
  double gdt0, gdt1, gdt2;
  int has_boundary;
  double z_min, band;
  float4* X[2];
  float4* V[2];
  int* UID[2];
  uint32_t* key;
  uint32_t* arrive;
  uint32_t* cnt;
  uint32_t* start;
  uint32_t* tile;
  int* tmp;
  float4* Xs;
  float4* V0;
  float4* W[2];
  float4* cgeo;
  int* coth;
  float4* cvb;
  int* ccount;
  const gg_body* bodies;  // [batch][nb]
  const DevGrid* grids;
  const double* gvals;
  Acc* acc;
  double* ke_part;  // [nblocks]
  double* bm_part;  // [nblocks][nb][3]
  double* bm_glob;  // [nb][3] fallback accumulators for bodies >= kRegBodies
  gg_report* reports;
  double* bm_out;   // [batch][nb][3]
  Ctl* ctl;
};

// ---------------------------------------------------------------------------
__device__ __forceinline__ void raise_err(Ctl* ctl, int code) {
  if (atomicCAS(&ctl->err, 0, code) == 0) ctl->err_step = ctl->step;
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nmin(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block reduction of a double (deterministic).  All threads call.
template <int kOp>  // 0 sum, 1 max, 2 min
__device__ __forceinline__ double block_reduce(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = kOp == 0 ? warp_sum(v) : (kOp == 1 ? warp_max(v) : warp_min(v));
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  double r = sm[0];
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      r = kOp == 0 ? r + sm[w] : (kOp == 1 ? nmax(r, sm[w]) : nmin(r, sm[w]));
  }
  return r;  // valid on thread 0
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v,
                                                            unsigned long long* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  unsigned long long r = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sm[w];
  return r;
}

// block-uniform early exit: every kernel that syncs reads err through smem
__device__ __forceinline__ bool block_should_exit(const Ctl* ctl) {
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = *((volatile const int*)&ctl->err);
  __syncthreads();
  return s_err != 0;
}

// ---------------------------------------------------------------------------
// batch begin: reset per-batch control + per-step accumulators
// ---------------------------------------------------------------------------
__global__ void k_batch_begin(Dev D) {
  Ctl* c = D.ctl;
  c->step = 0;
  c->err = 0;
  c->err_step = -1;
  c->cap_needed = 0;
  c->n_bad = 0;
  Acc* a = D.acc;
  a->n_pp = a->n_cand = a->n_body = a->n_coinc = a->n_deg = 0;
  a->max_psi_bits = 0;
  a->max_viol_bits = 0;
  a->min_b1_bits = dbits(__longlong_as_double(0x7ff0000000000000ll));
  for (int i = 0; i < D.nb * 3; ++i) D.bm_glob[i] = 0.0;
}

// ---------------------------------------------------------------------------
// K1: cell + hash + bucket occupancy (build_hashmap, broadphase.py:89-130)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_hash_count(Dev D) {
  const Ctl* ctl = D.ctl;
  if (ctl->err) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  const float4 p = D.X[ctl->cur][i];
  if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z)) {
    raise_err(D.ctl, GG_EPOSITIONS);
    return;
  }
  const long long c0 = cell_coord(p.x, D.two_r);
  const long long c1 = cell_coord(p.y, D.two_r);
  const long long c2 = cell_coord(p.z, D.two_r);
  const uint32_t h = hash_cell(c0, c1, c2, D.H);
  D.key[i] = h;
  D.arrive[i] = atomicAdd(&D.cnt[h], 1u);
}

// ---------------------------------------------------------------------------
// K2: exclusive scan of cnt[0..n_h) -> start[0..n_h)   (start[n_h] = n fixed)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* sm, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t s = lane < nw ? sm[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sm[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t warp_off = wid ? sm[wid - 1] : 0u;
  *total = sm[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_off + x - v;
}

__global__ void __launch_bounds__(kBlock) k_scan_tiles(Dev D) {
  if (D.ctl->err) return;
  __shared__ uint32_t sm[32];
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile + threadIdx.x * 8;
  uint32_t s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (base + e < D.H.n_h) s += D.cnt[base + e];
  uint32_t total;
  (void)block_excl_scan_u32(s, sm, &total);
  if (threadIdx.x == 0) D.tile[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_top(Dev D, int ntiles) {
  if (D.ctl->err) return;
  __shared__ uint32_t sm[32];
  const int per = (ntiles + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  uint32_t s = 0;
  for (int e = 0; e < per; ++e)
    if (b0 + e < ntiles) s += D.tile[b0 + e];
  uint32_t total;
  uint32_t run = block_excl_scan_u32(s, sm, &total);
  for (int e = 0; e < per; ++e)
    if (b0 + e < ntiles) {
      const uint32_t t = D.tile[b0 + e];
      D.tile[b0 + e] = run;
      run += t;
    }
}

__global__ void __launch_bounds__(kBlock) k_scan_apply(Dev D) {
  if (D.ctl->err) return;
  __shared__ uint32_t sm[32];
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile + threadIdx.x * 8;
  uint32_t v[8];
  uint32_t s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    v[e] = (base + e < D.H.n_h) ? D.cnt[base + e] : 0u;
    s += v[e];
  }
  uint32_t total;
  uint32_t run = block_excl_scan_u32(s, sm, &total) + D.tile[blockIdx.x];
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (base + e < D.H.n_h) {
      D.start[base + e] = run;
      run += v[e];
    }
}

// ---------------------------------------------------------------------------
// K3: counting-sort scatter (arrival order inside a bucket)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_scatter(Dev D) {
  if (D.ctl->err) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  D.tmp[D.start[D.key[i]] + D.arrive[i]] = i;
}

// ---------------------------------------------------------------------------
// K4: stable fix-up + reorder.  Final position inside a bucket = number of
// bucket members with a smaller USER id, which reproduces
// np.argsort(hashes, kind="stable") / lexsort((rank, hashes)) exactly
// (broadphase.py:122,160).  Gathers x, v into the sorted layout.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_reorder(Dev D) {
  const Ctl* ctl = D.ctl;
  if (ctl->err) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = ctl->cur;
  const int* __restrict__ uid_in = D.UID[cur];
  const int p = D.tmp[k];
  const int uid = uid_in[p];
  const uint32_t h = D.key[p];
  const uint32_t s = D.start[h], e = D.start[h + 1];
  uint32_t rank = 0;
  for (uint32_t m = s; m < e; ++m) rank += (uid_in[D.tmp[m]] < uid) ? 1u : 0u;
  const uint32_t f = s + rank;
  D.UID[cur ^ 1][f] = uid;
  D.Xs[f] = D.X[cur][p];
  D.V0[f] = D.V[cur][p];
}

// ---------------------------------------------------------------------------
// K5: narrowphase (narrowphase_contacts, contact.py:244-300 with
// candidate_pairs_with_distances, broadphase.py:149-221).  One thread per
// sorted particle; 27 neighbour buckets, duplicates among the non-empty ones
// skipped (the reference's sort + dedupe, broadphase.py:164-171).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_narrow(Dev D) {
  __shared__ double smd[32];
  __shared__ unsigned long long smu[32];
  const Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const int step = ctl->step;
  const gg_body* __restrict__ bodies = D.bodies + static_cast<long long>(step) * D.nb;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = k < D.n;
  unsigned long long n_pp = 0, n_cand = 0, n_coinc = 0, n_body = 0, n_deg = 0;
  double max_psi = 0.0;
  if (active) {
    const float4 pf = D.Xs[k];
    const double px = pf.x, py = pf.y, pz = pf.z;
    const long long c0 = cell_coord(px, D.two_r);
    const long long c1 = cell_coord(py, D.two_r);
    const long long c2 = cell_coord(pz, D.two_r);
    uint32_t tx[3], ty[3], tz[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      tx[d] = hash_term32(c0 + d - 1, kP0);
      ty[d] = hash_term32(c1 + d - 1, kP1);
      tz[d] = hash_term32(c2 + d - 1, kP2);
    }
    const long long K = D.K;
    const long long n = D.n;
    int cnt = 0;
    uint32_t seen[27];
    int nseen = 0;
    for (int o = 0; o < 27; ++o) {
      const int ox = o / 9, oy = (o / 3) % 3, oz = o % 3;
      const uint32_t h =
          D.H.pow2 ? ((tx[ox] ^ ty[oy] ^ tz[oz]) & D.H.mask)
                   : hash_cell64(c0 + ox - 1, c1 + oy - 1, c2 + oz - 1, D.H.n_h);
      const uint32_t s = D.start[h], e = D.start[h + 1];
      if (s == e) continue;
      bool dup = false;
      for (int q = 0; q < nseen; ++q) dup |= (seen[q] == h);
      if (dup) continue;
      seen[nseen++] = h;
      n_cand += e - s;
      for (uint32_t m = s; m < e; ++m) {
        if (static_cast<int>(m) == k) continue;
        const float4 qf = D.Xs[m];
        const double dx = __dsub_rn(px, static_cast<double>(qf.x));
        const double dy = __dsub_rn(py, static_cast<double>(qf.y));
        const double dz = __dsub_rn(pz, static_cast<double>(qf.z));
        // einsum("ij,ij->i") on this numpy build: (dx^2 + dz^2) + dy^2
        const double d2 =
            __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
        if (!(d2 >= D.coinc_d2)) {
          ++n_coinc;
          continue;
        }
        if (d2 < D.contact_d2) {
          const double dist = __dsqrt_rn(d2);
          const double psi = __dsub_rn(D.two_r, dist);
          if (cnt < K) {
            const long long sl = cnt * n + k;
            D.cgeo[sl] = make_float4(static_cast<float>(__ddiv_rn(dx, dist)),
                                     static_cast<float>(__ddiv_rn(dy, dist)),
                                     static_cast<float>(__ddiv_rn(dz, dist)),
                                     static_cast<float>(psi));
            D.coth[sl] = static_cast<int>(m);
          }
          ++cnt;
          max_psi = nmax(max_psi, psi);
        }
      }
    }
    n_cand -= 1;  // the self pair (one per particle, broadphase.py:441-447)
    n_pp = cnt;
    // body pass (contact.py:274-286), bodies in index order
    for (int b = 0; b < D.nb; ++b) {
      const gg_body& B = bodies[b];
      if (B.bounded) {
        if (!(px >= B.aabb_lo[0] && px <= B.aabb_hi[0] && py >= B.aabb_lo[1] &&
              py <= B.aabb_hi[1] && pz >= B.aabb_lo[2] && pz <= B.aabb_hi[2]))
          continue;
      }
      double psi;
      d3 nrm;
      int deg;
      if (penetrate(B, D.grids, D.gvals, px, py, pz, D.r, &psi, &nrm, &deg)) {
        if (cnt < K) {
          const long long sl = cnt * n + k;
          const d3 vb = body_surface_velocity(B, px, py, pz, nrm, D.r, psi);
          D.cgeo[sl] = make_float4(static_cast<float>(nrm.x), static_cast<float>(nrm.y),
                                   static_cast<float>(nrm.z), static_cast<float>(psi));
          D.coth[sl] = -(b + 1);
          D.cvb[sl] = make_float4(static_cast<float>(vb.x), static_cast<float>(vb.y),
                                  static_cast<float>(vb.z), 0.f);
        }
        ++cnt;
        ++n_body;
        max_psi = nmax(max_psi, psi);
      }
      n_deg += deg;
    }
    D.ccount[k] = cnt < K ? cnt : static_cast<int>(K);
    if (cnt > K) {
      atomicMax(&D.ctl->cap_needed, cnt);
      raise_err(D.ctl, GG_ECAPACITY);
    }
  }
  // reductions (integers are order-independent; max via bit pattern of a
  // non-negative double)
  unsigned long long t;
  t = block_sum_u64(n_pp, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_pp, t);
  t = block_sum_u64(n_cand, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_cand, t);
  t = block_sum_u64(n_coinc, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_coinc, t);
  t = block_sum_u64(n_body, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_body, t);
  t = block_sum_u64(n_deg, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_deg, t);
  const double mp = block_reduce<1>(max_psi, smd);
  if (threadIdx.x == 0 && mp > 0.0) atomicMax(&D.acc->max_psi_bits, dbits(mp));
}

// ---------------------------------------------------------------------------
// K7: one projected-Jacobi sweep (solve_contacts_pja, contact.py:463-501).
// w = v + dv is the predicted velocity; every contact of owner i reads w of
// the previous sweep for both i and j, so the sweep is Jacobi-synchronous and
// each thread writes only its own w (no atomics).  The tangential impulse is
// -(u - (u.e1) e1), identical to e2*b2 + e3*b3 for the orthonormal frame the
// reference builds (contact.py:47-56), so the frame is never materialised.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_sweep(Dev D, int s) {
  __shared__ double smd[32];
  const Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const float4* __restrict__ Win = (s == 0) ? D.V0 : D.W[(s - 1) & 1];
  float4* __restrict__ Wout = D.W[s & 1];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = k < D.n;
  double maxviol = 0.0;
  double minb1 = __longlong_as_double(0x7ff0000000000000ll);
  double bm[kRegBodies][3];
#pragma unroll
  for (int b = 0; b < kRegBodies; ++b) bm[b][0] = bm[b][1] = bm[b][2] = 0.0;
  if (active) {
    const float4 wf = Win[k];
    const double wx = wf.x, wy = wf.y, wz = wf.z;
    double ax = 0.0, ay = 0.0, az = 0.0;
    const int c = D.ccount[k];
    const long long n = D.n;
    for (int sl = 0; sl < c; ++sl) {
      const long long idx = sl * n + k;
      const float4 g = D.cgeo[idx];
      const int j = D.coth[idx];
      double vjx, vjy, vjz, eff;
      if (j >= 0) {
        const float4 q = Win[j];
        vjx = q.x; vjy = q.y; vjz = q.z;
        eff = 0.5;  // both partners mobile (contact.py:457-460)
      } else {
        const float4 q = D.cvb[idx];
        vjx = q.x; vjy = q.y; vjz = q.z;
        eff = 1.0;
      }
      const double e1x = g.x, e1y = g.y, e1z = g.z, psi = g.w;
      const double ux = (wx - D.gamma * vjx) + D.gdt0;
      const double uy = (wy - D.gamma * vjy) + D.gdt1;
      const double uz = (wz - D.gamma * vjz) + D.gdt2;
      const double un = ux * e1x + uy * e1y + uz * e1z;
      const double bias = D.alpha * psi / D.dt;
      const double b1 = nmax(-un + bias, 0.0);
      double btx = -(ux - un * e1x), bty = -(uy - un * e1y), btz = -(uz - un * e1z);
      const double tn = sqrt(btx * btx + bty * bty + btz * btz);
      const double lim = D.mu * b1;
      const double scale = (tn > lim) ? lim / fmax(tn, 1e-300) : 1.0;
      btx *= scale; bty *= scale; btz *= scale;
      const double ix = (e1x * b1 + btx) * eff;
      const double iy = (e1y * b1 + bty) * eff;
      const double iz = (e1z * b1 + btz) * eff;
      ax += ix; ay += iy; az += iz;
      maxviol = nmax(maxviol, tn * scale - lim);
      minb1 = nmin(minb1, b1);
      if (j < 0) {
        const int b = -j - 1;
        const double mx = -D.mass * ix, my = -D.mass * iy, mz = -D.mass * iz;
        bool placed = false;
#pragma unroll
        for (int q = 0; q < kRegBodies; ++q)
          if (q == b) { bm[q][0] += mx; bm[q][1] += my; bm[q][2] += mz; placed = true; }
        if (!placed) {
          atomicAdd(&D.bm_glob[b * 3 + 0], mx);
          atomicAdd(&D.bm_glob[b * 3 + 1], my);
          atomicAdd(&D.bm_glob[b * 3 + 2], mz);
        }
      }
    }
    Wout[k] = make_float4(static_cast<float>(wx + ax), static_cast<float>(wy + ay),
                          static_cast<float>(wz + az), 0.f);
  }
  const double mv = block_reduce<1>(maxviol, smd);
  if (threadIdx.x == 0 && mv > 0.0) atomicMax(&D.acc->max_viol_bits, dbits(mv));
  const double mb = block_reduce<2>(minb1, smd);
  if (threadIdx.x == 0 && mb == mb) atomicMin(&D.acc->min_b1_bits, dbits(mb));
  const int nreg = D.nb < kRegBodies ? D.nb : kRegBodies;
  for (int b = 0; b < nreg; ++b) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kRegBodies; ++q)
        if (q == b) v = bm[q][a];
      const double tot = block_reduce<0>(v, smd);
      if (threadIdx.x == 0) {
        double* dst = &D.bm_part[(static_cast<long long>(blockIdx.x) * D.nb + b) * 3 + a];
        *dst = (s == 0) ? tot : *dst + tot;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K8: integrate (stepper.py:102-106) + SolverError check (contact.py:503-509)
// + kinetic energy partials (stepper.py:118).  Writes the uncommitted state
// buffer; k_finalize commits it only when the step raised nothing.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_integrate(Dev D) {
  __shared__ double smd[32];
  const Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const int cur = ctl->cur;
  const float4* __restrict__ Wf = D.S > 0 ? D.W[(D.S - 1) & 1] : D.V0;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  double ke = 0.0;
  if (k < D.n) {
    const float4 xo = D.Xs[k];
    const float4 vo = D.V0[k];
    const float4 wf = Wf[k];
    const bool has = D.ccount[k] > 0;
    const double dvx = has ? (double)wf.x - (double)vo.x : 0.0;
    const double dvy = has ? (double)wf.y - (double)vo.y : 0.0;
    const double dvz = has ? (double)wf.z - (double)vo.z : 0.0;
    if (!isfinite(dvx) || !isfinite(dvy) || !isfinite(dvz)) {
      const int slot = atomicAdd(&D.ctl->n_bad, 1);
      if (slot < kMaxBad) D.ctl->bad_uid[slot] = D.UID[cur ^ 1][k];
      raise_err(D.ctl, GG_ENONFINITE);
    }
    // v += dt*g + dv ; x += dt*v
    const double vx = __dadd_rn((double)vo.x, __dadd_rn(D.gdt0, dvx));
    const double vy = __dadd_rn((double)vo.y, __dadd_rn(D.gdt1, dvy));
    const double vz = __dadd_rn((double)vo.z, __dadd_rn(D.gdt2, dvz));
    const double x = __dadd_rn((double)xo.x, __dmul_rn(D.dt, vx));
    const double y = __dadd_rn((double)xo.y, __dmul_rn(D.dt, vy));
    double z = __dadd_rn((double)xo.z, __dmul_rn(D.dt, vz));
    if (D.has_boundary && z < D.z_min) z = __dadd_rn(z, D.band);  // stepper.py:138-144
    D.X[cur ^ 1][k] = make_float4(static_cast<float>(x), static_cast<float>(y),
                                  static_cast<float>(z), 0.f);
    D.V[cur ^ 1][k] = make_float4(static_cast<float>(vx), static_cast<float>(vy),
                                  static_cast<float>(vz), 0.f);
    ke = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
  }
  const double kb = block_reduce<0>(ke, smd);
  if (threadIdx.x == 0) D.ke_part[blockIdx.x] = kb;
}

// ---------------------------------------------------------------------------
// K9: fixed-order reduction of the per-block partials -> StepReport; commit.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_finalize(Dev D) {
  __shared__ double smd[32];
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const int step = ctl->step;
  double ke = 0.0;
  for (int b = threadIdx.x; b < D.nblocks; b += blockDim.x) ke += D.ke_part[b];
  const double ke_tot = block_reduce<0>(ke, smd);
  for (int q = 0; q < D.nb * 3; ++q) {
    double v = 0.0;
    const int b = q / 3;
    if (b < kRegBodies)
      for (int blk = threadIdx.x; blk < D.nblocks; blk += blockDim.x)
        v += D.bm_part[static_cast<long long>(blk) * D.nb * 3 + q];
    const double tot = block_reduce<0>(v, smd);
    if (threadIdx.x == 0) {
      D.bm_out[static_cast<long long>(step) * D.nb * 3 + q] =
          b < kRegBodies ? (D.S > 0 ? tot : 0.0) : D.bm_glob[q];
      D.bm_glob[q] = 0.0;
    }
  }
  if (threadIdx.x == 0) {
    Acc* a = D.acc;
    gg_report& R = D.reports[step];
    R.n_contacts = static_cast<long long>(a->n_pp);
    R.n_candidates = static_cast<long long>(a->n_cand);
    R.n_body_contacts = static_cast<long long>(a->n_body);
    R.n_coincident = static_cast<long long>(a->n_coinc);
    R.n_degenerate = static_cast<long long>(a->n_deg);
    R.max_penetration = __longlong_as_double(static_cast<long long>(a->max_psi_bits));
    R.kinetic_energy = 0.5 * D.mass * ke_tot;
    R.max_cone_violation = __longlong_as_double(static_cast<long long>(a->max_viol_bits));
    R.min_normal_impulse = __longlong_as_double(static_cast<long long>(a->min_b1_bits));
    a->n_pp = a->n_cand = a->n_body = a->n_coinc = a->n_deg = 0;
    a->max_psi_bits = 0;
    a->max_viol_bits = 0;
    a->min_b1_bits = dbits(__longlong_as_double(0x7ff0000000000000ll));
    ctl->cur ^= 1;
    ctl->step = step + 1;
  }
}

// ---------------------------------------------------------------------------
// state upload / download helpers
// ---------------------------------------------------------------------------
__global__ void k_load_f64(Dev D, const double* __restrict__ x, const double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  const int cur = D.ctl->cur;
  D.X[cur][i] = make_float4(static_cast<float>(x[3 * i]), static_cast<float>(x[3 * i + 1]),
                            static_cast<float>(x[3 * i + 2]), 0.f);
  D.V[cur][i] = make_float4(static_cast<float>(v[3 * i]), static_cast<float>(v[3 * i + 1]),
                            static_cast<float>(v[3 * i + 2]), 0.f);
  D.UID[cur][i] = i;
}

__global__ void k_store_f64(Dev D, double* __restrict__ x, double* __restrict__ v) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = D.ctl->cur;
  const int u = D.UID[cur][k];
  const float4 p = D.X[cur][k], q = D.V[cur][k];
  x[3 * u] = p.x; x[3 * u + 1] = p.y; x[3 * u + 2] = p.z;
  v[3 * u] = q.x; v[3 * u + 1] = q.y; v[3 * u + 2] = q.z;
}

__global__ void k_load_f4(Dev D, const float4* __restrict__ x, const float4* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  const int cur = D.ctl->cur;
  float4 a = x[i], b = v[i];
  a.w = 0.f; b.w = 0.f;
  D.X[cur][i] = a;
  D.V[cur][i] = b;
  D.UID[cur][i] = i;
}

__global__ void k_store_f4(Dev D, float4* __restrict__ x, float4* __restrict__ v) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = D.ctl->cur;
  const int u = D.UID[cur][k];
  x[u] = D.X[cur][k];
  v[u] = D.V[cur][k];
}

// cells + hashes of the committed state, user order (parity tap)
__global__ void k_tap_cells(Dev D, long long* __restrict__ cells, long long* __restrict__ hashes) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = D.ctl->cur;
  const int u = D.UID[cur][k];
  const float4 p = D.X[cur][k];
  const long long c0 = cell_coord(p.x, D.two_r);
  const long long c1 = cell_coord(p.y, D.two_r);
  const long long c2 = cell_coord(p.z, D.two_r);
  cells[3 * u] = c0; cells[3 * u + 1] = c1; cells[3 * u + 2] = c2;
  hashes[u] = hash_cell(c0, c1, c2, D.H);
}

__global__ void k_hash_cells(const long long* __restrict__ cells, long long k, HashCfg H,
                             long long* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  out[i] = H.pow2 ? static_cast<long long>(hash_cell(cells[3 * i], cells[3 * i + 1], cells[3 * i + 2], H))
                  : hash_cell64_full(cells[3 * i], cells[3 * i + 1], cells[3 * i + 2], H.n_h);
}

__global__ void k_penetration(gg_body B, const DevGrid* __restrict__ grids,
                              const double* __restrict__ gvals, const double* __restrict__ pts,
                              long long n, double r, double* __restrict__ psi,
                              double* __restrict__ nrm, int* __restrict__ hit,
                              unsigned long long* __restrict__ ndeg) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ps = 0.0;
  d3 nv{0.0, 0.0, 0.0};
  int deg = 0;
  const int h = penetrate(B, grids, gvals, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], r, &ps,
                          &nv, &deg);
  psi[i] = h ? ps : 0.0;
  nrm[3 * i] = h ? nv.x : 0.0;
  nrm[3 * i + 1] = h ? nv.y : 0.0;
  nrm[3 * i + 2] = h ? nv.z : 0.0;
  hit[i] = h;
  if (deg) atomicAdd(ndeg, 1ull);
}

}  // namespace gg
