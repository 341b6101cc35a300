// gg_kernels.cuh — the per-step kernels of the split pipeline
// (stepper.py:57-135, TWO_LOOPS_SPLIT), B200 layout:
//
//   physical order   particles live in a spatially coherent order (Morton
//                    code of their cell, low bits), re-sorted every
//                    `resort_every` steps by the same deterministic counting
//                    sort the hash index uses (R1-R4).  Neighbours of a warp's
//                    particles are then neighbours in memory, so the
//                    narrowphase and solver gathers hit L1/L2.
//   hash index       rebuilt every step over the physical order (H1-H4):
//                    bucket counts -> scan -> scatter -> stable fill of
//                    Xh[bucket order] = (x, y, z, physical index), ties by
//                    user id, i.e. exactly np.argsort(hashes, kind="stable")
//                    (broadphase.py:160) — candidates are read with ONE
//                    float4 load each.
//   K5 k_narrow      pp narrowphase over the 27 neighbour buckets (de-duplicated,
//                    broadphase.py:164-171) + body SDF contacts -> slot-major
//                    contact records.
//   K7 k_solve       one cooperative persistent kernel: S projected-Jacobi
//                    sweeps separated by grid barriers, symplectic Euler,
//                    cyclic boundary, NaN check, fixed-order reductions into
//                    the StepReport and the commit.
//
// Buffers (n particles, K slots):
//   X[2], V[2]  float4  committed state (physical order), ping-pong on commit
//   UID[2]      int32   physical index -> user id, flips on re-sort steps
//   Xs, V0      float4  re-sorted layout of this step (re-sort steps only)
//   Xh          float4  bucket-ordered copy (x, y, z, bits(physical index))
//   W[2]        float4  predicted velocity w = v + dv, ping-ponged per sweep
//   cgeo[K][n]  float4  (e1.xyz, psi)     coth[K][n] int32 other (<0: body)
//   cvb[K][n]   float4  body surface velocity (body contacts only)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gg_device.cuh"

namespace gg {

constexpr int kBlock = 256;
constexpr int kScanTile = 2048;  // elements per scan tile (256 thr x 8)
constexpr int kMaxBad = 32;
constexpr int kMaxFusedBlocks = 1024;  // neighbour-flag sweeps: block-set bitmask size

struct Ctl {
  int cur;         // committed state buffer
  int ucur;        // committed uid buffer
  int step;        // steps committed in this batch
  int err;         // first error code (0 = none)
  int err_step;    // batch-relative step of the error
  int cap_needed;  // largest per-owner contact count seen (capacity hint)
  int n_bad;       // non-finite particles recorded
  int pad;
  unsigned bar_count;  // grid barrier arrivals (monotonic within a launch, reset per launch)
  unsigned done_count; // last-block-done counter of the solve kernel
  unsigned bar_gen;    // last completed barrier target (reset with bar_count)
  unsigned pad2;
  int bad_uid[kMaxBad];
};

struct Acc {
  unsigned long long n_pp, n_cand, n_body, n_coinc, n_deg;
  unsigned long long max_psi_bits, max_viol_bits, min_b1_bits;
};

// body reaction momentum is accumulated in 64-bit fixed point so the sum is
// independent of the order in which contacts add to it (deterministic)
constexpr double kMomScale = 68719476736.0;  // 2^36
__device__ __forceinline__ unsigned long long to_fix(double v) {
  return static_cast<unsigned long long>(__double2ll_rn(v * kMomScale));
}

struct Dev {
  int n, K, nb, S, nblocks;
  int resort;     // this graph re-sorts the physical order first
  int key_morton; // counting-sort key of the current pass (R: 1, H: 0)
  HashCfg H;
  uint32_t mmask;  // Morton key mask (power of two <= n_h, minus one)
  double r, two_r, contact_d2, coinc_d2, mass, mu, alpha, dt, gamma, bias_coef;
  float reject_d2f;  // float32 pre-filter: d2_f32 > this  =>  d2 >= contact_d2 exactly
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
  float4* Xh;
  float4* W[2];
  float4* cgeo;
  int* coth;
  float4* cvb;
  int* ccount;
  const gg_body* bodies;  // [batch][nb]
  const DevGrid* grids;
  const double* gvals;
  Acc* acc;
  unsigned long long* tstamp;  // optional phase timestamps of the fused kernel (64)
  unsigned* bflags;  // [fused grid] per-block sweep progress (fused kernel)
  double* part;     // [nblocks_solve] per-block kinetic-energy partials
  unsigned long long* bm_fix;  // [nb][3] fixed-point body momentum of the step
  gg_report* reports;
  double* bm_out;  // [batch][nb][3]
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

// Fixed-order block reduction of a double (deterministic); result on thread 0.
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
  return r;
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

// Grid-wide barrier for the cooperative kernel (all blocks co-resident).
// One release-add per block on a counter that only grows during a launch
// (zeroed by a memset node before the launch); blocks wait with acquire loads
// until it reaches the barrier's target (nblocks x barrier ordinal).
__device__ __forceinline__ void grid_barrier(Ctl* ctl, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // arrive on the counter; the last arriver publishes the barrier ordinal
    // on a separate generation word, which is all the waiters poll (they
    // never contend with the arrival atomics)
    unsigned v;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(&ctl->bar_count) : "memory");
    if (v + 1 == target) {
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&ctl->bar_gen), "r"(target) : "memory");
    } else {
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&ctl->bar_gen) : "memory");
      } while (static_cast<int>(v - target) < 0);
    }
    // gpu-scope fence: invalidates this SM's L1 (CCTL.IVALL) so no block
    // reads a line cached before other SMs rewrote it in the previous phase
    __threadfence();
  }
  __syncthreads();
}

// the layout the step works on: re-sorted this step, or the committed one
struct Layout {
  const float4* x;
  const float4* v;
  const int* uid;
};
__device__ __forceinline__ Layout layout(const Dev& D, const Ctl* ctl) {
  const int cur = ctl->cur, u = ctl->ucur;
  if (D.resort) return {D.Xs, D.V0, D.UID[u ^ 1]};
  return {D.X[cur], D.V[cur], D.UID[u]};
}

// ---------------------------------------------------------------------------
// Morton key of a cell: interleaved low bits (wraps into tiles), masked to
// the table size.  Only locality matters; any deterministic key is correct.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__device__ __forceinline__ uint32_t morton_key(long long c0, long long c1, long long c2,
                                               uint32_t mask) {
  return (spread3(static_cast<uint32_t>(c0)) | (spread3(static_cast<uint32_t>(c1)) << 1) |
          (spread3(static_cast<uint32_t>(c2)) << 2)) & mask;
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
  c->bar_count = 0;
  c->done_count = 0;
  c->bar_gen = 0;
  Acc* a = D.acc;
  a->n_pp = a->n_cand = a->n_body = a->n_coinc = a->n_deg = 0;
  a->max_psi_bits = a->max_viol_bits = 0;
  a->min_b1_bits = dbits(__longlong_as_double(0x7ff0000000000000ll));
  for (int i = 0; i < D.nb * 3; ++i) D.bm_fix[i] = 0ull;
}

// ===========================================================================
// Phases.  Element-wise phases (ph_count, ph_scatter, ph_resort, ph_fill)
// handle one index; block phases (ph_scan_*, ph_narrow, ph_bodies) contain
// __syncthreads and must be called by every thread of the block.  The
// standalone kernels and the fused small-n kernel are thin drivers.
// ===========================================================================

// R1/H1: key + bucket occupancy.  R (Morton key) reads the committed state;
// H (spatial hash, build_hashmap broadphase.py:89-130) reads the layout.
__device__ __forceinline__ void ph_count(const Dev& D, Ctl* ctl, int i, bool morton) {
  const float4 p = morton ? D.X[ctl->cur][i] : layout(D, ctl).x[i];
  if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z)) {
    raise_err(ctl, GG_EPOSITIONS);
    return;
  }
  const long long c0 = cell_coord(p.x, D.two_r);
  const long long c1 = cell_coord(p.y, D.two_r);
  const long long c2 = cell_coord(p.z, D.two_r);
  const uint32_t h = morton ? morton_key(c0, c1, c2, D.mmask) : hash_cell(c0, c1, c2, D.H);
  D.key[i] = h;
  D.arrive[i] = atomicAdd(&D.cnt[h], 1u);
}

// exclusive scan of cnt[0..n_h) -> start[0..n_h)   (start[n_h] = n fixed)
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
    if (lane < nw) sm[lane] = s;
  }
  __syncthreads();
  const uint32_t warp_off = wid ? sm[wid - 1] : 0u;
  *total = sm[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_off + x - v;
}

// 8 consecutive counts of a tile (kScanTile = 8 x kBlock)
__device__ __forceinline__ void load8(const Dev& D, long long base, uint32_t v[8]) {
  if (base + 8 <= D.H.n_h) {
    const uint4 a = *reinterpret_cast<const uint4*>(D.cnt + base);
    const uint4 b = *reinterpret_cast<const uint4*>(D.cnt + base + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (base + e < D.H.n_h) ? D.cnt[base + e] : 0u;
  }
}

__device__ __forceinline__ void ph_scan_tile(const Dev& D, int t, uint32_t* sm) {
  uint32_t v[8];
  load8(D, static_cast<long long>(t) * kScanTile + threadIdx.x * 8, v);
  uint32_t s = v[0] + v[1] + v[2] + v[3] + v[4] + v[5] + v[6] + v[7];
  uint32_t total;
  (void)block_excl_scan_u32(s, sm, &total);
  if (threadIdx.x == 0) D.tile[t] = total;
}

__device__ __forceinline__ void ph_scan_top(const Dev& D, int ntiles, uint32_t* sm) {
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

// Tile t's exclusive bucket offsets.  `tile_counts`: tile[] still holds the
// per-tile totals (few tiles: each block sums its predecessors); otherwise
// k_scan_top has already turned tile[] into exclusive offsets.
__device__ __forceinline__ void ph_scan_apply(const Dev& D, int t, uint32_t* sm, bool tile_counts) {
  const long long base = static_cast<long long>(t) * kScanTile + threadIdx.x * 8;
  uint32_t prefix;
  if (tile_counts) {
    uint32_t part = 0;
    for (int q = threadIdx.x; q < t; q += blockDim.x) part += D.tile[q];
    uint32_t total;
    (void)block_excl_scan_u32(part, sm, &total);
    prefix = total;
  } else {
    prefix = D.tile[t];
  }
  uint32_t v[8];
  load8(D, base, v);
  const uint32_t s = v[0] + v[1] + v[2] + v[3] + v[4] + v[5] + v[6] + v[7];
  uint32_t total;
  uint32_t run = block_excl_scan_u32(s, sm, &total) + prefix;
  uint32_t o[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    o[e] = run;
    run += v[e];
  }
  if (base + 8 <= D.H.n_h) {
    *reinterpret_cast<uint4*>(D.start + base) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4*>(D.start + base + 4) = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
    for (int e = 0; e < 8; ++e)
      if (base + e < D.H.n_h) D.start[base + e] = o[e];
  }
}

// R3/H3: counting-sort scatter (arrival order inside a bucket)
__device__ __forceinline__ void ph_scatter(const Dev& D, int i) {
  D.tmp[D.start[D.key[i]] + D.arrive[i]] = i;
}

// Once the scan has consumed them, bucket and tile counts are zeroed in the
// scatter phase, so the next pass starts from zero without its own pass.
__device__ __forceinline__ void ph_zero_counts(const Dev& D, long long t0, long long G) {
  uint4* c4 = reinterpret_cast<uint4*>(D.cnt);
  const long long n4 = D.H.n_h / 4;
  for (long long i = t0; i < n4; i += G) c4[i] = make_uint4(0u, 0u, 0u, 0u);
  for (long long i = 4 * n4 + t0; i < D.H.n_h; i += G) D.cnt[i] = 0u;
  const long long nt = (D.H.n_h + kScanTile - 1) / kScanTile;
  for (long long i = t0; i < nt; i += G) D.tile[i] = 0u;
}

// rank of a member inside its bucket by user id (the stable tie order)
__device__ __forceinline__ uint32_t rank_in_bucket(const Dev& D, const int* uid,
                                                   uint32_t s, uint32_t e, int my_uid) {
  uint32_t rank = 0;
  for (uint32_t m = s; m < e; ++m) rank += (uid[D.tmp[m]] < my_uid) ? 1u : 0u;
  return rank;
}

// R4: re-sort the committed state into Morton order (deterministic: ties by uid)
__device__ __forceinline__ void ph_resort(const Dev& D, const Ctl* ctl, int k) {
  const int cur = ctl->cur, u = ctl->ucur;
  const int* uid_in = D.UID[u];
  const int p = D.tmp[k];
  const int uid = uid_in[p];
  const uint32_t h = D.key[p];
  const uint32_t s = D.start[h];
  const uint32_t f = s + rank_in_bucket(D, uid_in, s, D.start[h + 1], uid);
  D.UID[u ^ 1][f] = uid;
  D.Xs[f] = D.X[cur][p];
  D.V0[f] = D.V[cur][p];
}

// H4: fill the bucket-ordered candidate array Xh = (x, y, z, physical index)
__device__ __forceinline__ void ph_fill(const Dev& D, const Ctl* ctl, int k) {
  const Layout L = layout(D, ctl);
  const int p = D.tmp[k];
  const uint32_t h = D.key[p];
  const uint32_t s = D.start[h], e = D.start[h + 1];
  const uint32_t f = (e - s == 1) ? s : s + rank_in_bucket(D, L.uid, s, e, L.uid[p]);
  const float4 x = L.x[p];
  D.Xh[f] = make_float4(x.x, x.y, x.z, __int_as_float(p));
}

// ---------------------------------------------------------------------------
// K5 narrowphase helpers
// ---------------------------------------------------------------------------
// Can two of the 27 neighbour cells share a bucket?  For power-of-two tables
// decided exactly from the per-axis hash terms (63 XOR tests).
__device__ __forceinline__ bool may_alias(const uint32_t tx[3], const uint32_t ty[3],
                                          const uint32_t tz[3], uint32_t mask) {
  const uint32_t ax[4] = {0u, tx[0] ^ tx[1], tx[1] ^ tx[2], tx[0] ^ tx[2]};
  const uint32_t ay[4] = {0u, ty[0] ^ ty[1], ty[1] ^ ty[2], ty[0] ^ ty[2]};
  const uint32_t az[4] = {0u, tz[0] ^ tz[1], tz[1] ^ tz[2], tz[0] ^ tz[2]};
  bool hit = false;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i | j | k) hit |= ((ax[i] ^ ay[j] ^ az[k]) & mask) == 0u;
  return hit;
}

__device__ __forceinline__ uint32_t nb_hash(const Dev& D, int o, long long c0, long long c1,
                                            long long c2, const uint32_t tx[3], const uint32_t ty[3],
                                            const uint32_t tz[3]) {
  const int ox = o / 9, oy = (o / 3) % 3, oz = o % 3;
  if (D.H.pow2) return (tx[ox] ^ ty[oy] ^ tz[oz]) & D.H.mask;
  return hash_cell64(c0 + ox - 1, c1 + oy - 1, c2 + oz - 1, D.H.n_h);
}

// The exact pp test on one candidate (contact.py:257-272): float64 from
// float32-representable inputs in the reference's operation order.
__device__ __forceinline__ void pp_candidate(const Dev& D, int k, double px, double py, double pz,
                                             float4 qf, int q, int& cnt, unsigned long long& n_coinc,
                                             double& max_psi) {
  const double dx = __dsub_rn(px, static_cast<double>(qf.x));
  const double dy = __dsub_rn(py, static_cast<double>(qf.y));
  const double dz = __dsub_rn(pz, static_cast<double>(qf.z));
  // einsum("ij,ij->i") on the reference host: (dx^2 + dz^2) + dy^2
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
  if (!(d2 >= D.coinc_d2)) {
    ++n_coinc;
    return;
  }
  if (d2 < D.contact_d2) {
    const double dist = __dsqrt_rn(d2);
    const double psi = __dsub_rn(D.two_r, dist);
    if (cnt < D.K) {
      const long long sl = static_cast<long long>(cnt) * D.n + k;
      D.cgeo[sl] = make_float4(static_cast<float>(__ddiv_rn(dx, dist)),
                               static_cast<float>(__ddiv_rn(dy, dist)),
                               static_cast<float>(__ddiv_rn(dz, dist)), static_cast<float>(psi));
      D.coth[sl] = q;
    }
    ++cnt;
    max_psi = nmax(max_psi, psi);
  }
}

struct NarrowSmem {
  uint32_t beg[27][kBlock];
  uint16_t len[27][kBlock];  // bucket sizes are < 2^16
  double d[32];
  unsigned long long u[32];
};

// Particle k = base + threadIdx.x.  Phase 1: the 27 neighbour-bucket bounds,
// loaded in three batches of 9 independent loads; empty and duplicate buckets
// are dropped and the rest compacted into a per-thread list in shared memory.
// Phase 2: ONE flat loop over the concatenated candidates (lanes stay
// converged; the next candidate is prefetched while the current one is
// tested), a conservative float32 reject, then the exact float64 test.
__device__ __forceinline__ void ph_narrow(const Dev& D, Ctl* ctl, int base, NarrowSmem& sm) {
  // plain (coherent) loads: in the fused kernel these buffers are written
  // earlier in the same launch, so the read-only (.nc) path is not allowed
  const float4* LX = layout(D, ctl).x;
  const float4* Xh = D.Xh;
  const uint32_t* start = D.start;
  const int tid = threadIdx.x;
  const int k = base + tid;
  unsigned long long n_pp = 0, n_cand = 0, n_coinc = 0;
  double max_psi = 0.0;
  if (k < D.n) {
    const float4 pf = LX[k];
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
    const bool dedup = !D.H.pow2 || may_alias(tx, ty, tz, D.H.mask);
    int nb = 0;
    uint32_t total = 0;
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      uint32_t hb[9], sb[9], eb[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        hb[j] = nb_hash(D, g * 9 + j, c0, c1, c2, tx, ty, tz);
        sb[j] = start[hb[j]];
        eb[j] = start[hb[j] + 1];
      }
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        bool keep = eb[j] > sb[j];
        if (keep && dedup) {
          for (int q = 0; q < g * 9 + j; ++q) keep &= nb_hash(D, q, c0, c1, c2, tx, ty, tz) != hb[j];
        }
        if (keep) {
          sm.beg[nb][tid] = sb[j];
          sm.len[nb][tid] = static_cast<uint16_t>(eb[j] - sb[j]);
          total += eb[j] - sb[j];
          ++nb;
        }
      }
    }
    n_cand = total - 1;  // minus the self pair (one per particle, broadphase.py:441-447)
    int cnt = 0;
    int b = 0;
    uint32_t m = sm.beg[0][tid];
    uint32_t left = sm.len[0][tid];
    constexpr int kDepth = 4;  // candidates in flight per thread
    for (uint32_t i = 0; i < total; i += kDepth) {
      uint32_t mi[kDepth];
#pragma unroll
      for (int u = 0; u < kDepth; ++u) {
        mi[u] = m;
        if (i + u + 1 < total) {  // advance the cursor to the next candidate
          ++m;
          if (--left == 0) {
            ++b;
            m = sm.beg[b][tid];
            left = sm.len[b][tid];
          }
        }
      }
      float4 qv[kDepth];
#pragma unroll
      for (int u = 0; u < kDepth; ++u)
        if (i + u < total) qv[u] = Xh[mi[u]];
#pragma unroll
      for (int u = 0; u < kDepth; ++u) {
        if (i + u >= total) break;
        const float4 qf = qv[u];
        const int q = __float_as_int(qf.w);
        if (q == k) continue;
        // float32 pre-filter, conservative by a 1e-5 relative margin (the
        // float32 estimate is within ~4e-7 relative of the exact square)
        const float fx = pf.x - qf.x, fy = pf.y - qf.y, fz = pf.z - qf.z;
        if (fx * fx + fy * fy + fz * fz <= D.reject_d2f)
          pp_candidate(D, k, px, py, pz, qf, q, cnt, n_coinc, max_psi);
      }
    }
    n_pp = cnt;
    D.ccount[k] = cnt < D.K ? cnt : D.K;
    if (cnt > D.K) {
      atomicMax(&ctl->cap_needed, cnt);
      raise_err(ctl, GG_ECAPACITY);
    }
  }
  unsigned long long t;
  t = block_sum_u64(n_pp, sm.u);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_pp, t);
  t = block_sum_u64(n_cand, sm.u);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_cand, t);
  t = block_sum_u64(n_coinc, sm.u);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_coinc, t);
  const double mp = block_reduce<1>(max_psi, sm.d);
  if (threadIdx.x == 0 && mp > 0.0) atomicMax(&D.acc->max_psi_bits, dbits(mp));
}

// K6: particle-body contacts (contact.py:274-286): world-AABB prefilter
// (`_near_body`, contact.py:187-203) then the SDF penetration test
// (sdf.py:472-512); appended after the particle's pp slots, bodies in index
// order, like the reference's per-body concatenation.
__device__ __forceinline__ void ph_bodies(const Dev& D, Ctl* ctl, int base, double* smd,
                                          unsigned long long* smu) {
  const gg_body* bodies = D.bodies + static_cast<long long>(ctl->step) * D.nb;
  const int k = base + threadIdx.x;
  unsigned long long n_body = 0, n_deg = 0;
  double max_psi = 0.0;
  if (k < D.n) {
    const float4 pf = layout(D, ctl).x[k];
    const double px = pf.x, py = pf.y, pz = pf.z;
    int cnt = D.ccount[k];
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
        if (cnt < D.K) {
          const long long sl = static_cast<long long>(cnt) * D.n + k;
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
    if (n_body) {
      D.ccount[k] = cnt < D.K ? cnt : D.K;
      if (cnt > D.K) {
        atomicMax(&ctl->cap_needed, cnt);
        raise_err(ctl, GG_ECAPACITY);
      }
    }
  }
  unsigned long long t;
  t = block_sum_u64(n_body, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_body, t);
  t = block_sum_u64(n_deg, smu);
  if (threadIdx.x == 0 && t) atomicAdd(&D.acc->n_deg, t);
  const double mp = block_reduce<1>(max_psi, smd);
  if (threadIdx.x == 0 && mp > 0.0) atomicMax(&D.acc->max_psi_bits, dbits(mp));
}

// ---------------------------------------------------------------------------
// K7: projected-Jacobi sweep (solve_contacts_pja, contact.py:463-501).
// w = v + dv is the predicted velocity; every contact of owner i reads w of
// the previous sweep for both i and j (Jacobi), writes only w_i (no atomics).
// The tangential impulse is -(u - (u.e1) e1), identical to e2*b2 + e3*b3 for
// the orthonormal frame of contact.py:47-56, so the frame is never built.
// ---------------------------------------------------------------------------
// Body reaction momentum is summed per block in shared memory (exact int64
// fixed-point adds: order-independent) and flushed to the global per-body
// accumulators once per block per kernel — a per-contact global atomic on
// the same three addresses per body serialises every body contact of the
// floor at the L2 and sits on the critical path of every sweep.
constexpr int kSmemBodies = 16;

struct SweepAcc {
  double maxviol, minb1;
  unsigned long long* sbm;  // shared [kSmemBodies][3]
};

__device__ __forceinline__ void sweep_acc_init(SweepAcc& A, unsigned long long* sbm) {
  A.maxviol = 0.0;
  A.minb1 = __longlong_as_double(0x7ff0000000000000ll);
  A.sbm = sbm;
  for (int i = threadIdx.x; i < kSmemBodies * 3; i += blockDim.x) sbm[i] = 0ull;
  __syncthreads();
}

// per block: diagnostics (block max/min, one atomic each) + body momentum
// (one atomic per non-zero component).  Called by every thread.
__device__ __forceinline__ void sweep_acc_flush(const Dev& D, const SweepAcc& A, double* smd) {
  const double mv = block_reduce<1>(A.maxviol, smd);
  if (threadIdx.x == 0 && mv > 0.0) atomicMax(&D.acc->max_viol_bits, dbits(mv));
  const double mb = block_reduce<2>(A.minb1, smd);
  if (threadIdx.x == 0 && mb == mb && mb < __longlong_as_double(0x7ff0000000000000ll))
    atomicMin(&D.acc->min_b1_bits, dbits(mb));
  __syncthreads();
  const int m = (D.nb < kSmemBodies ? D.nb : kSmemBodies) * 3;
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    if (A.sbm[i]) atomicAdd(&D.bm_fix[i], A.sbm[i]);
}

__device__ __forceinline__ void contact_impulse(const Dev& D, double wx, double wy, double wz,
                                                float4 g, int j, float4 q, double& ax, double& ay,
                                                double& az, SweepAcc& A) {
  const double eff = (j >= 0) ? 0.5 : 1.0;  // both partners mobile (contact.py:457-460)
  const double e1x = g.x, e1y = g.y, e1z = g.z;
  const double ux = (wx - D.gamma * q.x) + D.gdt0;
  const double uy = (wy - D.gamma * q.y) + D.gdt1;
  const double uz = (wz - D.gamma * q.z) + D.gdt2;
  const double un = ux * e1x + uy * e1y + uz * e1z;
  const double b1 = nmax(D.bias_coef * (double)g.w - un, 0.0);
  double btx = un * e1x - ux, bty = un * e1y - uy, btz = un * e1z - uz;
  const double tn2 = btx * btx + bty * bty + btz * btz;
  const double lim = D.mu * b1;
  if (tn2 > lim * lim) {  // sliding: project onto the Coulomb cone
    const double tn = sqrt(tn2);
    const double sc = lim / fmax(tn, 1e-300);
    btx *= sc;
    bty *= sc;
    btz *= sc;
    A.maxviol = nmax(A.maxviol, tn * sc - lim);
  }
  const double ix = (e1x * b1 + btx) * eff;
  const double iy = (e1y * b1 + bty) * eff;
  const double iz = (e1z * b1 + btz) * eff;
  ax += ix;
  ay += iy;
  az += iz;
  A.minb1 = nmin(A.minb1, b1);
  if (j < 0) {  // reaction momentum on the body (contact.py:489-495)
    const int b = -j - 1;
    unsigned long long* bm = (b < kSmemBodies) ? A.sbm + 3 * b : D.bm_fix + 3 * b;
    atomicAdd(bm + 0, to_fix(-D.mass * ix));
    atomicAdd(bm + 1, to_fix(-D.mass * iy));
    atomicAdd(bm + 2, to_fix(-D.mass * iz));
  }
}

__device__ __forceinline__ void sweep_particle(const Dev& D, int k, const float4* Win, float4* Wout,
                                               SweepAcc& A) {
  // slot 0 is fetched together with the count and w_k (one round trip)
  const int c = D.ccount[k];
  const float4 wf = Win[k];
  const float4 g0 = D.cgeo[k];
  const int j0 = D.coth[k];
  const double wx = wf.x, wy = wf.y, wz = wf.z;
  double ax = 0.0, ay = 0.0, az = 0.0;
  if (c > 0) {
    const float4 q0 = (j0 >= 0) ? Win[j0] : D.cvb[k];
    contact_impulse(D, wx, wy, wz, g0, j0, q0, ax, ay, az, A);
    const int n = D.n;
    for (int sl = 1; sl < c; ++sl) {
      const int idx = sl * n + k;
      const float4 g = D.cgeo[idx];
      const int j = D.coth[idx];
      const float4 q = (j >= 0) ? Win[j] : D.cvb[idx];
      contact_impulse(D, wx, wy, wz, g, j, q, ax, ay, az, A);
    }
  }
  Wout[k] = make_float4(static_cast<float>(wx + ax), static_cast<float>(wy + ay),
                        static_cast<float>(wz + az), 0.f);
}

// Register-resident variant for the fused kernel (one particle per thread):
// the first kRegSlots contacts and the particle's own w are loaded once and
// kept across all sweeps; each sweep issues its neighbour gathers together.
// Arithmetic and accumulation order are exactly those of sweep_particle.
constexpr int kRegSlots = 4;
struct RegContacts {
  int c;
  float4 g[kRegSlots];
  int j[kRegSlots];
  float4 qb[kRegSlots];
  float wx, wy, wz;

  __device__ __forceinline__ void load(const Dev& D, int k, float4 w0) {
    c = D.ccount[k];
    const int n = D.n;
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s) {
      j[s] = 0;
      if (s < c) {
        g[s] = D.cgeo[s * n + k];
        j[s] = D.coth[s * n + k];
        if (j[s] < 0) qb[s] = D.cvb[s * n + k];
      }
    }
    wx = w0.x;
    wy = w0.y;
    wz = w0.z;
  }

  __device__ __forceinline__ void sweep(const Dev& D, int k, const float4* Win, float4* Wout,
                                        SweepAcc& A) {
    float4 q[kRegSlots];
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s)
      if (s < c) q[s] = (j[s] >= 0) ? Win[j[s]] : qb[s];
    double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s)
      if (s < c) contact_impulse(D, wx, wy, wz, g[s], j[s], q[s], ax, ay, az, A);
    const int n = D.n;
    for (int s = kRegSlots; s < c; ++s) {
      const int idx = s * n + k;
      const float4 gg = D.cgeo[idx];
      const int jj = D.coth[idx];
      const float4 qq = (jj >= 0) ? Win[jj] : D.cvb[idx];
      contact_impulse(D, wx, wy, wz, gg, jj, qq, ax, ay, az, A);
    }
    const float4 out = make_float4(static_cast<float>(wx + ax), static_cast<float>(wy + ay),
                                   static_cast<float>(wz + az), 0.f);
    Wout[k] = out;
    wx = out.x;
    wy = out.y;
    wz = out.z;
  }
};

// Symplectic Euler (stepper.py:102-106), SolverError check
// (contact.py:503-509), kinetic energy (stepper.py:118); the last block to
// finish reduces the per-block partials in fixed order into the StepReport
// and commits the new state.  Called by every thread of every block.
__device__ __forceinline__ void integrate_and_finish(const Dev& D, Ctl* ctl, int t0, int G,
                                                     double* smd, int* s_last) {
  const int cur = ctl->cur;
  const int step = ctl->step;
  const Layout L = layout(D, ctl);
  const float4* Wf = D.W[(D.S - 1) & 1];
  double ke = 0.0;
  for (int k = t0; k < D.n; k += G) {
    const float4 xo = L.x[k];
    const float4 vo = L.v[k];
    const float4 wf = Wf[k];
    const bool has = D.ccount[k] > 0;
    const double dvx = has ? (double)wf.x - (double)vo.x : 0.0;
    const double dvy = has ? (double)wf.y - (double)vo.y : 0.0;
    const double dvz = has ? (double)wf.z - (double)vo.z : 0.0;
    if (!isfinite(dvx) || !isfinite(dvy) || !isfinite(dvz)) {
      const int slot = atomicAdd(&ctl->n_bad, 1);
      if (slot < kMaxBad) ctl->bad_uid[slot] = L.uid[k];
      raise_err(ctl, GG_ENONFINITE);
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
    ke += __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
  }
  const double r = block_reduce<0>(ke, smd);
  if (threadIdx.x == 0) {
    D.part[blockIdx.x] = r;
    __threadfence();
    *s_last = atomicAdd(&ctl->done_count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!*s_last) return;
  __threadfence();
  double v0 = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v0 += *((volatile double*)&D.part[b]);
  const double ke_tot = block_reduce<0>(v0, smd);
  if (threadIdx.x < D.nb * 3) {
    const long long f =
        static_cast<long long>(*((volatile unsigned long long*)&D.bm_fix[threadIdx.x]));
    D.bm_out[static_cast<long long>(step) * D.nb * 3 + threadIdx.x] = static_cast<double>(f) / kMomScale;
    D.bm_fix[threadIdx.x] = 0ull;
  }
  // every other block has finished (it incremented done_count last), so the
  // barrier words and sweep flags can be reset here for the next launch
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    if (D.bflags) D.bflags[b] = 0u;
  if (threadIdx.x == 0) {
    ctl->done_count = 0;
    ctl->bar_count = 0;
    ctl->bar_gen = 0;
    if (*((volatile int*)&ctl->err)) return;  // an error was raised this step: no commit
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
    a->max_psi_bits = a->max_viol_bits = 0;
    a->min_b1_bits = dbits(__longlong_as_double(0x7ff0000000000000ll));
    ctl->cur = cur ^ 1;
    if (D.resort) ctl->ucur ^= 1;
    ctl->step = step + 1;
  }
}

// ===========================================================================
// Large-n drivers: one kernel per phase, one thread per element.
// ===========================================================================
__global__ void __launch_bounds__(kBlock) k_count(Dev D) {
  Ctl* ctl = D.ctl;
  if (ctl->err) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < D.n) ph_count(D, ctl, i, D.key_morton != 0);
}

__global__ void __launch_bounds__(kBlock) k_scan_tiles(Dev D) {
  __shared__ uint32_t sm[32];
  if (D.ctl->err) return;
  ph_scan_tile(D, blockIdx.x, sm);
}

__global__ void __launch_bounds__(1024) k_scan_top(Dev D, int ntiles) {
  __shared__ uint32_t sm[32];
  if (D.ctl->err) return;
  ph_scan_top(D, ntiles, sm);
}

__global__ void __launch_bounds__(kBlock) k_scan_apply(Dev D) {
  __shared__ uint32_t sm[32];
  if (D.ctl->err) return;
  ph_scan_apply(D, blockIdx.x, sm, false);
}

__global__ void __launch_bounds__(kBlock) k_scatter(Dev D) {
  if (D.ctl->err) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < D.n) ph_scatter(D, i);
  ph_zero_counts(D, i, static_cast<long long>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(kBlock) k_resort(Dev D) {
  if (D.ctl->err) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < D.n) ph_resort(D, D.ctl, k);
}

__global__ void __launch_bounds__(kBlock) k_fill(Dev D) {
  if (D.ctl->err) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < D.n) ph_fill(D, D.ctl, k);
}

__global__ void __launch_bounds__(kBlock, 2) k_narrow(Dev D) {
  __shared__ NarrowSmem sm;
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  ph_narrow(D, ctl, blockIdx.x * blockDim.x, sm);
}

__global__ void __launch_bounds__(kBlock) k_bodies(Dev D) {
  __shared__ double smd[32];
  __shared__ unsigned long long smu[32];
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  ph_bodies(D, ctl, blockIdx.x * blockDim.x, smd, smu);
}

__global__ void __launch_bounds__(kBlock) k_sweep(Dev D, int s) {
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  __shared__ double smd[32];
  const Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const Layout L = layout(D, ctl);
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  SweepAcc A;
  sweep_acc_init(A, sbm);
  if (k < D.n) sweep_particle(D, k, (s == 0) ? L.v : D.W[(s - 1) & 1], D.W[s & 1], A);
  sweep_acc_flush(D, A, smd);
}

__global__ void __launch_bounds__(kBlock) k_finish(Dev D) {
  __shared__ double smd[32];
  __shared__ int s_last;
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  integrate_and_finish(D, ctl, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, smd,
                       &s_last);
}

// ===========================================================================
// Small-n driver: the WHOLE step in one persistent kernel (grid = co-resident
// blocks, cooperative launch), grid barriers between phases instead of
// kernel launches.  Blocks never leave early: after every barrier each block
// re-reads the error flag (all errors raised before a barrier are visible
// after it) and skips work, so every block reaches every barrier.
// ===========================================================================
// optional phase timestamps (block 0, %globaltimer) for the bench breakdown
__device__ __forceinline__ void stamp(const Dev& D, int& idx) {
  if (D.tstamp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    D.tstamp[idx] = t;
  }
  ++idx;
}

__device__ __forceinline__ bool barrier_ok(const Dev& D, Ctl* ctl, unsigned& target, int* s_flag,
                                           int& ts) {
  target += gridDim.x;
  grid_barrier(ctl, target);
  if (threadIdx.x == 0) *s_flag = *((volatile int*)&ctl->err);
  __syncthreads();
  stamp(D, ts);
  return *s_flag == 0;
}

__global__ void __launch_bounds__(kBlock, 2) k_step_fused(Dev D) {
  __shared__ NarrowSmem sm;
  __shared__ uint32_t smu[32];
  __shared__ int s_flag;
  __shared__ int s_last;
  Ctl* ctl = D.ctl;
  int ts = 0;
  stamp(D, ts);
  if (threadIdx.x == 0) s_flag = *((volatile int*)&ctl->err);
  __syncthreads();
  bool ok = s_flag == 0;
  unsigned target = 0;
  const int G = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int ntiles = static_cast<int>((D.H.n_h + kScanTile - 1) / kScanTile);
  // bucket/tile counts are zero on entry (zeroed by the previous scatter)
  for (int pass = D.resort ? 0 : 1; pass < 2; ++pass) {
    const bool morton = pass == 0;
    if (ok)
      for (int i = t0; i < D.n; i += G) ph_count(D, ctl, i, morton);
    ok = barrier_ok(D, ctl, target, &s_flag, ts);
    if (ok)
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ph_scan_tile(D, t, smu);
    ok = barrier_ok(D, ctl, target, &s_flag, ts);
    if (ok)
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ph_scan_apply(D, t, smu, true);
    ok = barrier_ok(D, ctl, target, &s_flag, ts);
    if (ok) {
      for (int i = t0; i < D.n; i += G) ph_scatter(D, i);
      ph_zero_counts(D, t0, G);
    }
    ok = barrier_ok(D, ctl, target, &s_flag, ts);
    if (ok) {
      for (int k = t0; k < D.n; k += G) {
        if (morton)
          ph_resort(D, ctl, k);
        else
          ph_fill(D, ctl, k);
      }
    }
    ok = barrier_ok(D, ctl, target, &s_flag, ts);
  }
  // narrowphase + bodies; the sweeps below use the same particle -> thread
  // map, so a particle's contacts are read by the thread that wrote them
  if (ok) {
    for (int base = blockIdx.x * blockDim.x; base < D.n; base += G) {
      ph_narrow(D, ctl, base, sm);
      if (D.nb > 0) ph_bodies(D, ctl, base, sm.d, sm.u);
    }
  }
  stamp(D, ts);
  const Layout L = layout(D, ctl);
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  SweepAcc A;
  sweep_acc_init(A, sbm);
  if (G >= D.n && gridDim.x <= kMaxFusedBlocks) {
    // One particle per thread: its contacts (first kRegSlots) and its own w
    // stay in registers for all sweeps.  Jacobi sweep s of a block only needs
    // sweep s-1 of the blocks that own its particles' contact partners, and
    // (contacts being symmetric) those are also the only blocks that read its
    // w — so instead of a grid barrier a block waits on its neighbour blocks'
    // progress flags (release/acquire), then publishes its own.
    __shared__ unsigned s_nbmask[kMaxFusedBlocks / 32];
    __shared__ int s_nblist[kMaxFusedBlocks];
    __shared__ int s_nnb;
    RegContacts RC;
    RC.c = 0;
    if (ok && t0 < D.n) RC.load(D, t0, L.v[t0]);
    for (int w = threadIdx.x; w < kMaxFusedBlocks / 32; w += blockDim.x) s_nbmask[w] = 0u;
    __syncthreads();
    {
      const int n = D.n;
      const int c = RC.c < D.K ? RC.c : D.K;
      for (int sl = 0; sl < c; ++sl) {
        const int j = sl < kRegSlots ? RC.j[sl] : D.coth[sl * n + t0];
        if (j >= 0) {
          const int b = j / blockDim.x;
          if (b != static_cast<int>(blockIdx.x)) atomicOr(&s_nbmask[b >> 5], 1u << (b & 31));
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int m = 0;
      for (int w = 0; w < (int)((gridDim.x + 31) / 32); ++w) {
        unsigned bits = s_nbmask[w];
        while (bits) {
          const int bit = __ffs(bits) - 1;
          bits &= bits - 1;
          s_nblist[m++] = w * 32 + bit;
        }
      }
      s_nnb = m;
    }
    __syncthreads();
    unsigned* flags = D.bflags;
    for (int s = 0; s < D.S; ++s) {
      if (s > 0) {
        for (int q = threadIdx.x; q < s_nnb; q += blockDim.x) {
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flags + s_nblist[q]) : "memory");
          } while (static_cast<int>(v - static_cast<unsigned>(s)) < 0);
        }
        __syncthreads();
        if (threadIdx.x == 0) __threadfence();  // invalidate stale L1 lines (CCTL.IVALL)
        __syncthreads();
        if (threadIdx.x == 0) s_flag = *((volatile int*)&ctl->err);
        __syncthreads();
        ok = ok && s_flag == 0;
        stamp(D, ts);
      }
      if (ok && t0 < D.n) RC.sweep(D, t0, (s == 0) ? L.v : D.W[(s - 1) & 1], D.W[s & 1], A);
      __syncthreads();
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(s + 1) : "memory");
    }
  } else {
    for (int s = 0; s < D.S; ++s) {
      if (s > 0) ok = barrier_ok(D, ctl, target, &s_flag, ts) && ok;
      if (ok) {
        const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
        float4* Wout = D.W[s & 1];
        for (int k = t0; k < D.n; k += G) sweep_particle(D, k, Win, Wout, A);
      }
    }
  }
  stamp(D, ts);
  sweep_acc_flush(D, A, sm.d);
  integrate_and_finish(D, ctl, t0, G, sm.d, &s_last);
  stamp(D, ts);
}

// Small-n solve only (cooperative): S sweeps with grid barriers + finish.
__global__ void __launch_bounds__(kBlock, 3) k_solve(Dev D) {
  __shared__ double smd[32];
  __shared__ int s_last;
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;  // uniform: err cannot change before the last barrier
  const Layout L = layout(D, ctl);
  const int G = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  SweepAcc A;
  sweep_acc_init(A, sbm);
  for (int s = 0; s < D.S; ++s) {
    if (s > 0) grid_barrier(ctl, gridDim.x * static_cast<unsigned>(s));
    const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
    float4* Wout = D.W[s & 1];
    for (int k = t0; k < D.n; k += G) sweep_particle(D, k, Win, Wout, A);
  }
  sweep_acc_flush(D, A, smd);
  integrate_and_finish(D, ctl, t0, G, smd, &s_last);
}

// ---------------------------------------------------------------------------
// state upload / download helpers (committed layout)
// ---------------------------------------------------------------------------
__global__ void k_load_f64(Dev D, const double* __restrict__ x, const double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  const int cur = D.ctl->cur;
  D.X[cur][i] = make_float4(static_cast<float>(x[3 * i]), static_cast<float>(x[3 * i + 1]),
                            static_cast<float>(x[3 * i + 2]), 0.f);
  D.V[cur][i] = make_float4(static_cast<float>(v[3 * i]), static_cast<float>(v[3 * i + 1]),
                            static_cast<float>(v[3 * i + 2]), 0.f);
  D.UID[D.ctl->ucur][i] = i;
}

__global__ void k_store_f64(Dev D, double* __restrict__ x, double* __restrict__ v) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = D.ctl->cur;
  const int u = D.UID[D.ctl->ucur][k];
  const float4 p = D.X[cur][k], q = D.V[cur][k];
  x[3 * u] = p.x; x[3 * u + 1] = p.y; x[3 * u + 2] = p.z;
  v[3 * u] = q.x; v[3 * u + 1] = q.y; v[3 * u + 2] = q.z;
}

__global__ void k_load_f4(Dev D, const float4* __restrict__ x, const float4* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  const int cur = D.ctl->cur;
  float4 a = x[i], b = v[i];
  a.w = 0.f;
  b.w = 0.f;
  D.X[cur][i] = a;
  D.V[cur][i] = b;
  D.UID[D.ctl->ucur][i] = i;
}

__global__ void k_store_f4(Dev D, float4* __restrict__ x, float4* __restrict__ v) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = D.ctl->cur;
  const int u = D.UID[D.ctl->ucur][k];
  x[u] = D.X[cur][k];
  v[u] = D.V[cur][k];
}

// cells + hashes of the committed state, user order (parity tap)
__global__ void k_tap_cells(Dev D, long long* __restrict__ cells, long long* __restrict__ hashes) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const int cur = D.ctl->cur;
  const int u = D.UID[D.ctl->ucur][k];
  const float4 p = D.X[cur][k];
  const long long c0 = cell_coord(p.x, D.two_r);
  const long long c1 = cell_coord(p.y, D.two_r);
  const long long c2 = cell_coord(p.z, D.two_r);
  cells[3 * u] = c0; cells[3 * u + 1] = c1; cells[3 * u + 2] = c2;
  hashes[u] = hash_cell(c0, c1, c2, D.H);
}

// bucket order as user ids (the stable argsort tap)
__global__ void k_tap_order(Dev D, long long* __restrict__ order) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  order[k] = D.UID[D.ctl->ucur][__float_as_int(D.Xh[k].w)];
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
