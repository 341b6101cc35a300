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

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gg_device.cuh"

namespace gg {

constexpr int kBlock = 256;
constexpr int GG_EBUCKET = 6;  // device-internal: a bucket too long for the contact kernel's lists
constexpr int kScanTile = 2048;  // elements per scan tile (256 thr x 8)
constexpr int kMaxBad = 32;
constexpr int kMaxFusedBlocks = 1024;  // neighbour-flag sweeps: block-set bitmask size

struct Ctl {
  int cur;         // committed state buffer
  int ucur;        // committed uid buffer
  // bar_count and err share one aligned 8-byte word: the grid barrier's
  // final 64-bit acquire load returns the error flag with the arrival count
  unsigned bar_count;  // grid barrier arrivals (monotonic within a launch, reset per launch)
  int err;         // first error code (0 = none)
  int step;        // steps committed in this batch
  int err_step;    // batch-relative step of the error
  int cap_needed;  // largest per-owner contact count seen (capacity hint)
  int n_bad;       // non-finite particles recorded
  unsigned done_count; // last-block-done counter of the solve kernel
  unsigned bar_gen;    // (unused; reset with bar_count)
  unsigned long long ccursor;  // contact records allocated this step (warp allocator)
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

#ifndef GG_FIXED_SLOTS
#define GG_FIXED_SLOTS 1
#endif
constexpr int kFixedSlots = GG_FIXED_SLOTS;  // records per particle at fixed indices (1 or 2)

struct Dev {
  int n, K, nb, S, nblocks;
  int resort;     // this graph re-sorts the physical order first
  int fused_stop; // k_step_fused ends after the contacts (the cluster kernel solves)
  int sweep_barrier;  // fused sweeps: 1 grid barrier per sweep, 0 neighbour-block flags
  int env_kernel;     // E > 1: per-env reports + body momentum written by k_env_reports
  // PipelineMode (stepper.py:34-37, 74-98): 0 TWO_LOOPS_SPLIT (records for
  // contacts only), 1 TWO_LOOPS_FUSED (a record for every candidate, masked:
  // null if not colliding), 2 ONE_LOOP (no records used: every sweep repeats
  // the collision test over the candidates).  Same results in all three.
  int pipeline;
  int key_morton; // counting-sort key of the current pass (R: 1, H: 0)
  // Independent environments (segments).  E == 1 is a single bed.  With
  // E > 1 env e owns particles [e*ne, (e+1)*ne) of the physical order and
  // buckets [e*n_h, (e+1)*n_h) of the index (its own table, the reference's
  // per-scene hash): every sort key is env-major, so the physical order stays
  // env-contiguous and no candidate ever crosses an env boundary.
  int E, ne;
  // Slab mode (one bed over several GPUs): particles
  // [0, n_own) are owned, [n_own, n) are ghosts received from the
  // neighbouring slabs — candidates for the owned particles, but they own no
  // contacts, are not swept (their w arrives by halo exchange) and are not
  // integrated.  n_own == n otherwise.
  int n_own;
  // Slab steps replayed as a CUDA graph: the particle counts change on the
  // device every step (migration, ghosts), so kernels take them from dn
  // ({n, n_own}) and grids are sized for the capacity.  nullptr otherwise.
  const int* dn;
  long long nh_tot;  // E * n_h: length of cnt / start
  HashCfg H;         // the per-env table (n_h buckets)
  uint32_t mmask;  // Morton key mask (power of two <= n_h, minus one)
  uint32_t mspan;  // mmask + 1: Morton key range per env
  // Morton window: the key of cell c is built from (c - mlo) >> msh per axis,
  // so the bulk of the bed spans at most the key's bits per axis and the
  // low-bit key does not wrap (wrapping interleaves cells 2^b apart and
  // breaks the locality of the physical order).  Set by the host from the
  // uploaded state; 0 / 0 = the plain low-bit key.
  int mlo[3], msh[3];
  int mbits;   // bits per axis of the curve key: 3 * mbits <= log2(mspan)
  int mclamp;  // 1: cells outside the window clamp to its faces (else wrap)
  unsigned long long* ke_fix;  // [E] fixed-point sum |v|^2 (E > 1)
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
  float4* cgeo;     // contact records [cap_tot]: (e1.xyz, psi)
  int* coth;        // partner: physical index, or -(body + 1)
  float4* cvb;      // body surface velocity (body records)
  int2* cinfo;      // per particle {CSR offset of its record 1, record count}
  int xh_pad;       // Xh's allocated length: Xh[xh_pad .. xh_pad + kXhPad) is far padding
  int* bad;         // [n] uid + 1 of a particle whose correction was non-finite (0: fine)
  long long cap_tot;  // record capacity
  // Records 0 .. kFixedSlots-1 of particle k live at fixed indices i * n + k
  // (slot-major columns, coalesced); records kFixedSlots.. are warp-contiguous
  // CSR entries allocated from nrec0 = kFixedSlots * n on.  A sweep fetches a
  // particle's first contacts together with its cinfo instead of after it.
  long long nrec0;
  long long wcap;  // CSR records per warp region (32 x (K - kFixedSlots))
  // k_solve_staged: particles per block and contact records staged in each
  // block's shared memory (the rest are read from global memory)
  int stage_pb, stage_cap;
  long long stage_smem;             // dynamic shared memory of a k_solve_staged block
  unsigned long long* stage_seg;    // [grid] work of the fixed segments (k_solve_staged plan)
  const gg_body* bodies;  // [batch][nb]
  const DevGrid* grids;
  const double* gvals;
  Acc* acc;
  unsigned long long* tstamp;  // optional phase timestamps of the fused kernel (64)
  unsigned* bflags;  // [fused grid] per-block sweep progress (fused kernel)
  double* part;     // [nblocks_solve] per-block kinetic-energy partials
  double* wpart;    // [n / 32] per-warp kinetic-energy partials (last sweep integrates)
  unsigned* gcnt;   // [n / 256] warps of a 256-particle group done (reset by the last)
  unsigned long long* bm_fix;  // [nb][3] fixed-point body momentum of the step
  gg_report* reports;
  double* bm_out;  // [batch][nb][3]
  Ctl* ctl;
};


// live particle counts: the device's (graph-replayed slab step) or the Dev's
// (DC: the kernel instantiation replayed in the slab graph; the others read
// the by-value Dev and pay nothing for it)
template <bool DC>
__device__ __forceinline__ int live_n(const Dev& D) { return DC ? __ldcg(D.dn) : D.n; }
template <bool DC>
__device__ __forceinline__ int live_own(const Dev& D) { return DC ? __ldcg(D.dn + 1) : D.n_own; }
// the slab kernels shared by the graph and the per-call paths decide at run time
__device__ __forceinline__ int live_n_rt(const Dev& D) { return D.dn ? __ldcg(D.dn) : D.n; }
__device__ __forceinline__ int live_own_rt(const Dev& D) { return D.dn ? __ldcg(D.dn + 1) : D.n_own; }

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
// Max / min over a warp of non-negative doubles held as bit patterns (for
// x >= +0.0 the IEEE order is the unsigned order of the bits): two 32-bit
// REDUX reductions instead of five float64 shuffle + compare rounds.
__device__ __forceinline__ unsigned long long warp_umax64(unsigned long long v) {
  const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(v >> 32));
  const unsigned lo =
      __reduce_max_sync(0xffffffffu, static_cast<unsigned>(v >> 32) == hi ? static_cast<unsigned>(v) : 0u);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}
__device__ __forceinline__ unsigned long long warp_umin64(unsigned long long v) {
  const unsigned hi = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(v >> 32));
  const unsigned lo = __reduce_min_sync(
      0xffffffffu, static_cast<unsigned>(v >> 32) == hi ? static_cast<unsigned>(v) : 0xffffffffu);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;

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

// ---------------------------------------------------------------------------
// Per-env accumulation.  E == 1: fixed-order block reduction, one atomic per
// block (the single-bed path).  E > 1: a warp whose lanes all belong to one
// env reduces and issues one atomic; a warp straddling an env boundary (at
// most one per env) issues per-lane atomics.  Integer adds and max/min on
// the bit patterns of non-negative doubles are order-independent, so the
// result is deterministic either way.  Called by every thread of the block.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int env_of(const Dev& D, int k) {
  if (D.E == 1) return 0;
  const int e = k / D.ne;
  return e < D.E ? e : D.E - 1;
}

__device__ __forceinline__ bool warp_env_uniform(int env, int* e0) {
  *e0 = __shfl_sync(0xffffffffu, env, 0);
  return __all_sync(0xffffffffu, env == *e0);
}

// field: byte offset of an unsigned long long member of Acc
__device__ __forceinline__ unsigned long long* acc_field(const Dev& D, int env, size_t off) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(D.acc + env) + off);
}

__device__ __forceinline__ void acc_add(const Dev& D, int env, unsigned long long v, size_t off,
                                        unsigned long long* smu) {
  if (D.E == 1) {
    const unsigned long long t = block_sum_u64(v, smu);
    if (threadIdx.x == 0 && t) atomicAdd(acc_field(D, 0, off), t);
    return;
  }
  int e0;
  if (warp_env_uniform(env, &e0)) {
    const unsigned long long t = warp_sum(v);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(acc_field(D, e0, off), t);
  } else if (v) {
    atomicAdd(acc_field(D, env, off), v);
  }
}

// kOp 1: max of non-negative doubles, 2: min (NaN and +inf are ignored)
template <int kOp>
__device__ __forceinline__ void acc_ext(const Dev& D, int env, double v, size_t off, double* smd) {
  double t;
  int tgt;
  bool issue;
  if (D.E == 1) {
    t = block_reduce<kOp>(v, smd);
    tgt = 0;
    issue = threadIdx.x == 0;
  } else {
    int e0;
    if (warp_env_uniform(env, &e0)) {
      t = kOp == 1 ? warp_max(v) : warp_min(v);
      tgt = e0;
      issue = (threadIdx.x & 31) == 0;
    } else {
      t = v;
      tgt = env;
      issue = true;
    }
  }
  if (!issue) return;
  if (kOp == 1) {
    if (t > 0.0) atomicMax(acc_field(D, tgt, off), dbits(t));
  } else {
    if (t == t && t < __longlong_as_double(0x7ff0000000000000ll)) atomicMin(acc_field(D, tgt, off), dbits(t));
  }
}

#define GG_ACC(f) offsetof(Acc, f)

// block-uniform early exit: every kernel that syncs reads err through smem
__device__ __forceinline__ bool block_should_exit(const Ctl* ctl) {
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = *((volatile const int*)&ctl->err);
  __syncthreads();
  return s_err != 0;
}

// Grid-wide barrier for the cooperative kernel (all blocks co-resident).
// One release-add per block on a counter that only grows during a launch
// (zeroed before the launch); thread 0 polls the counter itself with acquire
// loads until it reaches the barrier's target (nblocks x barrier ordinal).
// The acquire load is LD.STRONG.GPU + CCTL.IVALL: it also invalidates this
// SM's L1, so no block reads a line cached before other SMs rewrote it.
// (Measured on B200, 148-296 blocks: 1.1 us per barrier; a separate
// generation word 1.8 us, plus a __threadfence 2.0 us — tools/microbench_sync.cu.)
// Returns ctl->err as seen after the barrier (every error is raised before
// its block arrives, i.e. before a release the final acquire synchronises
// with, and err is read by the same 64-bit load at the L2).
#ifndef GG_BAR_SLEEP
#define GG_BAR_SLEEP 0
#endif
__device__ __forceinline__ int grid_barrier(Ctl* ctl, unsigned target) {
  __shared__ int s_err;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned v;
    unsigned long long w;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(&ctl->bar_count) : "memory");
    v += 1;
    // spin with relaxed (L1-bypassing) loads, then ONE acquire load: the
    // L1 invalidation happens once, not on every poll (an invalidation per
    // poll also evicts the lines the other block on this SM is working on)
    while (static_cast<int>(v - target) < 0) {
#if GG_BAR_SLEEP
      __nanosleep(GG_BAR_SLEEP);
#endif
      asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&ctl->bar_count) : "memory");
    }
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(w) : "l"(&ctl->bar_count) : "memory");
    s_err = static_cast<int>(w >> 32);
  }
  __syncthreads();
  return s_err;
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
__device__ __forceinline__ void acc_reset(Acc* a) {
  a->n_pp = a->n_cand = a->n_body = a->n_coinc = a->n_deg = 0;
  a->max_psi_bits = a->max_viol_bits = 0;
  a->min_b1_bits = dbits(__longlong_as_double(0x7ff0000000000000ll));
}

__global__ void k_batch_begin(Dev D) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int G = gridDim.x * blockDim.x;
  if (t == 0) {
    Ctl* c = D.ctl;
    c->step = 0;
    c->err = 0;
    c->err_step = -1;
    c->cap_needed = 0;
    c->n_bad = 0;
    c->bar_count = 0;
    c->done_count = 0;
    c->bar_gen = 0;
    c->ccursor = static_cast<unsigned long long>(D.nrec0);
  }
  for (int e = t; e < D.E; e += G) {
    acc_reset(D.acc + e);
    if (D.ke_fix) D.ke_fix[e] = 0ull;
  }
  for (int i = t; i < D.E * D.nb * 3; i += G) D.bm_fix[i] = 0ull;
}

// ===========================================================================
// Phases.  Element-wise phases (ph_count, ph_scatter, ph_resort, ph_fill)
// handle one index; block phases (ph_scan_*, ph_contacts) contain
// __syncthreads and must be called by every thread of the block.  The
// standalone kernels and the fused small-n kernel are thin drivers.

// Hilbert key of a cell (the physical-order key, R passes): consecutive keys
// are always face-adjacent cells, so a block of consecutive particles fills
// a compact region — the Morton curve's jumps across its tile boundaries put
// a quarter of 256-particle blocks into boxes of thousands of cells.
// Skilling's transpose form (AxestoTranspose), then the bits interleaved
// axis 0 first.  Cells are taken relative to the window (Dev::mlo, msh).
__device__ __forceinline__ uint32_t curve_key(const Dev& D, long long c0, long long c1, long long c2) {
  const int b = D.mbits;
  if (b <= 0) return 0u;
  const long long top = (1ll << b) - 1;
  long long q[3] = {(c0 - D.mlo[0]) >> D.msh[0], (c1 - D.mlo[1]) >> D.msh[1], (c2 - D.mlo[2]) >> D.msh[2]};
  uint32_t X[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long v = D.mclamp ? (q[a] < 0 ? 0 : (q[a] > top ? top : q[a])) : (q[a] & top);
    X[a] = static_cast<uint32_t>(v);
  }
  const uint32_t M = 1u << (b - 1);
  for (uint32_t Q = M; Q > 1; Q >>= 1) {
    const uint32_t P = Q - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  X[1] ^= X[0];
  X[2] ^= X[1];
  uint32_t t = 0;
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  X[0] ^= t;
  X[1] ^= t;
  X[2] ^= t;
  return (spread3(X[0]) << 2) | (spread3(X[1]) << 1) | spread3(X[2]);
}
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
  const uint32_t env = static_cast<uint32_t>(env_of(D, i));
  const uint32_t h = morton ? env * D.mspan + curve_key(D, c0, c1, c2)
                            : env * static_cast<uint32_t>(D.H.n_h) + hash_cell(c0, c1, c2, D.H);
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
  if (base + 8 <= D.nh_tot) {
    const uint4 a = *reinterpret_cast<const uint4*>(D.cnt + base);
    const uint4 b = *reinterpret_cast<const uint4*>(D.cnt + base + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (base + e < D.nh_tot) ? D.cnt[base + e] : 0u;
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
  if (base + 8 <= D.nh_tot) {
    *reinterpret_cast<uint4*>(D.start + base) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4*>(D.start + base + 4) = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
    for (int e = 0; e < 8; ++e)
      if (base + e < D.nh_tot) D.start[base + e] = o[e];
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
  const long long n4 = D.nh_tot / 4;
  for (long long i = t0; i < n4; i += G) c4[i] = make_uint4(0u, 0u, 0u, 0u);
  for (long long i = 4 * n4 + t0; i < D.nh_tot; i += G) D.cnt[i] = 0u;
  const long long nt = (D.nh_tot + kScanTile - 1) / kScanTile;
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
  // selects instead of array indexing: o is a runtime value in the
  // de-duplication loop, and an indexed array would live in local memory
  if (D.H.pow2) {
    const uint32_t a = ox == 0 ? tx[0] : (ox == 1 ? tx[1] : tx[2]);
    const uint32_t b = oy == 0 ? ty[0] : (oy == 1 ? ty[1] : ty[2]);
    const uint32_t c = oz == 0 ? tz[0] : (oz == 1 ? tz[1] : tz[2]);
    return (a ^ b ^ c) & D.H.mask;
  }
  return hash_cell64(c0 + ox - 1, c1 + oy - 1, c2 + oz - 1, D.H.n_h);
}

// The exact pp distance (contact.py:257-262): float64 from float32-representable
// inputs in the reference's operation order.  einsum("ij,ij->i") on the
// reference host sums (dx^2 + dz^2) + dy^2.
__device__ __forceinline__ double pp_d2(double px, double py, double pz, float4 qf, double& dx,
                                        double& dy, double& dz) {
  dx = __dsub_rn(px, static_cast<double>(qf.x));
  dy = __dsub_rn(py, static_cast<double>(qf.y));
  dz = __dsub_rn(pz, static_cast<double>(qf.z));
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
}

// index of record i of particle k whose CSR records start at off
__device__ __forceinline__ long long ridx(const Dev& D, int k, long long off, int i) {
  return i < kFixedSlots ? static_cast<long long>(i) * D.n + k : off + i - kFixedSlots;
}

// One pp contact record (contact.py:264-272): e1 = d / |d| (j -> i),
// psi = 2r - |d|, partner q (physical index).  Returns psi.
__device__ __forceinline__ double pp_write(const Dev& D, long long dst, double dx, double dy,
                                           double dz, double d2, int q) {
  // |d| and d / |d| from one reciprocal square root (1 ulp; both are stored
  // as float32, and psi's absolute error stays ~1e-17 m)
  const double inv = rsqrt(d2);
  const double dist = d2 * inv;
  const double psi = __dsub_rn(D.two_r, dist);
  D.cgeo[dst] = make_float4(static_cast<float>(dx * inv), static_cast<float>(dy * inv),
                            static_cast<float>(dz * inv), static_cast<float>(psi));
  D.coth[dst] = q;
  return psi;
}

#ifndef GG_PASSCAP
#define GG_PASSCAP 12
#endif
constexpr int kXhPad = 16;  // padding entries after the bucket-ordered candidate copy
#ifndef GG_KDEPTH
#define GG_KDEPTH 6
#endif
#ifndef GG_NARROW_MINB
#define GG_NARROW_MINB 2
#endif
#ifndef GG_PASS_PRED
#define GG_PASS_PRED 1
#endif
#ifndef GG_CULL
#define GG_CULL 1  // large-n contact kernel
#endif
#ifndef GG_FAR_SENTINEL
#define GG_FAR_SENTINEL 1
#endif
#ifndef GG_FUSED_CULL
#define GG_FUSED_CULL 0  // fused small-n kernel (measured slower there: a latency-bound chain)
#endif
constexpr int kPassCap = GG_PASSCAP;  // prefilter passes queued per owner (more: exact inline path)
constexpr int kNullContact = 0x7fffffff;  // partner of a null record (a pass that is no contact)
constexpr int kWarps = kBlock / 32;

#ifndef GG_LEN32
#define GG_LEN32 0
#endif
#if GG_LEN32
using NarrowLen = uint32_t;  // any bucket size (a tiny table may put every particle in one bucket)
constexpr uint32_t kLenSentinel = 0xffffffffu;
#else
using NarrowLen = uint16_t;
constexpr uint32_t kLenSentinel = 0xffffu;
#endif

// B threads per block; Depth candidates in flight per thread; the 27
// neighbour-bucket bounds requested in Groups rounds.  The large-n kernel
// (throughput) and the fused small-n kernel (latency) are tuned apart.
template <int B, int Depth = GG_KDEPTH, int Groups = 3>
struct NarrowSmemT {
  static constexpr int kW = B / 32;
  static constexpr int kDepth = Depth;
  static constexpr int kGroups = Groups;
  static_assert(27 % Groups == 0, "bucket rounds");
  uint32_t beg[28][B];        // compacted non-empty buckets + a sentinel
  NarrowLen len[28][B];       // bucket sizes
  uint32_t pass[kPassCap][B]; // Xh index of every prefilter pass, per owner, in order
  float4 pos[B];              // owner positions
  uint32_t off[kW][32];       // per-warp exclusive offsets of the owners' queue segments
  uint8_t qown[kW][32 * kPassCap];  // per-warp queue: owner lane of each entry
  double d[32];
  unsigned long long u[32];
};
#ifndef GG_FUSED_KDEPTH
#define GG_FUSED_KDEPTH 6
#endif
#ifndef GG_FUSED_GROUPS
#define GG_FUSED_GROUPS 3
#endif
using NarrowSmem = NarrowSmemT<kBlock, GG_FUSED_KDEPTH, GG_FUSED_GROUPS>;  // the fused kernel's
#ifndef GG_NARROW_BLOCK
#define GG_NARROW_BLOCK 256
#endif
constexpr int kNarrowBlock = GG_NARROW_BLOCK;  // k_narrow block size (large-n contact kernel)
#ifndef GG_NARROW_GROUPS
#define GG_NARROW_GROUPS 3
#endif
using NarrowSmemN = NarrowSmemT<kNarrowBlock, GG_KDEPTH, GG_NARROW_GROUPS>;

// Iterate over a thread's concatenated candidate list (its compacted
// neighbour buckets) — the cursor of the flat candidate loop.
struct CandCursor {
  int b;
  uint32_t m, left;
  template <class SM>
  __device__ __forceinline__ void init(const SM& sm, int tid) {
    b = 0;
    m = sm.beg[0][tid];
    left = sm.len[0][tid];
  }
  template <class SM>
  __device__ __forceinline__ uint32_t next(const SM& sm, int tid, bool more) {
    const uint32_t cur = m;
    if (more) {
      ++m;
      if (--left == 0) {
        ++b;
        m = sm.beg[b][tid];
        left = sm.len[b][tid];
      }
    }
    return cur;
  }
};

// Exact inline pass over ALL candidates of one owner (owners with more than
// kPassCap prefilter passes): counts (write == false) or writes records from
// dst on (write == true), in candidate order — the same order the queue gives.
// c_slots: records (= contacts, or every candidate in TWO_LOOPS_FUSED);
// c_pp: contacts.
template <class SM>
__device__ __forceinline__ void scan_exact(const Dev& D, const SM& sm, const float4* cand, int tid,
                                           int k, float4 pf, uint32_t total, bool write, long long off,
                                           int& c_slots, int& c_pp, unsigned long long& n_coinc,
                                           double& max_psi) {
  const double px = pf.x, py = pf.y, pz = pf.z;
  CandCursor cur;
  cur.init(sm, tid);
  c_slots = 0;
  c_pp = 0;
  n_coinc = 0;
  for (uint32_t i = 0; i < total; ++i) {
    const uint32_t mi = cur.next(sm, tid, i + 1 < total);
    const float4 qf = cand[mi];
    const int q = __float_as_int(qf.w);
    if (q == k) continue;
    const float fx = pf.x - qf.x, fy = pf.y - qf.y, fz = pf.z - qf.z;
    const bool all = D.pipeline == 1;  // TWO_LOOPS_FUSED: every candidate gets a record
    if (!all && !(fx * fx + fy * fy + fz * fz <= D.reject_d2f)) continue;
    double dx, dy, dz;
    const double d2 = pp_d2(px, py, pz, qf, dx, dy, dz);
    const bool coi = !(d2 >= D.coinc_d2);
    if (coi) ++n_coinc;
    if (!coi && d2 < D.contact_d2) {
      if (write) max_psi = nmax(max_psi, pp_write(D, ridx(D, k, off, c_slots), dx, dy, dz, d2, q));
      ++c_slots;
      ++c_pp;
    } else if (all) {
      if (write) D.coth[ridx(D, k, off, c_slots)] = kNullContact;
      ++c_slots;  // a masked candidate
    }
  }
}

// K6: particle-body contacts of one particle (contact.py:274-286): world-AABB
// prefilter (`_near_body`, contact.py:187-203), then the SDF penetration test
// (sdf.py:472-512); bodies in index order after the particle's pp records,
// like the reference's per-body concatenation.  write == false only counts.
// Records of particle k at positions first, first + 1, ... (CSR base off).
__device__ __forceinline__ int body_contacts(const Dev& D, const gg_body* bodies, float4 pf,
                                             bool write, int k, long long off, int first,
                                             unsigned long long& n_deg, double& max_psi) {
  const double px = pf.x, py = pf.y, pz = pf.z;
  int c = 0;
  n_deg = 0;
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
      if (write) {
        const long long sl = ridx(D, k, off, first + c);
        const d3 vb = body_surface_velocity(B, px, py, pz, nrm, D.r, psi);
        D.cgeo[sl] = make_float4(static_cast<float>(nrm.x), static_cast<float>(nrm.y),
                                 static_cast<float>(nrm.z), static_cast<float>(psi));
        D.coth[sl] = -(b + 1);
        D.cvb[sl] = make_float4(static_cast<float>(vb.x), static_cast<float>(vb.y),
                                static_cast<float>(vb.z), 0.f);
        max_psi = nmax(max_psi, psi);
      }
      ++c;
    }
    n_deg += deg;
  }
  return c;
}

// The contact phase's six per-step counters in one pass: warp sums (and the
// max of max_psi on its bit pattern, which orders like the value for x >= +0),
// one block barrier, then six threads each reduce one counter over the warps
// and issue its atomic.  E > 1: env-uniform warps issue their own atomics,
// warps straddling two envs per lane.  Called by every thread of the block.
__device__ __forceinline__ void acc_contacts(const Dev& D, int env, unsigned long long n_pp,
                                             unsigned long long n_cand, unsigned long long n_coinc,
                                             unsigned long long n_body, unsigned long long n_deg,
                                             double max_psi) {
  __shared__ unsigned long long s_acc[kWarps][6];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long mp = dbits(max_psi > 0.0 ? max_psi : 0.0);
  // counter f's byte offset in Acc (selects, not an indexed array: f can be
  // a runtime value and an array would live in local memory)
  auto offs = [](int f) -> size_t {
    return f == 0 ? GG_ACC(n_pp)
                  : f == 1 ? GG_ACC(n_cand)
                           : f == 2 ? GG_ACC(n_coinc)
                                    : f == 3 ? GG_ACC(n_body) : f == 4 ? GG_ACC(n_deg) : GG_ACC(max_psi_bits);
  };
  int e0 = 0;
  const bool uni = D.E == 1 || warp_env_uniform(env, &e0);
  if (uni) {
    const unsigned long long v[6] = {warp_sum(n_pp), warp_sum(n_cand), warp_sum(n_coinc),
                                     warp_sum(n_body), warp_sum(n_deg), warp_umax64(mp)};
    if (D.E == 1) {
      if (lane == 0)
#pragma unroll
        for (int f = 0; f < 6; ++f) s_acc[w][f] = v[f];
    } else if (lane == 0) {
#pragma unroll
      for (int f = 0; f < 5; ++f)
        if (v[f]) atomicAdd(acc_field(D, e0, offs(f)), v[f]);
      if (v[5]) atomicMax(acc_field(D, e0, offs(5)), v[5]);
    }
  } else {
    const unsigned long long v[6] = {n_pp, n_cand, n_coinc, n_body, n_deg, mp};
#pragma unroll
    for (int f = 0; f < 5; ++f)
      if (v[f]) atomicAdd(acc_field(D, env, offs(f)), v[f]);
    if (mp) atomicMax(acc_field(D, env, offs(5)), mp);
  }
  if (D.E != 1) return;
  __syncthreads();
  if (threadIdx.x < 6) {
    const int f = threadIdx.x;
    unsigned long long t = 0;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q)
      t = f < 5 ? t + s_acc[q][f] : (s_acc[q][f] > t ? s_acc[q][f] : t);
    if (t) {
      if (f < 5)
        atomicAdd(acc_field(D, 0, offs(f)), t);
      else
        atomicMax(acc_field(D, 0, offs(f)), t);
    }
  }
}

// contact-kernel sub-phase stamps of block 0, thread 0 (tstamp[48 + i];
// phase timer, debug builds with -DGG_CSTAMP=1 only: the check costs the
// large-n contact kernel registers)
#ifndef GG_CSTAMP
#define GG_CSTAMP 0
#endif
__device__ __forceinline__ void cstamp(const Dev& D, int i) {
  if (GG_CSTAMP && D.tstamp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    D.tstamp[48 + i] = t;
  }
}

// Phase B of the contact kernel (after a phase A filled sm.pass / the
// candidate lists): warp-cooperative exact test of the queued prefilter
// passes, body contacts, one record allocation per block, the records, the
// counters.  `cand` is the array the queue and lists index (the
// bucket-ordered copy Xh).  Called by every thread of the block.
template <class SM>
__device__ __forceinline__ void contacts_finish(const Dev& D, Ctl* ctl, int base, SM& sm,
                                                const float4* cand, bool live, int k, int env,
                                                float4 pf, uint32_t total, uint32_t npass,
                                                unsigned long long n_cand, unsigned long long n_coinc,
                                                unsigned long long n_deg) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5, wb = w * 32;
  sm.pos[tid] = pf;
  cstamp(D, 3);
  // ---- phase B: warp-cooperative exact test, one pass --------------------------
  // Every queued candidate (a prefilter pass) gets a record slot: its owner's
  // offset + its index in the owner's queue, so slots are known before the
  // exact test runs.  The rare pass that is not a contact (coincident, or
  // inside the prefilter's 1e-5 margin) leaves a null record the sweeps skip.
  const uint32_t np = npass < kPassCap ? npass : kPassCap;
  const bool ovf = npass > kPassCap;
  uint32_t incl = np;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t excl = incl - np;
  const uint32_t Tw = __shfl_sync(0xffffffffu, incl, 31);
  sm.off[w][lane] = excl;
  for (uint32_t i = 0; i < np; ++i) sm.qown[w][excl + i] = static_cast<uint8_t>(lane);
  int c_pp = 0;           // hits counted by this lane (queue entries it tested)
  int c_own = np;         // record slots this owner needs for pp contacts
  double max_psi = 0.0;
  if (ovf) {  // more prefilter passes than the queue holds: exact inline count
    int s_ex = 0, c_ex = 0;
    unsigned long long co_ex = 0;
    scan_exact(D, sm, cand, tid, k, pf, total, false, 0, s_ex, c_ex, co_ex, max_psi);
    c_own = s_ex;
  }
  // this env's bodies at this step: bodies[step][env][nb]
  const gg_body* bodies = D.bodies + (static_cast<long long>(ctl->step) * D.E + env) * D.nb;
  cstamp(D, 4);
  const int c_b = (live && D.nb > 0) ? body_contacts(D, bodies, pf, false, k, 0, 0, n_deg, max_psi) : 0;
  cstamp(D, 5);
  // ---- allocation: a fixed region per warp -----------------------------------
  // (records 0 .. kFixedSlots-1 of each owner are its fixed slots; records
  // kFixedSlots.. of the warp's 32 owners are laid end to end, in lane
  // order, from nrec0 + warp * wcap — an address the sweeps know without
  // reading anything, so they request a warp's records with its heads)
  const int tot = c_own + c_b;
  const int talloc = tot > kFixedSlots ? tot - kFixedSlots : 0;
  int wincl = talloc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, wincl, o);
    if (lane >= o) wincl += y;
  }
  const long long wbase = D.nrec0 + (static_cast<long long>(base + wb) >> 5) * D.wcap;
  const long long my_off = wbase + (wincl - talloc);
  const int wtot = __shfl_sync(0xffffffffu, wincl, 31);
  const bool fits = wtot <= D.wcap;
  if (!fits && lane == 0) {
    // slots per particle that would hold this warp's records
    const long long need = (static_cast<long long>(wtot) + 31) / 32 + kFixedSlots + 1;
    atomicMax(&ctl->cap_needed, static_cast<int>(need < (1 << 30) ? need : (1 << 30)));
    raise_err(ctl, GG_ECAPACITY);
  }
  __syncwarp();  // sm.pos / off / qown / pass of the warp's lanes
  const uint32_t* offw = sm.off[w];
  if (fits) {
    // pp records, cooperatively in queue order
    const bool uni = (D.E == 1) || __all_sync(0xffffffffu, env == __shfl_sync(0xffffffffu, env, 0));
    for (uint32_t r = 0; r * 32 < Tw; ++r) {
      const uint32_t idx = r * 32 + lane;
      const int o = idx < Tw ? sm.qown[w][idx] : 0;
      const long long oo = __shfl_sync(0xffffffffu, my_off, o);
      const bool oovf = __shfl_sync(0xffffffffu, ovf, o);
      if (idx < Tw && !oovf) {
        const uint32_t i = idx - offw[o];
        const long long dst = ridx(D, base + wb + o, oo, static_cast<int>(i));
        const float4 qf = cand[sm.pass[i][wb + o]];
        const float4 of = sm.pos[wb + o];
        double dx, dy, dz;
        const double d2 = pp_d2(of.x, of.y, of.z, qf, dx, dy, dz);
        const bool coi = !(d2 >= D.coinc_d2);
        if (!coi && d2 < D.contact_d2) {
          const double psi = pp_write(D, dst, dx, dy, dz, d2, __float_as_int(qf.w));
          if (uni) {
            max_psi = nmax(max_psi, psi);
            ++c_pp;
          } else {  // warp straddles two envs (rare): the owner's env directly
            Acc* a = D.acc + env_of(D, base + wb + o);
            if (psi > 0.0) atomicMax(&a->max_psi_bits, dbits(psi));
            atomicAdd(&a->n_pp, 1ull);
          }
        } else {
          D.coth[dst] = kNullContact;
          if (coi) {
            if (uni)
              ++n_coinc;
            else
              atomicAdd(&D.acc[env_of(D, base + wb + o)].n_coinc, 1ull);
          }
        }
      }
    }
    if (live) {
      if (ovf) {
        int s_ex = 0, c_ex = 0;
        unsigned long long co_ex = 0;
        scan_exact(D, sm, cand, tid, k, pf, total, true, my_off, s_ex, c_ex, co_ex, max_psi);
        c_pp += c_ex;
        n_coinc += co_ex;
      }
      if (c_b > 0) body_contacts(D, bodies, pf, true, k, my_off, c_own, n_deg, max_psi);
      D.cinfo[k] = make_int2(static_cast<int>(my_off), tot);
    }
  }
  cstamp(D, 6);
  acc_contacts(D, env, static_cast<unsigned long long>(c_pp), n_cand, n_coinc,
               static_cast<unsigned long long>(c_b), n_deg, max_psi);
}

// The flat candidate loop of phase A over the thread's bucket list (ttest
// candidates, kDepth in flight): the float32 prefilter, passes queued in
// sm.pass.  CHK: every candidate is checked against ttest; without it the
// sentinel entry points at Xh's far padding (GG_FAR_SENTINEL), whose
// entries never pass the prefilter — not usable when every candidate passes
// (TWO_LOOPS_FUSED).
template <bool CHK, class SM>
__device__ __forceinline__ void cand_loop(SM& sm, int tid, int k, float4 pf, const float4* Xh, uint32_t ttest,
                                          float rej, bool all, uint32_t& npass) {
  CandCursor cur;
  cur.init(sm, tid);
  constexpr int kDepth = SM::kDepth;  // candidates in flight per thread
  static_assert(kDepth <= kXhPad, "the sentinel bucket reads up to kDepth - 1 entries past n");
  for (uint32_t i = 0; i < ttest; i += kDepth) {
    uint32_t mi[kDepth];
#pragma unroll
    for (int u = 0; u < kDepth; ++u) mi[u] = cur.next(sm, tid, true);
    float4 qv[kDepth];
#pragma unroll
    for (int u = 0; u < kDepth; ++u) qv[u] = Xh[mi[u]];
#pragma unroll
    for (int u = 0; u < kDepth; ++u) {
      const float4 qf = qv[u];
      // float32 pre-filter, conservative by a 1e-5 relative margin (the
      // float32 estimate is within ~4e-7 relative of the exact square)
      const float fx = pf.x - qf.x, fy = pf.y - qf.y, fz = pf.z - qf.z;
#if GG_PASS_PRED
      // branch-free: every candidate is stored at the queue's next slot
      // (a candidate that does not pass leaves a value the next pass
      // overwrites, or one past the queue's end that nothing reads), and
      // only passes advance it — no divergent branch per candidate
      const bool valid = (!CHK || i + u < ttest) & (__float_as_int(qf.w) != k);
      const bool pass = valid & ((fx * fx + fy * fy + fz * fz <= rej) | all);
      if (npass < kPassCap) sm.pass[npass][tid] = mi[u];
      npass += pass ? 1u : 0u;
#else
      const bool pass = (!CHK || i + u < ttest) && __float_as_int(qf.w) != k &&
                        (fx * fx + fy * fy + fz * fz <= rej || all);
      if (pass) {
        if (npass < kPassCap) sm.pass[npass][tid] = mi[u];
        ++npass;
      }
#endif
    }
  }
}

// K5+K6: all contacts of particles base .. base+blockDim (contact.py:244-300).
//
// Phase A (per thread): the 27 neighbour-bucket bounds (three batches of 9
//   independent loads; empty and duplicate buckets dropped) compacted into a
//   per-thread list in shared memory, then ONE flat loop over the candidates
//   with a conservative float32 reject; survivors are queued (shared memory).
// Phase B (per warp): the warp's queued candidates are laid end to end and
//   tested exactly in float64 by all 32 lanes (no lane idles on a
//   neighbour's contact); ballots give each owner its contacts in candidate
//   order.  Bodies are counted per thread, the warp allocates its records
//   with ONE atomic (warp-contiguous CSR: cinfo[k] = {offset, count}), and
//   the records are written in a second cooperative pass.  Records of one
//   owner stay in candidate order, then bodies in index order, so results
//   do not depend on where the allocator put them.
// Particles base .. base + count - 1 (count <= blockDim.x) belong to this block.
template <class SM, bool DC = false, bool CULL = (GG_CULL != 0), bool FAR = (GG_FAR_SENTINEL != 0)>
__device__ __forceinline__ void ph_contacts(const Dev& D, Ctl* ctl, int base, int count,
                                            SM& sm) {
  // plain (coherent) loads: in the fused kernel these buffers are written
  // earlier in the same launch, so the read-only (.nc) path is not allowed
  const float4* LX = layout(D, ctl).x;
  const float4* Xh = D.Xh;
  const int tid = threadIdx.x;
  const int k = base + tid;
  const bool live = tid < count && k < live_own<DC>(D);
  const int env = env_of(D, live ? k : D.n - 1);
  cstamp(D, 0);
  unsigned long long n_cand = 0, n_coinc = 0, n_deg = 0;
  uint32_t total = 0, npass = 0;
  uint32_t ttest = 0;  // candidates in the walked buckets (total less the culled ones)
  float4 pf = make_float4(0.f, 0.f, 0.f, 0.f);
  // ---- phase A ------------------------------------------------------------
  if (live) {
    // this env's table: buckets [env*n_h, (env+1)*n_h)
    const uint32_t* start = D.start + static_cast<long long>(env) * D.H.n_h;
    pf = LX[k];
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
    // Geometric bucket culling: neighbour cell o's members lie in its box, so
    // none is within reach if the box's nearest point is farther than the
    // prefilter radius (+0.1%): such a bucket still counts its members as
    // candidates (n_candidates) but is not walked.  Every prefilter pass
    // survives, so the queue, the records and the results are unchanged.
    // Off where one bucket may serve two neighbour cells (dedup) and where
    // every candidate gets a record (TWO_LOOPS_FUSED).
    const bool cull_on = CULL && !dedup && D.pipeline != 1;
    float fq[3][3];  // per axis: squared distance to the lower / own / upper neighbour cell
    {
      const double pc[3] = {px, py, pz};
      const long long cc[3] = {c0, c1, c2};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double lo = pc[a] - (static_cast<double>(cc[a]) - 0.5) * D.two_r;
        const double hi = (static_cast<double>(cc[a]) + 0.5) * D.two_r - pc[a];
        fq[a][0] = static_cast<float>(lo * lo);
        fq[a][1] = 0.f;
        fq[a][2] = static_cast<float>(hi * hi);
      }
    }
    const float cull_d2 = D.reject_d2f * 1.001f;
    // bit o: neighbour o's bucket was already visited at an earlier offset
    // (rare: only particles whose 27 cells can alias run this loop; a real
    // branch, not predicated code every lane would issue)
    uint32_t dupmask = 0u;
    if (dedup) {
      uint32_t hh[27];
#pragma unroll
      for (int o = 0; o < 27; ++o) hh[o] = nb_hash(D, o, c0, c1, c2, tx, ty, tz);
#pragma unroll
      for (int o = 1; o < 27; ++o) {
        bool dup = false;
#pragma unroll
        for (int q = 0; q < o; ++q) dup |= hh[q] == hh[o];
        dupmask |= dup ? (1u << o) : 0u;
      }
    }
    int nb = 0;
    bool big = false;
    constexpr int kPerG = 27 / SM::kGroups;
#pragma unroll
    for (int g = 0; g < SM::kGroups; ++g) {
      uint32_t hb[kPerG], sb[kPerG], eb[kPerG];
      // the table kind is tested once per round, not once per bucket
      if (D.H.pow2) {
#pragma unroll
        for (int j = 0; j < kPerG; ++j) {
          const int o = g * kPerG + j, ox = o / 9, oy = (o / 3) % 3, oz = o % 3;
          hb[j] = (tx[ox] ^ ty[oy] ^ tz[oz]) & D.H.mask;
        }
      } else {
#pragma unroll
        for (int j = 0; j < kPerG; ++j) {
          const int o = g * kPerG + j;
          hb[j] = hash_cell64(c0 + o / 9 - 1, c1 + (o / 3) % 3 - 1, c2 + o % 3 - 1, D.H.n_h);
        }
      }
#pragma unroll
      for (int j = 0; j < kPerG; ++j) {
        sb[j] = start[hb[j]];
        eb[j] = start[hb[j] + 1];
      }
#pragma unroll
      for (int j = 0; j < kPerG; ++j) {
        const bool keep = eb[j] > sb[j] && !((dupmask >> (g * kPerG + j)) & 1u);
#if GG_PASS_PRED
        // branch-free: stored at the list's next entry, kept buckets advance
        // it (a dropped one is overwritten by the next kept bucket or by the
        // sentinel)
        const int o = g * kPerG + j;  // (a constant: both loops are unrolled)
        const bool reach = !cull_on || fq[0][o / 9] + fq[1][(o / 3) % 3] + fq[2][o % 3] <= cull_d2;
        const uint32_t L = keep ? eb[j] - sb[j] : 0u;
        total += L;
        big |= L >= kLenSentinel;
        const uint32_t Lt = reach ? L : 0u;
        ttest += Lt;
        sm.beg[nb][tid] = sb[j];
        sm.len[nb][tid] = static_cast<NarrowLen>(Lt);
        nb += (keep && reach) ? 1 : 0;
#else
        if (keep) {
          const uint32_t L = eb[j] - sb[j];
          total += L;
          ttest += L;
          big |= L >= kLenSentinel;
          sm.beg[nb][tid] = sb[j];
          sm.len[nb][tid] = static_cast<NarrowLen>(L);
          ++nb;
        }
#endif
      }
    }
    if (big) {
      // a bucket longer than the 16-bit list lengths (a tiny table with very
      // many particles per bucket): rebuild the list with such buckets as
      // consecutive entries of at most kLenSentinel - 1 (candidate order
      // unchanged); more entries than the list holds is refused, never truncated
      nb = 0;
      for (int o = 0; o < 27; ++o) {
        if ((dupmask >> o) & 1u) continue;
        const uint32_t h = nb_hash(D, o, c0, c1, c2, tx, ty, tz);
        uint32_t s0 = start[h];
        for (uint32_t left = start[h + 1] - s0; left > 0;) {
          const uint32_t c = left < kLenSentinel - 1 ? left : kLenSentinel - 1;
          if (nb >= 27) {
            raise_err(ctl, GG_EBUCKET);
            left = 0;
            break;
          }
          sm.beg[nb][tid] = s0;
          sm.len[nb][tid] = static_cast<NarrowLen>(c);
          ++nb;
          s0 += c;
          left -= c;
        }
      }
      ttest = total;  // (every bucket walked)
    }
    cstamp(D, 1);
    n_cand = total - 1;  // minus the self pair (one per particle, broadphase.py:441-447)
    // sentinel after the last bucket: the cursor may run up to kDepth - 1
    // candidates past the end without a guard (indices < n + kXhPad: Xh is
    // padded; never tested)
    sm.beg[nb][tid] = FAR ? static_cast<uint32_t>(D.xh_pad) : sm.beg[0][tid];
    sm.len[nb][tid] = static_cast<NarrowLen>(kLenSentinel);
    const bool all = D.pipeline == 1;
    const float rej = D.reject_d2f;
    if (FAR && !all)
      cand_loop<false>(sm, tid, k, pf, Xh, ttest, rej, all, npass);
    else
      cand_loop<true>(sm, tid, k, pf, Xh, ttest, rej, all, npass);
  }
  cstamp(D, 2);
  contacts_finish(D, ctl, base, sm, Xh, live, k, env, pf, ttest, npass, n_cand, n_coinc, n_deg);
  cstamp(D, 7);
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

// Body reaction momentum of the first kRegBodies bodies is summed per thread
// in registers (exact fixed-point adds), reduced across the warp with
// shuffles and only then added to shared memory: 64-bit shared atomics are
// CAS loops, and the floor contacts of a warp all hit the same three words.
constexpr int kRegBodies = 1;

struct SweepAcc {
  double maxviol, minb1;
  int env;                  // env of the particle being swept (E > 1)
  int gb_lo;                // first global body slot (env * nb + b) held in sbm
  unsigned long long* sbm;  // shared [kSmemBodies][3]
  unsigned long long rb[kRegBodies][3];  // this thread's momentum of bodies 0..kRegBodies-1
};

// k0: the first particle this thread sweeps (its env seeds A.env); kb: the
// block's first particle (-1: blockIdx.x * blockDim.x)
__device__ __forceinline__ void sweep_acc_init(const Dev& D, SweepAcc& A, unsigned long long* sbm,
                                               int k0, int kb = -1) {
  A.maxviol = 0.0;
  A.minb1 = __longlong_as_double(0x7ff0000000000000ll);
  A.sbm = sbm;
  A.env = env_of(D, k0 < D.n ? k0 : D.n - 1);
  if (kb < 0) kb = static_cast<int>(blockIdx.x) * static_cast<int>(blockDim.x);
  A.gb_lo = env_of(D, kb < D.n ? kb : D.n - 1) * D.nb;
#pragma unroll
  for (int b = 0; b < kRegBodies; ++b) A.rb[b][0] = A.rb[b][1] = A.rb[b][2] = 0ull;
  for (int i = threadIdx.x; i < kSmemBodies * 3; i += blockDim.x) sbm[i] = 0ull;
  __syncthreads();
}

// this thread's register momentum straight to the global accumulators of env
__device__ __forceinline__ void sweep_acc_rb_global(const Dev& D, SweepAcc& A) {
#pragma unroll
  for (int b = 0; b < kRegBodies; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (A.rb[b][c]) atomicAdd(&D.bm_fix[(A.env * D.nb + b) * 3 + c], A.rb[b][c]);
      A.rb[b][c] = 0ull;
    }
}

// Strided loops (persistent kernels) may hand a thread particles of several
// envs: diagnostics gathered for the previous env are flushed lane-wise
// before the next particle's are accumulated.
__device__ __forceinline__ void sweep_acc_env(const Dev& D, SweepAcc& A, int k) {
  if (D.E == 1) return;
  const int e = env_of(D, k);
  if (e == A.env) return;
  Acc* a = D.acc + A.env;
  sweep_acc_rb_global(D, A);
  if (A.maxviol > 0.0) atomicMax(&a->max_viol_bits, dbits(A.maxviol));
  if (A.minb1 == A.minb1 && A.minb1 < __longlong_as_double(0x7ff0000000000000ll))
    atomicMin(&a->min_b1_bits, dbits(A.minb1));
  A.maxviol = 0.0;
  A.minb1 = __longlong_as_double(0x7ff0000000000000ll);
  A.env = e;
}


// per block: diagnostics (max cone violation, min normal impulse: warp
// reductions on the bit patterns, one atomic each per block) + body momentum
// (warp sums only where a lane holds momentum, one atomic per non-zero
// component).  One block barrier.  Called by every thread.
// maxviol >= +0.0 and minb1 in [+0.0, +inf] by construction (contact_impulse
// never stores a NaN: a NaN impulse makes w non-finite and the step raises).
__device__ __forceinline__ void sweep_acc_flush(const Dev& D, SweepAcc& A, double* /*unused*/) {
  __shared__ unsigned long long s_wred[2 * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int e0 = A.env;
  const bool uni = D.E == 1 || warp_env_uniform(A.env, &e0);
  if (uni) {
    const unsigned long long m1 = warp_umax64(dbits(A.maxviol));
    const unsigned long long m2 = warp_umin64(dbits(A.minb1));
#pragma unroll
    for (int b = 0; b < kRegBodies; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (__any_sync(0xffffffffu, A.rb[b][c] != 0ull)) {
          const unsigned long long t = warp_sum(A.rb[b][c]);
          if (lane == 0 && t && b < D.nb) {
            const int gb = e0 * D.nb + b;
            const int sl = gb - A.gb_lo;
            atomicAdd((sl >= 0 && sl < kSmemBodies) ? A.sbm + 3 * sl + c : D.bm_fix + 3 * gb + c, t);
          }
        }
        A.rb[b][c] = 0ull;
      }
    if (lane == 0) {
      if (D.E == 1) {
        s_wred[2 * w] = m1;
        s_wred[2 * w + 1] = m2;
      } else {
        Acc* a = D.acc + e0;
        if (m1 != 0ull) atomicMax(&a->max_viol_bits, m1);
        if (m2 < kInfBits) atomicMin(&a->min_b1_bits, m2);
      }
    }
  } else {
    sweep_acc_rb_global(D, A);
    Acc* a = D.acc + A.env;
    if (A.maxviol > 0.0) atomicMax(&a->max_viol_bits, dbits(A.maxviol));
    if (A.minb1 < __longlong_as_double(kInfBits)) atomicMin(&a->min_b1_bits, dbits(A.minb1));
  }
  A.maxviol = 0.0;
  A.minb1 = __longlong_as_double(kInfBits);
  __syncthreads();
  if (D.E == 1 && threadIdx.x == 0) {
    unsigned long long m1 = 0ull, m2 = kInfBits;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
      m1 = s_wred[2 * q] > m1 ? s_wred[2 * q] : m1;
      m2 = s_wred[2 * q + 1] < m2 ? s_wred[2 * q + 1] : m2;
    }
    if (m1 != 0ull) atomicMax(&D.acc->max_viol_bits, m1);
    if (m2 < kInfBits) atomicMin(&D.acc->min_b1_bits, m2);
  }
  for (int i = threadIdx.x; i < kSmemBodies * 3; i += blockDim.x)
    if (A.sbm[i]) atomicAdd(&D.bm_fix[A.gb_lo * 3 + i], A.sbm[i]);
}

// Barrier-free variant for the per-sweep kernel (no shared accumulators):
// every warp reduces its diagnostics and register momentum and issues its
// own global atomics.  A diagnostic atomic is skipped when the warp's value
// cannot change the global one (compared against a plain read of it: the
// global max only grows and the min only shrinks, so a stale read is a safe
// lower / upper bound), so nearly all warps issue none; body momentum atomics
// come only from warps with body contacts.  Bodies >= kRegBodies go straight
// to the global accumulators (sweep_acc_init_nobar).  Same sums (integer
// fixed point) and extrema as sweep_acc_flush.
__device__ __forceinline__ void sweep_acc_init_nobar(const Dev& D, SweepAcc& A, int k0) {
  A.maxviol = 0.0;
  A.minb1 = __longlong_as_double(kInfBits);
  A.sbm = nullptr;
  A.env = env_of(D, k0 < D.n ? k0 : D.n - 1);
  A.gb_lo = -(1 << 30);  // no shared slots: contact_impulse uses bm_fix
#pragma unroll
  for (int b = 0; b < kRegBodies; ++b) A.rb[b][0] = A.rb[b][1] = A.rb[b][2] = 0ull;
}

__device__ __forceinline__ void sweep_acc_flush_nobar(const Dev& D, SweepAcc& A) {
  const int lane = threadIdx.x & 31;
  int e0 = A.env;
  const bool uni = D.E == 1 || warp_env_uniform(A.env, &e0);
  if (uni) {
    const unsigned long long m1 = warp_umax64(dbits(A.maxviol));
    const unsigned long long m2 = warp_umin64(dbits(A.minb1));
#pragma unroll
    for (int b = 0; b < kRegBodies; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (__any_sync(0xffffffffu, A.rb[b][c] != 0ull)) {
          const unsigned long long t = warp_sum(A.rb[b][c]);
          if (lane == 0 && t && b < D.nb) atomicAdd(D.bm_fix + 3 * (e0 * D.nb + b) + c, t);
        }
    if (lane == 0) {
      Acc* a = D.acc + e0;
      if (m1 != 0ull && m1 > *((volatile unsigned long long*)&a->max_viol_bits))
        atomicMax(&a->max_viol_bits, m1);
      if (m2 < kInfBits && m2 < *((volatile unsigned long long*)&a->min_b1_bits))
        atomicMin(&a->min_b1_bits, m2);
    }
  } else {
    sweep_acc_rb_global(D, A);
    Acc* a = D.acc + A.env;
    if (A.maxviol > 0.0) atomicMax(&a->max_viol_bits, dbits(A.maxviol));
    if (A.minb1 < __longlong_as_double(kInfBits)) atomicMin(&a->min_b1_bits, dbits(A.minb1));
  }
}

// The owner's adds of its records' impulses in chunk [cb, cb + 32): records
// a0 .. a1 - 1 in order.  GG_OWNER_UNIFORM: every lane runs the warp's
// largest count with predicated adds (no divergent loop); the same adds in
// the same order either way.
#ifndef GG_OWNER_UNIFORM
#define GG_OWNER_UNIFORM 1
#endif
#ifndef GG_SLIDE_PRED
#define GG_SLIDE_PRED 0
#endif
#ifndef GG_MINE_PRED
#define GG_MINE_PRED 0
#endif
__device__ __forceinline__ void owner_sums(const double (*imp)[32], uint32_t a0, uint32_t a1, uint32_t cb,
                                           double& ax, double& ay, double& az) {
  if (GG_OWNER_UNIFORM) {
    const uint32_t cnt = a1 > a0 ? a1 - a0 : 0u;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, cnt);
    const uint32_t b = a1 > a0 ? a0 - cb : 0u;
    for (uint32_t q = 0; q < mx; ++q) {
      const bool on = q < cnt;
      const uint32_t i = on ? b + q : 0u;
      const double vx = imp[0][i], vy = imp[1][i], vz = imp[2][i];
      ax = on ? ax + vx : ax;
      ay = on ? ay + vy : ay;
      az = on ? az + vz : az;
    }
  } else {
    for (uint32_t rr = a0; rr < a1; ++rr) {
      ax += imp[0][rr - cb];
      ay += imp[1][rr - cb];
      az += imp[2][rr - cb];
    }
  }
}

// The impulse of one contact record on its owner (contact.py:463-488), in
// float64 with explicit fused multiply-adds (the library is built with
// --fmad=false so that contact DECISIONS follow numpy's operation order;
// the solver's arithmetic only has to meet the 1e-5 parity bar, and every
// schedule evaluates this same function, so they stay bitwise identical).
__device__ __forceinline__ void contact_impulse(const Dev& D, double wx, double wy, double wz,
                                                float4 g, int j, float4 q, double& ax, double& ay,
                                                double& az, SweepAcc& A, bool on = true) {
  // on == false: evaluated but without effect (a lane with no record in a
  // warp-uniform call; its inputs may be anything)
  const double eff = (j >= 0) ? 0.5 : 1.0;  // both partners mobile (contact.py:457-460)
  const double e1x = g.x, e1y = g.y, e1z = g.z;
  const double ng = -D.gamma;
  const double ux = fma(ng, static_cast<double>(q.x), wx) + D.gdt0;
  const double uy = fma(ng, static_cast<double>(q.y), wy) + D.gdt1;
  const double uz = fma(ng, static_cast<double>(q.z), wz) + D.gdt2;
  const double un = fma(uz, e1z, fma(uy, e1y, ux * e1x));
  // np.maximum(x, 0): x if x > 0 or x is NaN, else +0.0 (one unordered compare)
  const double bx = fma(D.bias_coef, static_cast<double>(g.w), -un);
  const double b1 = !(bx <= 0.0) ? bx : 0.0;
  double btx = fma(un, e1x, -ux), bty = fma(un, e1y, -uy), btz = fma(un, e1z, -uz);
  const double tn2 = fma(btz, btz, fma(bty, bty, btx * btx));
  const double lim = D.mu * b1;
#if GG_SLIDE_PRED
  {  // sliding: the projection below as selects (no divergent branch)
    const bool slide = tn2 > lim * lim;
    const double inv = rsqrt(slide ? tn2 : 1.0);
    const double sc = lim * inv;
    btx = slide ? btx * sc : btx;
    bty = slide ? bty * sc : bty;
    btz = slide ? btz * sc : btz;
    const double viol = fma(tn2 * inv, sc, -lim);
    A.maxviol = (on && slide && viol > A.maxviol) ? viol : A.maxviol;
  }
#else
  if (tn2 > lim * lim) {  // sliding: project onto the Coulomb cone
    // scale = lim / |bt| with one reciprocal square root (tn2 > lim^2 >= 0,
    // so tn2 > 0); 1-ulp accurate, far inside the 1e-5 parity bar
    const double inv = rsqrt(tn2);
    const double sc = lim * inv;
    btx *= sc;
    bty *= sc;
    btz *= sc;
    const double viol = fma(tn2 * inv, sc, -lim);
    if (on && viol > A.maxviol) A.maxviol = viol;
  }
#endif
  const double ix = fma(e1x, b1, btx) * eff;
  const double iy = fma(e1y, b1, bty) * eff;
  const double iz = fma(e1z, b1, btz) * eff;
  ax = on ? ax + ix : ax;
  ay = on ? ay + iy : ay;
  az = on ? az + iz : az;
  A.minb1 = (on && b1 < A.minb1) ? b1 : A.minb1;
  if (on && j < 0) {  // reaction momentum on the body (contact.py:489-495)
    const int b = -j - 1;
    const unsigned long long fx = to_fix(-D.mass * ix), fy = to_fix(-D.mass * iy),
                             fz = to_fix(-D.mass * iz);
    if (b < kRegBodies) {
#pragma unroll
      for (int q = 0; q < kRegBodies; ++q)
        if (q == b) {
          A.rb[q][0] += fx;
          A.rb[q][1] += fy;
          A.rb[q][2] += fz;
        }
    } else {
      const int gb = A.env * D.nb + b;  // global body slot
      const int sl = gb - A.gb_lo;
      unsigned long long* bm = (sl >= 0 && sl < kSmemBodies) ? A.sbm + 3 * sl : D.bm_fix + 3 * gb;
      atomicAdd(bm + 0, fx);
      atomicAdd(bm + 1, fy);
      atomicAdd(bm + 2, fz);
    }
  }
}

// ONE_LOOP (stepper.py:86-98): the sweep repeats the collision test — the
// 27 de-duplicated buckets, the candidates, the exact test, the body SDFs —
// instead of reading contact records, and applies the impulses in the same
// order with the same float32-stored geometry, so the result is bitwise that
// of TWO_LOOPS_SPLIT.
__device__ __forceinline__ void sweep_oneloop(const Dev& D, int k, const float4* Win, double wx,
                                           double wy, double wz, double& ax, double& ay, double& az,
                                           SweepAcc& A) {
  const Layout L = layout(D, D.ctl);
  const int env = env_of(D, k);
  const uint32_t* start = D.start + static_cast<long long>(env) * D.H.n_h;
  const float4 pf = L.x[k];
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
  for (int o = 0; o < 27; ++o) {
    const uint32_t h = nb_hash(D, o, c0, c1, c2, tx, ty, tz);
    bool keep = true;
    if (dedup)
      for (int q = 0; q < o; ++q) keep &= nb_hash(D, q, c0, c1, c2, tx, ty, tz) != h;
    if (!keep) continue;
    for (uint32_t m = start[h]; m < start[h + 1]; ++m) {
      const float4 qf = D.Xh[m];
      const int q = __float_as_int(qf.w);
      if (q == k) continue;
      const float fx = pf.x - qf.x, fy = pf.y - qf.y, fz = pf.z - qf.z;
      if (!(fx * fx + fy * fy + fz * fz <= D.reject_d2f)) continue;
      double dx, dy, dz;
      const double d2 = pp_d2(px, py, pz, qf, dx, dy, dz);
      if (!(d2 >= D.coinc_d2) || !(d2 < D.contact_d2)) continue;
      const double inv = rsqrt(d2);
      const double psi = __dsub_rn(D.two_r, d2 * inv);
      const float4 g = make_float4(static_cast<float>(dx * inv), static_cast<float>(dy * inv),
                                   static_cast<float>(dz * inv), static_cast<float>(psi));
      contact_impulse(D, wx, wy, wz, g, q, Win[q], ax, ay, az, A);
    }
  }
  const gg_body* bodies = D.bodies + (static_cast<long long>(D.ctl->step) * D.E + env) * D.nb;
  for (int b = 0; b < D.nb; ++b) {
    const gg_body& B = bodies[b];
    if (B.bounded && !(px >= B.aabb_lo[0] && px <= B.aabb_hi[0] && py >= B.aabb_lo[1] &&
                       py <= B.aabb_hi[1] && pz >= B.aabb_lo[2] && pz <= B.aabb_hi[2]))
      continue;
    double psi;
    d3 nrm;
    int deg;
    if (!penetrate(B, D.grids, D.gvals, px, py, pz, D.r, &psi, &nrm, &deg)) continue;
    const d3 vb = body_surface_velocity(B, px, py, pz, nrm, D.r, psi);
    const float4 g = make_float4(static_cast<float>(nrm.x), static_cast<float>(nrm.y),
                                 static_cast<float>(nrm.z), static_cast<float>(psi));
    const float4 qb = make_float4(static_cast<float>(vb.x), static_cast<float>(vb.y),
                                  static_cast<float>(vb.z), 0.f);
    contact_impulse(D, wx, wy, wz, g, -(b + 1), qb, ax, ay, az, A);
  }
}

// The fixed records of particle k and its CSR info, fetched together: one
// dependent round trip fewer than reading cinfo first (and, with two fixed
// slots, a second one for particles with two contacts).
struct SweepHead {
  int2 ci;
  float4 g[kFixedSlots];
  int j[kFixedSlots];
  __device__ __forceinline__ void load(const Dev& D, int k) {
    ci = D.cinfo[k];
#pragma unroll
    for (int i = 0; i < kFixedSlots; ++i) {
      g[i] = D.cgeo[static_cast<long long>(i) * D.n + k];
      j[i] = D.coth[static_cast<long long>(i) * D.n + k];
    }
  }
};

// L2 eviction hints for the record-major sweep.  A sweep reads ~50 MB of
// records and heads once and gathers / writes ~30 MB of w; at ~80 MB the
// whole set does not stay in L2 from one sweep to the next (ncu without
// cache flushing: 70 MB of DRAM reads per sweep, 28% L2 hits).  GG_L2HINT:
// bit 0 — records and heads are loaded evict-first (streamed), bit 1 — w is
// loaded and stored evict-last (kept for the next sweep).
#ifndef GG_L2HINT
#define GG_L2HINT 1
#endif
struct L2Pol {
  unsigned long long first, last;
  __device__ __forceinline__ void init() {
#if GG_L2HINT
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(last));
#endif
  }
};
__device__ __forceinline__ float4 ld_hint(const float4* a, unsigned long long pol, bool use) {
  float4 v;
  if (use)
    asm("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
  else
    v = *a;
  return v;
}
__device__ __forceinline__ int ld_hint(const int* a, unsigned long long pol, bool use) {
  int v;
  if (use)
    asm("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  else
    v = *a;
  return v;
}
__device__ __forceinline__ int2 ld_hint(const int2* a, unsigned long long pol, bool use) {
  int2 v;
  if (use)
    asm("ld.global.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(pol));
  else
    v = *a;
  return v;
}
__device__ __forceinline__ void st_hint(float4* a, float4 v, unsigned long long pol, bool use) {
  if (use)
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
  else
    *a = v;
}
constexpr bool kHintRec = (GG_L2HINT & 1) != 0;
constexpr bool kHintW = (GG_L2HINT & 2) != 0;

// The sweep of one particle with its head already loaded.  A particle without
// contacts keeps w = v and is nobody's partner (contacts are symmetric), so
// its w is never read: it is skipped entirely (integrate uses dv = 0).
__device__ __forceinline__ void sweep_particle_h(const Dev& D, int k, const SweepHead& h,
                                                 const float4* Win, float4* Wout, SweepAcc& A) {
  if (h.ci.y == 0) return;
  sweep_acc_env(D, A, k);
  const float4 wf = Win[k];
  const double wx = wf.x, wy = wf.y, wz = wf.z;
  double ax = 0.0, ay = 0.0, az = 0.0;
  float4 q[kFixedSlots];
#pragma unroll
  for (int i = 0; i < kFixedSlots; ++i)
    if (i < h.ci.y && h.j[i] != kNullContact)
      q[i] = (h.j[i] >= 0) ? Win[h.j[i]] : D.cvb[static_cast<long long>(i) * D.n + k];
#pragma unroll
  for (int i = 0; i < kFixedSlots; ++i)
    if (i < h.ci.y && h.j[i] != kNullContact)
      contact_impulse(D, wx, wy, wz, h.g[i], h.j[i], q[i], ax, ay, az, A);
  // records kFixedSlots .. c-1 at ci.x, ci.x + 1, ...
  const float4* gp = D.cgeo + h.ci.x;
  const int* jp = D.coth + h.ci.x;
  const float4* vp = D.cvb + h.ci.x;
  for (int sl = 0; sl < h.ci.y - kFixedSlots; ++sl) {
    const float4 g = gp[sl];
    const int j = jp[sl];
    if (j == kNullContact) continue;
    const float4 qq = (j >= 0) ? Win[j] : vp[sl];
    contact_impulse(D, wx, wy, wz, g, j, qq, ax, ay, az, A);
  }
  Wout[k] = make_float4(static_cast<float>(wx + ax), static_cast<float>(wy + ay),
                        static_cast<float>(wz + az), 0.f);
}

__device__ __forceinline__ void sweep_particle(const Dev& D, int k, const float4* Win, float4* Wout,
                                               SweepAcc& A) {
  SweepHead h;
  h.load(D, k);
  sweep_particle_h(D, k, h, Win, Wout, A);
}

// Register-resident variant for the fused kernel (one particle per thread):
// the first kRegSlots contacts and the particle's own w are loaded once and
// kept across all sweeps; each sweep issues its neighbour gathers together.
// Arithmetic and accumulation order are exactly those of sweep_particle.
#ifndef GG_REG_SLOTS
#define GG_REG_SLOTS 6
#endif
constexpr int kRegSlots = GG_REG_SLOTS;
#ifndef GG_REG_QB
#define GG_REG_QB 0
#endif
struct RegContacts {
  int c;
  float4 g[kRegSlots];
  int j[kRegSlots];
#if GG_REG_QB
  float4 qb[kRegSlots];  // body records' surface velocity (else re-read from cvb per sweep)
#endif
  float wx, wy, wz;

  int off;
  __device__ __forceinline__ void load(const Dev& D, int k, float4 w0) {
    // the fixed records are requested together with the count (their
    // indices do not depend on it), the CSR ones after it
#pragma unroll
    for (int s = 0; s < kFixedSlots; ++s) {
      const long long r = static_cast<long long>(s) * D.n + k;
      g[s] = D.cgeo[r];
      j[s] = D.coth[r];
    }
    const int2 ci = D.cinfo[k];
    c = ci.y;
    off = ci.x;
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s) {
      if (s < kFixedSlots) {
        if (s >= c) j[s] = 0;
#if GG_REG_QB
        else if (j[s] < 0) qb[s] = D.cvb[static_cast<long long>(s) * D.n + k];
#endif
        continue;
      }
      j[s] = 0;
      if (s < c) {
        const long long r = ridx(D, k, off, s);
        g[s] = D.cgeo[r];
        j[s] = D.coth[r];
#if GG_REG_QB
        if (j[s] < 0) qb[s] = D.cvb[r];
#endif
      }
    }
    wx = w0.x;
    wy = w0.y;
    wz = w0.z;
  }

  __device__ __forceinline__ void sweep(const Dev& D, int k, const float4* Win, float4* Wout,
                                        SweepAcc& A) {
    if (c == 0) return;  // no contacts: w is never read (see sweep_particle)
    float4 q[kRegSlots];
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s)
      if (s < c && j[s] != kNullContact)
#if GG_REG_QB
        q[s] = (j[s] >= 0) ? Win[j[s]] : qb[s];
#else
        q[s] = (j[s] >= 0) ? Win[j[s]] : D.cvb[ridx(D, k, off, s)];
#endif
    double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s)
      if (s < c && j[s] != kNullContact) contact_impulse(D, wx, wy, wz, g[s], j[s], q[s], ax, ay, az, A);
    for (int s = kRegSlots; s < c; ++s) {
      const long long idx = ridx(D, k, off, s);
      const float4 gg = D.cgeo[idx];
      const int jj = D.coth[idx];
      if (jj == kNullContact) continue;
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

// Record-major, register-resident sweeps for the fused kernel (one particle
// per thread): a warp keeps its 32 particles' record 0 (one per lane) and its
// first 64 CSR records (two per lane, ONE RECORD PER LANE per chunk) in
// registers across the sweeps, like k_sweep_rm does per launch: a particle
// with many contacts no longer makes its whole warp wait through a serial
// loop.  The owner adds its records' impulses in record order (record 0,
// then the CSR ones), exactly the sums of RegContacts::sweep.  A warp with
// more than 64 CSR records re-reads its records every sweep
// (sweep_particle_h).  Called by every lane of the warp.
#ifndef GG_FUSED_RM
#define GG_FUSED_RM 1
#endif
struct RegChunks {
  int c;                  // this lane's particle's record count
  uint32_t incl, excl, T;  // CSR records: inclusive / exclusive lane prefix, warp total
  float4 g0, g1, g2;       // record 0; CSR records lane and 32 + lane
  int j0, j1, j2;
  long long wb;            // the warp's CSR region
  float wx, wy, wz;        // this particle's w
  bool fallback;           // T > 64: per-particle sweeps from memory

  __device__ __forceinline__ void load(const Dev& D, int k, bool live, float4 w0) {
    const int lane = threadIdx.x & 31;
    c = 0;
    j0 = j1 = j2 = kNullContact;
    g0 = g1 = g2 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
      const int2 ci = D.cinfo[k];
      c = ci.y;
      g0 = D.cgeo[k];
      j0 = c > 0 ? D.coth[k] : kNullContact;
    }
    const uint32_t m = c > 1 ? static_cast<uint32_t>(c - 1) : 0u;
    incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    T = __shfl_sync(0xffffffffu, incl, 31);
    excl = incl - m;
    wb = D.nrec0 + static_cast<long long>(k >> 5) * D.wcap;
    fallback = T > 64;
    if (!fallback) {
      if (static_cast<uint32_t>(lane) < T) {
        g1 = D.cgeo[wb + lane];
        j1 = D.coth[wb + lane];
      }
      if (static_cast<uint32_t>(lane) + 32 < T) {
        g2 = D.cgeo[wb + 32 + lane];
        j2 = D.coth[wb + 32 + lane];
      }
    }
    wx = w0.x;
    wy = w0.y;
    wz = w0.z;
  }

  // the chunk whose lane-record is (g, j) at record index cb + lane: impulses
  // to shared memory, then each owner adds its records of the chunk in order
  __device__ __forceinline__ void chunk(const Dev& D, const float4* Win, uint32_t cb, float4 g, int j,
                                        double& ax, double& ay, double& az, SweepAcc& A,
                                        double (*imp)[32]) {
    const int lane = threadIdx.x & 31;
    const uint32_t r = cb + lane;
    const bool mine = r < T && j != kNullContact;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (mine) q = (j >= 0) ? Win[j] : D.cvb[wb + r];
    int o = 0;
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, incl, o + st - 1);
      if (v <= r) o += st;
    }
    o = o < 31 ? o : 31;
    const float owx = __shfl_sync(0xffffffffu, wx, o);
    const float owy = __shfl_sync(0xffffffffu, wy, o);
    const float owz = __shfl_sync(0xffffffffu, wz, o);
    double ix = 0.0, iy = 0.0, iz = 0.0;
    if (GG_MINE_PRED)
      contact_impulse(D, owx, owy, owz, g, j, q, ix, iy, iz, A, mine);
    else if (mine)
      contact_impulse(D, owx, owy, owz, g, j, q, ix, iy, iz, A);
    imp[0][lane] = ix;
    imp[1][lane] = iy;
    imp[2][lane] = iz;
    __syncwarp();
    const uint32_t a0 = excl > cb ? excl : cb;
    const uint32_t a1 = incl < cb + 32 ? incl : cb + 32;
    owner_sums(imp, a0, a1, cb, ax, ay, az);
    __syncwarp();
  }

  __device__ __forceinline__ void sweep(const Dev& D, int k, bool live, const float4* Win, float4* Wout,
                                        SweepAcc& A, double (*imp)[32]) {
    if (fallback) {  // (warp-uniform)
      if (live && c > 0) {
        SweepHead h;
        h.load(D, k);
        sweep_particle_h(D, k, h, Win, Wout, A);
      }
      return;
    }
    const bool has0 = c > 0 && j0 != kNullContact;
    float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (has0) q0 = (j0 >= 0) ? Win[j0] : D.cvb[k];
    double ax = 0.0, ay = 0.0, az = 0.0;
    if (has0) contact_impulse(D, wx, wy, wz, g0, j0, q0, ax, ay, az, A);
    if (T > 0) chunk(D, Win, 0, g1, j1, ax, ay, az, A, imp);
    if (T > 32) chunk(D, Win, 32, g2, j2, ax, ay, az, A, imp);
    if (c > 0) {
      const float4 out = make_float4(static_cast<float>(static_cast<double>(wx) + ax),
                                     static_cast<float>(static_cast<double>(wy) + ay),
                                     static_cast<float>(static_cast<double>(wz) + az), 0.f);
      Wout[k] = out;
      wx = out.x;
      wy = out.y;
      wz = out.z;
    }
  }
};

// per-env kinetic energy (E > 1): sum |v|^2 in 64-bit fixed point (2^-32),
// exact and order-independent like the body momentum
constexpr double kKeScale = 4294967296.0;  // 2^32
__device__ __forceinline__ unsigned long long to_ke_fix(double v2) {
  return static_cast<unsigned long long>(__double2ll_rn(v2 * kKeScale));
}

__device__ __forceinline__ void env_add_arr(const Dev& D, int env, unsigned long long v,
                                            unsigned long long* arr) {
  int e0;
  if (warp_env_uniform(env, &e0)) {
    const unsigned long long t = warp_sum(v);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(arr + e0, t);
  } else if (v) {
    atomicAdd(arr + env, v);
  }
}

__device__ __forceinline__ void write_report(const Dev& D, gg_report& R, const Acc* a, double ke_sum) {
  // L2 loads, all in flight together (other blocks / kernels wrote them;
  // volatile loads would be one round trip each)
  const unsigned long long n_pp = __ldcg(&a->n_pp), n_cand = __ldcg(&a->n_cand),
                           n_body = __ldcg(&a->n_body), n_coinc = __ldcg(&a->n_coinc),
                           n_deg = __ldcg(&a->n_deg), psi = __ldcg(&a->max_psi_bits),
                           viol = __ldcg(&a->max_viol_bits), b1 = __ldcg(&a->min_b1_bits);
  R.n_contacts = static_cast<long long>(n_pp);
  R.n_candidates = static_cast<long long>(n_cand);
  R.n_body_contacts = static_cast<long long>(n_body);
  R.n_coincident = static_cast<long long>(n_coinc);
  R.n_degenerate = static_cast<long long>(n_deg);
  R.max_penetration = __longlong_as_double(static_cast<long long>(psi));
  R.kinetic_energy = 0.5 * D.mass * ke_sum;
  R.max_cone_violation = __longlong_as_double(static_cast<long long>(viol));
  R.min_normal_impulse = __longlong_as_double(static_cast<long long>(b1));
}

// Symplectic Euler (stepper.py:102-106), SolverError check
// (contact.py:503-509), kinetic energy (stepper.py:118); the last block to
// finish reduces the per-block partials in fixed order into the StepReport(s)
// — one per env — and commits the new state.  Called by every thread of
// every block.
// This thread integrates particles kb, kb + step, ... < ke (its particles
// of the last sweep: another thread's w is not ordered before this read).
// Symplectic Euler of this thread's particles kb, kb + kstep, ... < kend and
// the block's kinetic-energy partial in D.part[blockIdx.x] (E == 1; E > 1
// adds to the per-env fixed-point sums).  Called by every thread.
__device__ __forceinline__ void integrate_range(const Dev& D, Ctl* ctl, int kb, int kend, int kstep,
                                                double* smd, int own) {
  const int cur = ctl->cur;
  const Layout L = layout(D, ctl);
  const float4* Wf = D.W[(D.S - 1) & 1];
  double ke = 0.0;
  unsigned long long kef = 0;  // E > 1: this thread's fixed-point sum for env kenv
  int kenv = env_of(D, kb < D.n ? kb : D.n - 1);
  const int klim = kend < own ? kend : own;
  for (int k = kb; k < klim; k += kstep) {
    const float4 xo = L.x[k];
    const float4 vo = L.v[k];
    const bool has = D.cinfo[k].y > 0;
    const float4 wf = has ? Wf[k] : vo;  // no contacts: no sweep wrote w
    const double dvx = has ? (double)wf.x - (double)vo.x : 0.0;
    const double dvy = has ? (double)wf.y - (double)vo.y : 0.0;
    const double dvz = has ? (double)wf.z - (double)vo.z : 0.0;
    if (!isfinite(dvx) || !isfinite(dvy) || !isfinite(dvz)) {
      const int slot = atomicAdd(&ctl->n_bad, 1);
      if (slot < kMaxBad) ctl->bad_uid[slot] = L.uid[k];
      if (D.bad) D.bad[k] = L.uid[k] + 1;
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
    const double v2 = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
    if (D.E == 1) {
      ke += v2;
    } else {
      const int e = env_of(D, k);
      if (e != kenv) {  // strided loops only
        if (kef) atomicAdd(D.ke_fix + kenv, kef);
        kef = 0;
        kenv = e;
      }
      kef += to_ke_fix(v2);
    }
  }
  double r = 0.0;
  if (D.E == 1)
    r = block_reduce<0>(ke, smd);
  else
    env_add_arr(D, kenv, kef, D.ke_fix);
  if (threadIdx.x == 0) D.part[blockIdx.x] = r;
}

// The step's StepReport(s), body momenta and commit, by ONE block after all
// integration blocks (nparts partials in D.part) are done: fixed-order
// kinetic-energy sum, reports, reset of the per-step words, state flip.
// nflags: sweep flags of the persistent launch to reset (its grid size; 0
// after the per-sweep kernels, whose k_finish grid is larger than bflags).
__device__ __forceinline__ void commit_step(const Dev& D, Ctl* ctl, int nparts, double* smd,
                                            int nflags) {
  const int cur = ctl->cur;
  const int step = ctl->step;
  double ke_tot = 0.0;
  if (D.E == 1) {
    double v0 = 0.0;
    // L2 loads (another block / kernel wrote them; not volatile, so a
    // thread's loads are in flight together)
    // (eight loads per round in flight; the sum keeps the strided order)
    int b = threadIdx.x;
    for (; b + 7 * static_cast<int>(blockDim.x) < nparts; b += 8 * blockDim.x) {
      double t[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) t[q] = __ldcg(&D.part[b + q * blockDim.x]);
#pragma unroll
      for (int q = 0; q < 8; ++q) v0 += t[q];
    }
    for (; b < nparts; b += blockDim.x) v0 += __ldcg(&D.part[b]);
    ke_tot = block_reduce<0>(v0, smd);
  }
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = *((volatile int*)&ctl->err);
  __syncthreads();
  const long long nbm = static_cast<long long>(D.E) * D.nb * 3;
  for (long long i = threadIdx.x; !D.env_kernel && i < nbm; i += blockDim.x) {
    const long long f = static_cast<long long>(__ldcg(&D.bm_fix[i]));
    if (!s_err) D.bm_out[static_cast<long long>(step) * nbm + i] = static_cast<double>(f) / kMomScale;
    D.bm_fix[i] = 0ull;
  }
  // the barrier words and sweep flags of a persistent launch are reset here
  // for the next one (every other block of it has finished)
  for (int b = threadIdx.x; b < nflags; b += blockDim.x)
    if (D.bflags) D.bflags[b] = 0u;
  if (D.E > 1 && !s_err && !D.env_kernel) {
    for (int e = threadIdx.x; e < D.E; e += blockDim.x) {
      volatile unsigned long long* kf = D.ke_fix + e;
      write_report(D, D.reports[static_cast<long long>(step) * D.E + e], D.acc + e,
                   static_cast<double>(static_cast<long long>(*kf)) / kKeScale);
      *kf = 0ull;
      acc_reset(D.acc + e);
    }
  }
  if (threadIdx.x == 0) {
    ctl->done_count = 0;
    ctl->bar_count = 0;
    ctl->bar_gen = 0;
    ctl->ccursor = static_cast<unsigned long long>(D.nrec0);
    if (s_err) return;  // an error was raised this step: no commit
    if (D.E == 1) {
      write_report(D, D.reports[step], D.acc, ke_tot);
      acc_reset(D.acc);
    }
    ctl->cur = cur ^ 1;
    if (D.resort) ctl->ucur ^= 1;
    ctl->step = step + 1;
  }
}

// Persistent kernels: integrate, then the last block to finish commits.
// This thread integrates particles kb, kb + kstep, ... < kend (its particles
// of the last sweep: another thread's w is not ordered before this read).
__device__ __forceinline__ void integrate_and_finish_range(const Dev& D, Ctl* ctl, int kb, int kend,
                                                           int kstep, double* smd, int* s_last) {
  integrate_range(D, ctl, kb, kend, kstep, smd, D.n_own);
  if (threadIdx.x == 0) {
    __threadfence();
    *s_last = atomicAdd(&ctl->done_count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!*s_last) return;
  __threadfence();
  commit_step(D, ctl, gridDim.x, smd, gridDim.x);
}

__device__ __forceinline__ void integrate_and_finish(const Dev& D, Ctl* ctl, int t0, int G,
                                                     double* smd, int* s_last) {
  integrate_and_finish_range(D, ctl, t0, D.n_own, G, smd, s_last);
}

// E > 1, large n: the per-env StepReports and body momenta of the step just
// committed, written by the whole grid after k_finish (the last block of
// k_finish alone would serialise 4096 envs x (report + 3 nb momenta)).
__global__ void __launch_bounds__(kBlock) k_env_reports(Dev D) {
  const Ctl* ctl = D.ctl;
  if (*((volatile const int*)&ctl->err)) return;  // nothing committed (k_batch_begin resets)
  const int step = ctl->step - 1;
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long G = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long e = t; e < D.E; e += G) {
    write_report(D, D.reports[static_cast<long long>(step) * D.E + e], D.acc + e,
                 static_cast<double>(static_cast<long long>(D.ke_fix[e])) / kKeScale);
    D.ke_fix[e] = 0ull;
    acc_reset(D.acc + e);
  }
  const long long nbm = static_cast<long long>(D.E) * D.nb * 3;
  for (long long i = t; i < nbm; i += G) {
    D.bm_out[static_cast<long long>(step) * nbm + i] =
        static_cast<double>(static_cast<long long>(D.bm_fix[i])) / kMomScale;
    D.bm_fix[i] = 0ull;
  }
}

// ===========================================================================
// Large-n drivers: one kernel per phase, one thread per element.
// ===========================================================================
template <bool DC>
__global__ void __launch_bounds__(kBlock) k_count(Dev D) {
  Ctl* ctl = D.ctl;
  if (ctl->err) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < live_n<DC>(D)) ph_count(D, ctl, i, D.key_morton != 0);
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

// tile_counts != 0: tile[] still holds the per-tile totals (no k_scan_top
// ran): each block sums its predecessors' totals itself — one launch fewer
// for up to a few thousand tiles
__global__ void __launch_bounds__(kBlock) k_scan_apply(Dev D, int tile_counts) {
  __shared__ uint32_t sm[32];
  if (D.ctl->err) return;
  ph_scan_apply(D, blockIdx.x, sm, tile_counts != 0);
}

template <bool DC>
__global__ void __launch_bounds__(kBlock) k_scatter(Dev D) {
  if (D.ctl->err) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < live_n<DC>(D)) ph_scatter(D, i);
  ph_zero_counts(D, i, static_cast<long long>(gridDim.x) * blockDim.x);
}

template <bool DC>
__global__ void __launch_bounds__(kBlock) k_resort(Dev D) {
  if (D.ctl->err) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < live_n<DC>(D)) ph_resort(D, D.ctl, k);
}

template <bool DC>
__global__ void __launch_bounds__(kBlock) k_fill(Dev D) {
  if (D.ctl->err) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < live_n<DC>(D)) ph_fill(D, D.ctl, k);
}

// NarrowSmem (> 48 KB) is dynamic shared memory: launch with sizeof(NarrowSmem)
extern __shared__ __align__(16) unsigned char g_dsmem[];

template <bool DC>
__global__ void __launch_bounds__(kNarrowBlock, GG_NARROW_MINB) k_narrow(Dev D) {
  // capacity-sized grid (slab graph): blocks past the owned particles leave
  if (DC && static_cast<int>(blockIdx.x * blockDim.x) >= live_own<true>(D)) return;
  NarrowSmemN& sm = *reinterpret_cast<NarrowSmemN*>(g_dsmem);
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  ph_contacts<NarrowSmemN, DC>(D, ctl, blockIdx.x * blockDim.x, blockDim.x, sm);
}

// One sweep, one thread per particle, no block barriers: the particle's
// head is requested first, then the error flag (nothing raises it during a
// sweep, so the exit is block-uniform) and the buffer selector — all in one
// round trip — and the accumulators are flushed warp by warp.
#ifndef GG_SWEEP_MINB
#define GG_SWEEP_MINB 4
#endif
template <bool DC>
__global__ void __launch_bounds__(kBlock, GG_SWEEP_MINB) k_sweep(Dev D, int s) {
  if (DC && static_cast<int>(blockIdx.x * blockDim.x) >= live_own<true>(D)) return;  // (slab graph)
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = k < live_own<DC>(D);
  SweepHead h;
  if (live) h.load(D, k);
  const Ctl* ctl = D.ctl;
  if (*((volatile const int*)&ctl->err) != 0) return;
  const float4* Win = (s == 0) ? layout(D, ctl).v : D.W[(s - 1) & 1];
  SweepAcc A;
  sweep_acc_init_nobar(D, A, k);
  if (live) sweep_particle_h(D, k, h, Win, D.W[s & 1], A);
  sweep_acc_flush_nobar(D, A);
}

// The last sweep integrates (GG_SWEEP_FIN, E == 1, one bed): the particle's
// symplectic Euler step exactly as integrate_range with w from registers, and
// the kinetic-energy partials in k_finish's order — a warp sum per 32
// particles, then the 8 warps of each 256-particle group added in warp order
// by the group's last warp (k_finish's block_reduce; warps past n add +0.0
// there, which leaves the sum unchanged) — so k_commit sums the same
// partials and every schedule stays bitwise identical.  Called by all lanes.
constexpr int kFinGroup = 256;  // = k_finish's block size
__device__ __forceinline__ void sweep_integrate(const Dev& D, int k, bool live, bool has, float4 wf) {
  Ctl* ctl = D.ctl;
  double v2 = 0.0;
  if (live) {
    const int cur = ctl->cur;
    const Layout L = layout(D, ctl);
    const float4 xo = L.x[k];
    const float4 vo = L.v[k];
    if (!has) wf = vo;
    const double dvx = has ? (double)wf.x - (double)vo.x : 0.0;
    const double dvy = has ? (double)wf.y - (double)vo.y : 0.0;
    const double dvz = has ? (double)wf.z - (double)vo.z : 0.0;
    if (!isfinite(dvx) || !isfinite(dvy) || !isfinite(dvz)) {
      const int slot = atomicAdd(&ctl->n_bad, 1);
      if (slot < kMaxBad) ctl->bad_uid[slot] = L.uid[k];
      if (D.bad) D.bad[k] = L.uid[k] + 1;
      raise_err(ctl, GG_ENONFINITE);
    }
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
    v2 = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
  }
  const double ws = warp_sum(v2);
  if ((threadIdx.x & 31) == 0) {
    constexpr int kW = kFinGroup / 32;
    const int w = k >> 5, g = w / kW;
    const int nwarps = (D.n_own + 31) >> 5;
    const int nw = min(kW, nwarps - g * kW);
    D.wpart[w] = ws;
    __threadfence();
    if (atomicAdd(&D.gcnt[g], 1u) == static_cast<unsigned>(nw - 1)) {
      __threadfence();
      double r = __ldcg(&D.wpart[g * kW]);
      for (int q = 1; q < nw; ++q) r += __ldcg(&D.wpart[g * kW + q]);
      D.part[g] = r;
      D.gcnt[g] = 0u;
    }
  }
}

// Record-major sweep (the large-n default).  A warp sweeps the 32 particles
// whose records the contact kernel allocated as one warp-contiguous block:
// record 0 of each particle sits at its fixed index, records 1.. of all 32
// owners are laid end to end in lane order from the warp base (= lane 0's CSR
// offset).  The warp walks those CSR records 32 at a time, ONE RECORD PER LANE
// (a particle with six contacts no longer keeps 31 lanes idle), the owner of
// record r found by a 5-step shuffle search over the lanes' inclusive record
// counts, and the owner's w fetched by shuffle.  Each lane's impulse goes to
// shared memory and the owner adds its records' impulses in record order —
// the same float64 sums, in the same order, as sweep_particle_h, so every
// schedule stays bitwise identical.  Latency: head -> {own w, partner 0, the
// first chunk of records} -> partners of the chunk, whatever the counts (the
// per-particle loop paid two dependent round trips per extra record).
// Warps whose lanes belong to two envs take the per-particle path.
#ifndef GG_SWEEP_BLOCK
#define GG_SWEEP_BLOCK 32
#endif
#ifndef GG_SWEEP_RM
#define GG_SWEEP_RM 1
#endif
#ifndef GG_RM_MAXT
#define GG_RM_MAXT 64
#endif
constexpr int kSweepBlockK = GG_SWEEP_BLOCK;
static_assert(kSweepBlockK % 32 == 0 && kSweepBlockK <= kBlock, "sweep block: whole warps");
#ifndef GG_SWEEP_RM_MINB
#define GG_SWEEP_RM_MINB 32
#endif
template <bool DC, bool FIN = false>
__global__ void __launch_bounds__(kSweepBlockK, GG_SWEEP_RM_MINB) k_sweep_rm(Dev D, int s) {
  if (DC && static_cast<int>(blockIdx.x * blockDim.x) >= live_own<true>(D)) return;  // (slab graph)
  static_assert(kFixedSlots == 1, "record-major sweep: one fixed record slot per particle");
  __shared__ double s_imp[kSweepBlockK / 32][3][32];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const bool live = k < live_own<DC>(D);
  L2Pol pol;
  pol.init();
  SweepHead h;
  h.ci = make_int2(0, 0);
  if (live) {
    h.ci = ld_hint(&D.cinfo[k], pol.first, kHintRec);
    h.g[0] = ld_hint(&D.cgeo[k], pol.first, kHintRec);
    h.j[0] = ld_hint(&D.coth[k], pol.first, kHintRec);
  }
  // the warp's CSR region is at a fixed address (contacts_finish): its first
  // 32 records are requested together with the heads
  const long long wb = D.nrec0 + static_cast<long long>(k >> 5) * D.wcap;
#ifndef GG_SWEEP_PREFETCH
#define GG_SWEEP_PREFETCH 1
#endif
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
  int j = kNullContact;
  if (GG_SWEEP_PREFETCH) {
    g = ld_hint(&D.cgeo[wb + lane], pol.first, kHintRec);
    j = ld_hint(&D.coth[wb + lane], pol.first, kHintRec);
  }
  const Ctl* ctl = D.ctl;
#ifndef GG_FIN_PREFETCH
#define GG_FIN_PREFETCH 1
#endif
  if (FIN && GG_FIN_PREFETCH && live) {  // the integration's x, v into L1 while the sweep runs
    const Layout L = layout(D, ctl);
#if defined(GG_FIN_L2) && GG_FIN_L2
    asm volatile("prefetch.global.L2 [%0];" ::"l"(L.x + k));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(L.v + k));
#else
    asm volatile("prefetch.global.L1 [%0];" ::"l"(L.x + k));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(L.v + k));
#endif
  }
  if (*((volatile const int*)&ctl->err) != 0) return;  // uniform: nothing raises during sweeps
  const float4* Win = (s == 0) ? layout(D, ctl).v : D.W[(s - 1) & 1];
  float4* Wout = D.W[s & 1];
  SweepAcc A;
  sweep_acc_init_nobar(D, A, k);
  int e0 = 0;
  if (D.E > 1 && !warp_env_uniform(env_of(D, live ? k : D.n - 1), &e0)) {
    if (live) sweep_particle_h(D, k, h, Win, Wout, A);
    sweep_acc_flush_nobar(D, A);
    if (FIN) sweep_integrate(D, k, live, h.ci.y > 0, h.ci.y > 0 ? Wout[k] : make_float4(0.f, 0.f, 0.f, 0.f));
    return;
  }
  const int c = h.ci.y;
  const uint32_t m = c > 1 ? static_cast<uint32_t>(c - 1) : 0u;  // this owner's CSR records
  uint32_t incl = m;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);  // CSR records of the warp
  // a densely packed warp (more than GG_RM_MAXT CSR records: every lane has
  // several) keeps its lanes busy record by record — the per-particle loop
  // is cheaper there than chunk after chunk of owner searches and sums
  if (T > GG_RM_MAXT) {
    if (live) sweep_particle_h(D, k, h, Win, Wout, A);
    sweep_acc_flush_nobar(D, A);
    if (FIN) sweep_integrate(D, k, live, c > 0, c > 0 ? Wout[k] : make_float4(0.f, 0.f, 0.f, 0.f));
    return;
  }
  const uint32_t excl = incl - m;
  if (!GG_SWEEP_PREFETCH && static_cast<uint32_t>(lane) < T) {
    g = D.cgeo[wb + lane];
    j = D.coth[wb + lane];
  }
  if (static_cast<uint32_t>(lane) >= T) j = kNullContact;  // past the warp's records
  // requested together: own w, record 0's partner, the first chunk's partners
  float4 wf = make_float4(0.f, 0.f, 0.f, 0.f), q0 = wf;
  const bool has0 = c > 0 && h.j[0] != kNullContact;
  if (c > 0) wf = ld_hint(&Win[k], pol.last, kHintW);
  if (has0) q0 = (h.j[0] >= 0) ? ld_hint(&Win[h.j[0]], pol.last, kHintW) : D.cvb[k];
  // ... and the first chunk's partners, in the same round trip
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j != kNullContact) q = (j >= 0) ? ld_hint(&Win[j], pol.last, kHintW) : D.cvb[wb + lane];
  double ax = 0.0, ay = 0.0, az = 0.0;
  if (has0) contact_impulse(D, wf.x, wf.y, wf.z, h.g[0], h.j[0], q0, ax, ay, az, A);
  for (uint32_t cb = 0; cb < T; cb += 32) {
    const uint32_t r = cb + lane;
    const bool mine = j != kNullContact;  // (r < T: j is null past the records)
    // this chunk's record and partner; the next chunk's requested now
    const float4 gc = g, qc = q;
    const int jc = j;
    if (cb + 32 < T) {
      j = kNullContact;
      if (cb + 32 + lane < T) {
        g = ld_hint(&D.cgeo[wb + cb + 32 + lane], pol.first, kHintRec);
        j = ld_hint(&D.coth[wb + cb + 32 + lane], pol.first, kHintRec);
      }
      if (j != kNullContact)
        q = (j >= 0) ? ld_hint(&Win[j], pol.last, kHintW) : D.cvb[wb + cb + 32 + lane];
    }
    // owner of record r: the first lane whose inclusive count exceeds r
    int o = 0;
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, incl, o + st - 1);
      if (v <= r) o += st;
    }
    o = o < 31 ? o : 31;
    const float owx = __shfl_sync(0xffffffffu, wf.x, o);
    const float owy = __shfl_sync(0xffffffffu, wf.y, o);
    const float owz = __shfl_sync(0xffffffffu, wf.z, o);
    double ix = 0.0, iy = 0.0, iz = 0.0;
    if (GG_MINE_PRED)
      contact_impulse(D, owx, owy, owz, gc, jc, qc, ix, iy, iz, A, mine);
    else if (mine)
      contact_impulse(D, owx, owy, owz, gc, jc, qc, ix, iy, iz, A);
    s_imp[wi][0][lane] = ix;
    s_imp[wi][1][lane] = iy;
    s_imp[wi][2][lane] = iz;
    __syncwarp();
    // the owner adds its records of this chunk in record order (a null
    // record adds +0.0, which leaves a sum that started at +0.0 unchanged)
    const uint32_t a0 = excl > cb ? excl : cb;
    const uint32_t a1 = incl < cb + 32 ? incl : cb + 32;
    owner_sums(s_imp[wi], a0, a1, cb, ax, ay, az);
    __syncwarp();
  }
  const float4 wn = make_float4(static_cast<float>(static_cast<double>(wf.x) + ax),
                                 static_cast<float>(static_cast<double>(wf.y) + ay),
                                 static_cast<float>(static_cast<double>(wf.z) + az), 0.f);
  if (c > 0 && !FIN) st_hint(&Wout[k], wn, pol.last, kHintW);
  sweep_acc_flush_nobar(D, A);
  if (FIN) sweep_integrate(D, k, live, c > 0, wn);
}

// ONE_LOOP sweep (its own kernel: the inline collision test would cost the
// record-reading sweep its registers)
__global__ void __launch_bounds__(kBlock) k_sweep_oneloop(Dev D, int s) {
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  __shared__ double smd[32];
  const Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const Layout L = layout(D, ctl);
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  SweepAcc A;
  sweep_acc_init(D, A, sbm, k);
  const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
  if (k < D.n_own) {
    sweep_acc_env(D, A, k);
    if (D.cinfo[k].y > 0) {  // same skip as sweep_particle
      const float4 wf = Win[k];
      double ax = 0.0, ay = 0.0, az = 0.0;
      sweep_oneloop(D, k, Win, wf.x, wf.y, wf.z, ax, ay, az, A);
      D.W[s & 1][k] = make_float4(static_cast<float>(static_cast<double>(wf.x) + ax),
                                  static_cast<float>(static_cast<double>(wf.y) + ay),
                                  static_cast<float>(static_cast<double>(wf.z) + az), 0.f);
    }
  }
  sweep_acc_flush(D, A, smd);
}

// Large-n integration: a pure stream (x, v, cinfo, w in; x, v out), one
// particle per thread, a kinetic-energy partial per block; k_commit (one
// block) then sums the partials in fixed order and commits the step.
template <bool DC>
__global__ void __launch_bounds__(kBlock) k_finish(Dev D) {
  __shared__ double smd[32];
  Ctl* ctl = D.ctl;
  if (block_should_exit(ctl)) return;
  const int own = live_own<DC>(D);
  if (DC && static_cast<int>(blockIdx.x * blockDim.x) >= own) {  // (slab graph: capacity grid)
    if (threadIdx.x == 0) D.part[blockIdx.x] = 0.0;
    return;
  }
  integrate_range(D, ctl, blockIdx.x * blockDim.x + threadIdx.x, own, gridDim.x * blockDim.x, smd, own);
}

__global__ void __launch_bounds__(kBlock) k_commit(Dev D, int nparts) {
  __shared__ double smd[32];
  commit_step(D, D.ctl, nparts, smd, 0);
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
  const int err = grid_barrier(ctl, target);
  stamp(D, ts);
  return err == 0;
}

__global__ void __launch_bounds__(kBlock, 2) k_step_fused(Dev D) {
  NarrowSmem& sm = *reinterpret_cast<NarrowSmem*>(g_dsmem);
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
  const int ntiles = static_cast<int>((D.nh_tot + kScanTile - 1) / kScanTile);
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
  // narrowphase + bodies; the sweeps below use the same particle -> block
  // map, so a particle's records were written by its own block (visible
  // after the __syncthreads in sweep_acc_init)
  // one particle per thread when G >= n: particle t0 (its contacts, sweeps
  // and integration all on this thread)
  const bool one_per_thread = G >= D.n;
  const int kr = t0;
  const bool kr_live = one_per_thread && kr < D.n_own;
  if (ok) {
    for (int base = blockIdx.x * blockDim.x; base < D.n; base += G)
      ph_contacts<NarrowSmem, false, (GG_FUSED_CULL != 0), false>(D, ctl, base, blockDim.x, sm);
  }
  stamp(D, ts);
  // split schedule: k_solve_cluster runs the sweeps and the commit (and
  // resets the barrier words this launch used)
  if (D.fused_stop) return;
  const Layout L = layout(D, ctl);
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  SweepAcc A;
  sweep_acc_init(D, A, sbm, t0);
  if (one_per_thread && gridDim.x <= kMaxFusedBlocks) {
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
    const bool rm = GG_FUSED_RM && D.sweep_barrier;  // record-major register sweeps
    // the chunk impulses live in the contact phase's pass queue (free now)
    static_assert(sizeof(NarrowSmem::pass) >= sizeof(double) * 3 * 32 * (kBlock / 32), "impulse scratch");
    double(*s_fimp)[3][32] = reinterpret_cast<double(*)[3][32]>(&sm.pass[0][0]);
    RegChunks RK;
    if (rm) {
      RK.load(D, kr, ok && kr_live, kr_live ? L.v[kr] : make_float4(0.f, 0.f, 0.f, 0.f));
    } else if (ok && kr_live) {
      RC.load(D, kr, L.v[kr]);
    }
    if (!D.sweep_barrier) {  // neighbour-block list for the flag-synchronised sweeps
      for (int w = threadIdx.x; w < kMaxFusedBlocks / 32; w += blockDim.x) s_nbmask[w] = 0u;
      __syncthreads();
      {
        for (int sl = 0; sl < RC.c; ++sl) {
          const int j = sl < kRegSlots ? RC.j[sl] : D.coth[RC.off + sl - 1];
          if (j >= 0 && j != kNullContact) {
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
    }
    unsigned* flags = D.bflags;
    for (int s = 0; s < D.S; ++s) {
      if (s > 0 && D.sweep_barrier) {
        ok = barrier_ok(D, ctl, target, &s_flag, ts) && ok;
      } else if (s > 0) {
        for (int q = threadIdx.x; q < s_nnb; q += blockDim.x) {
          unsigned v;
          do {
            asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flags + s_nblist[q]) : "memory");
          } while (static_cast<int>(v - static_cast<unsigned>(s)) < 0);
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flags + s_nblist[q]) : "memory");
        }
        // (the acquire loads above invalidated this SM's L1: CCTL.IVALL)
        __syncthreads();
        if (threadIdx.x == 0) s_flag = *((volatile int*)&ctl->err);
        __syncthreads();
        ok = ok && s_flag == 0;
        stamp(D, ts);
      }
      if (rm) {
        if (ok) RK.sweep(D, kr, kr_live, (s == 0) ? L.v : D.W[(s - 1) & 1], D.W[s & 1], A, s_fimp[threadIdx.x >> 5]);
      } else if (ok && kr_live) {
        RC.sweep(D, kr, (s == 0) ? L.v : D.W[(s - 1) & 1], D.W[s & 1], A);
      }
      if (!D.sweep_barrier) {
        __syncthreads();
        if (threadIdx.x == 0)
          asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(s + 1) : "memory");
      }
    }
  } else {
    for (int s = 0; s < D.S; ++s) {
      if (s > 0) ok = barrier_ok(D, ctl, target, &s_flag, ts) && ok;
      if (ok) {
        const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
        float4* Wout = D.W[s & 1];
        for (int k = t0; k < D.n_own; k += G) sweep_particle(D, k, Win, Wout, A);
      }
    }
  }
  stamp(D, ts);
  sweep_acc_flush(D, A, sm.d);
  // integrate exactly the particles this thread swept (t0, t0 + G, ...): the
  // last sweep's w of another block's particle is not ordered before the read
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
  sweep_acc_init(D, A, sbm, t0);
  for (int s = 0; s < D.S; ++s) {
    if (s > 0) grid_barrier(ctl, gridDim.x * static_cast<unsigned>(s));
    const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
    float4* Wout = D.W[s & 1];
    for (int k = t0; k < D.n_own; k += G) sweep_particle(D, k, Win, Wout, A);
  }
  sweep_acc_flush(D, A, smd);
  integrate_and_finish(D, ctl, t0, G, smd, &s_last);
}

// ---------------------------------------------------------------------------
// Large-n solve (mode 8, the auto choice when the step is not fused): the S
// sweeps, the integration and the report in ONE cooperative persistent
// launch (grid = co-resident blocks of kStageBlock threads, one per SM).
//
// Block b owns particles [b P, (b + 1) P), cut into chunks of 32 consecutive
// particles; warp w takes chunks w, w + 32, ...  Before sweep 0 the block
// copies its contact records (e1, psi, partner) and each record's owner lane
// into shared memory, in particle order, so every sweep reads them from
// there and gathers only w (own + partners, L2-resident) from global memory.
//
// A sweep is RECORD-parallel: the chunk's records are laid end to end and
// each lane evaluates one record's impulse (owner w by shuffle from the owner
// lane, partner w gathered); then each owner lane adds its records' impulses
// in record order, fetched by shuffle, and writes its w.  The per-particle
// loop of k_sweep runs as long as the busiest particle of the warp (SIMD
// efficiency ~13 of 32 lanes, ncu); here every lane evaluates a record.
// The impulse arithmetic and the per-owner accumulation order are those of
// sweep_particle_h (the owner adds its impulses to 0.0 in record order), so
// the result is bitwise that of the other schedules.  Records beyond the
// block's shared-memory capacity, and body surface velocities, are read
// from global memory.
// ---------------------------------------------------------------------------
constexpr int kStageBlock = 1024;
constexpr int kStageWarps = kStageBlock / 32;
constexpr int kStageSat = 255;  // a count this large is re-read from cinfo
constexpr int kStageMaxGrid = 511;  // blocks of k_solve_staged (one per SM)

// shared-memory layout of k_solve_staged (dynamic): counts[P] (u8), chunk
// record bases[ceil(P/32)] (u32), then per record float4 (e1, psi), int
// partner and u8 owner lane
__device__ __host__ __forceinline__ long long stage_head_bytes(long long pb) {
  const long long cnt = (pb + 15) & ~15ll;
  const long long base = (((pb + 31) / 32) * 4 + 15) & ~15ll;
  return cnt + base;
}
constexpr int kStageRecBytes = 16 + 4 + 1;

struct StageImp {
  double x[kStageWarps][32], y[kStageWarps][32], z[kStageWarps][32];  // per-warp impulse exchange
};

// First particle k of [lo, hi) whose exclusive work prefix E(k) reaches t,
// where E(lo) = e0 and a particle weighs its record count + 1 (block-wide;
// hi if none).  E is non-decreasing, so the first round with a hit decides.
__device__ __forceinline__ int stage_locate(const Dev& D, int lo, int hi, unsigned long long e0,
                                            unsigned long long t, uint32_t* smu, int* s_hit) {
  if (threadIdx.x == 0) *s_hit = hi;
  __syncthreads();
  unsigned long long run = e0;
  for (int base = lo; base < hi; base += kStageBlock) {
    const int k = base + static_cast<int>(threadIdx.x);
    const uint32_t w = k < hi ? static_cast<uint32_t>(D.cinfo[k].y) + 1u : 0u;
    uint32_t total;
    const uint32_t ex = block_excl_scan_u32(w, smu, &total);
    if (k < hi && run + ex >= t) atomicMin(s_hit, k);
    __syncthreads();
    if (*s_hit < hi) break;  // block-uniform
    run += total;
  }
  const int r = *s_hit;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kStageBlock, 1) k_solve_staged(Dev D) {
  __shared__ double smd[32];
  __shared__ uint32_t smu[32];
  __shared__ int s_last, s_hit, s_next[2];
  __shared__ unsigned long long s_pre[kStageMaxGrid + 1];
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  __shared__ StageImp simp;
  Ctl* ctl = D.ctl;
  int ts = 0;
  stamp(D, ts);
  if (block_should_exit(ctl)) return;  // uniform: err cannot change before the last barrier
  const int G = static_cast<int>(gridDim.x);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ---- plan: contiguous particle ranges of equal work ------------------------
  // (records + particles; the grid barrier of every sweep waits for the
  // busiest block).  Work of fixed segments, then each block locates its
  // bounds inside the segments that contain them.
  const int S0 = (D.n_own + G - 1) / G;
  {
    const int lo = min(static_cast<int>(blockIdx.x) * S0, D.n_own), hi = min(lo + S0, D.n_own);
    unsigned long long w = 0;
    for (int k = lo + static_cast<int>(threadIdx.x); k < hi; k += kStageBlock)
      w += static_cast<unsigned long long>(D.cinfo[k].y) + 1ull;
    w = block_sum_u64(w, reinterpret_cast<unsigned long long*>(smd));
    if (threadIdx.x == 0) D.stage_seg[blockIdx.x] = w;
  }
  grid_barrier(ctl, static_cast<unsigned>(G));
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int b = 0; b < G; ++b) {
      s_pre[b] = acc;
      acc += *((volatile unsigned long long*)&D.stage_seg[b]);
    }
    s_pre[G] = acc;
  }
  __syncthreads();
  const unsigned long long Wtot = s_pre[G];
  auto bound = [&](int b) -> int {
    if (b <= 0) return 0;
    if (b >= G) return D.n_own;
    const unsigned long long t = (Wtot * static_cast<unsigned long long>(b)) / static_cast<unsigned long long>(G);
    int j = 0;  // the segment holding t: the last with prefix <= t
    while (j + 1 < G && s_pre[j + 1] <= t) ++j;
    const int lo = min(j * S0, D.n_own), hi = min(lo + S0, D.n_own);
    return stage_locate(D, lo, hi, s_pre[j], t, smu, &s_hit);
  };
  const int kb = bound(static_cast<int>(blockIdx.x));
  const int ke = bound(static_cast<int>(blockIdx.x) + 1);
  const int P = ke - kb;
  // shared-memory layout for this block's P particles
  const long long head = stage_head_bytes(P);
  const long long capl = (static_cast<long long>(D.stage_smem) - head) / kStageRecBytes;
  const uint32_t CAP = capl > 0 ? static_cast<uint32_t>(capl) : 0u;
  const int nchunk = (P + 31) / 32;
  uint8_t* scnt = g_dsmem;
  uint32_t* sbase = reinterpret_cast<uint32_t*>(g_dsmem + ((P + 15) & ~15));
  float4* sg = reinterpret_cast<float4*>(g_dsmem + head);
  int* sj = reinterpret_cast<int*>(sg + CAP);
  uint8_t* sown = reinterpret_cast<uint8_t*>(sj + CAP);
  const bool counts_fit = head <= static_cast<long long>(D.stage_smem);
  const Layout L = layout(D, ctl);
  // ---- stage: counts, chunk bases, records (block scans in particle order) --
  uint32_t run = 0;  // records of the earlier rounds
  for (int m = 0; counts_fit && m * kStageBlock < P; ++m) {
    const int k = kb + m * kStageBlock + static_cast<int>(threadIdx.x);
    int2 ci = make_int2(0, 0);
    if (k < ke) {
      ci = D.cinfo[k];
      scnt[k - kb] = static_cast<uint8_t>(ci.y < kStageSat ? ci.y : kStageSat);
    }
    uint32_t total;
    const uint32_t ex = block_excl_scan_u32(static_cast<uint32_t>(ci.y), smu, &total) + run;
    const int chunk = m * kStageWarps + warp;
    if (lane == 0 && chunk < nchunk) sbase[chunk] = ex;
    for (int i = 0; i < ci.y && ex + i < CAP; ++i) {
      const long long idx = ridx(D, k, ci.x, i);
      sg[ex + i] = D.cgeo[idx];
      sj[ex + i] = D.coth[idx];
      sown[ex + i] = static_cast<uint8_t>(lane);
    }
    run += total;
  }
  SweepAcc A;
  sweep_acc_init(D, A, sbm, kb + static_cast<int>(threadIdx.x), kb);  // (__syncthreads: staging visible)
  double* ibx = simp.x[warp];
  double* iby = simp.y[warp];
  double* ibz = simp.z[warp];
  stamp(D, ts);
  // ---- sweeps ---------------------------------------------------------------
  // chunk counters, one per sweep parity: sweep s claims from s_next[s & 1]
  // and clears the other one, which no warp can still be using (every warp
  // left sweep s - 1 before the grid barrier)
  if (threadIdx.x == 0) s_next[0] = s_next[1] = 0;
  __syncthreads();
  for (int s = 0; s < D.S; ++s) {
    if (s > 0) {
      grid_barrier(ctl, static_cast<unsigned>(G) * static_cast<unsigned>(s + 1));
      stamp(D, ts);
    }
    if (threadIdx.x == 0) s_next[(s + 1) & 1] = 0;
    const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
    float4* Wout = D.W[s & 1];
    for (;;) {
      // chunks are claimed dynamically: warps of one block finish together
      int ch = 0;
      if (lane == 0) ch = atomicAdd(&s_next[s & 1], 1);
      ch = __shfl_sync(0xffffffffu, ch, 0);
      if (ch >= nchunk) break;
      const int k = kb + ch * 32 + lane;
      const bool live = k < ke;
      int c = (live && counts_fit) ? scnt[k - kb] : 0;
      const uint32_t base = counts_fit ? sbase[ch] : 0u;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int T = __shfl_sync(0xffffffffu, incl, 31);
      // staged records cover [base, base + T) unless a count saturated or
      // the chunk runs past the capacity: then records come from global
      // memory (record index from cinfo, owner by a search over the prefix)
      const bool glob = !counts_fit || __any_sync(0xffffffffu, c == kStageSat) ||
                        base + static_cast<uint32_t>(T) > CAP;
      int cix = 0;
      if (glob) {
        c = 0;
        if (live) {
          const int2 ci = D.cinfo[k];
          c = ci.y;
          cix = ci.x;
        }
        incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        T = __shfl_sync(0xffffffffu, incl, 31);
      }
      if (T == 0) continue;
      const int excl = incl - c;
      const float4 wf = (live && c > 0) ? Win[k] : make_float4(0.f, 0.f, 0.f, 0.f);
      double ax = 0.0, ay = 0.0, az = 0.0;  // this lane's particle: its impulses in record order
      for (int rb = 0; rb < T; rb += 32) {
        const int ri = rb + lane;  // this lane's record (chunk-relative)
        int o = 0;
        if (glob) {  // owner lane: the number of lanes whose records end at or before ri
#pragma unroll
          for (int b = 16; b >= 1; b >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, o + b - 1);
            if (v <= ri) o += b;
          }
        }
        const int oex = __shfl_sync(0xffffffffu, excl, min(o, 31));
        const int ocx = __shfl_sync(0xffffffffu, cix, min(o, 31));
        if (ri < T) {
          double ix = 0.0, iy = 0.0, iz = 0.0;
          float4 g;
          int j;
          long long gidx = -1;
          if (!glob) {
            const uint32_t r = base + static_cast<uint32_t>(ri);
            g = sg[r];
            j = sj[r];
            o = sown[r];
          }
          const int ko = kb + ch * 32 + o;
          if (glob) {
            gidx = ridx(D, ko, ocx, ri - oex);
            g = D.cgeo[gidx];
            j = D.coth[gidx];
          }
          if (j != kNullContact) {
            const float4 wo = Win[ko];
            float4 q;
            if (j >= 0) {
              q = Win[j];
            } else {
              if (gidx < 0) {
                int first = 0;  // the owner's first record in this chunk
                for (int l = 0; l < o; ++l) first += scnt[ko - o + l - kb];
                gidx = ridx(D, ko, D.cinfo[ko].x, ri - first);
              }
              q = D.cvb[gidx];
            }
            sweep_acc_env(D, A, ko);
            contact_impulse(D, wo.x, wo.y, wo.z, g, j, q, ix, iy, iz, A);
          }
          ibx[lane] = ix;
          iby[lane] = iy;
          ibz[lane] = iz;
        }
        __syncwarp();
        // each owner adds its records of this batch in record order
        const int lo = max(excl - rb, 0), hi = min(incl - rb, 32);
        for (int u = lo; u < hi; ++u) {
          ax += ibx[u];
          ay += iby[u];
          az += ibz[u];
        }
        __syncwarp();
      }
      if (live && c > 0)
        Wout[k] = make_float4(static_cast<float>(static_cast<double>(wf.x) + ax),
                              static_cast<float>(static_cast<double>(wf.y) + ay),
                              static_cast<float>(static_cast<double>(wf.z) + az), 0.f);
    }
  }
  stamp(D, ts);
  sweep_acc_flush(D, A, smd);  // (its __syncthreads orders the block's last-sweep writes)
  // the block's particles (its warps wrote their last-sweep w)
  integrate_and_finish_range(D, ctl, kb + static_cast<int>(threadIdx.x), ke, kStageBlock, smd, &s_last);
  stamp(D, ts);
}

// ---------------------------------------------------------------------------
// Small-n solve on ONE thread-block cluster (16 CTAs x 1024 threads, one CTA
// per SM): the S Jacobi sweeps are separated by the hardware cluster barrier
// (barrier.cluster arrive.release / wait.acquire, ~0.2 us, invalidates L1)
// instead of a grid barrier through L2 atomics (~4 us).  The sweep work of a
// small bed (tens of thousands of contacts) fits 16 SMs easily; the
// synchronisation was the cost.  Then integrate + StepReport + commit.
// ---------------------------------------------------------------------------
constexpr int kClusterCTAs = 16;
constexpr int kClusterBlock = 1024;

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __launch_bounds__(kClusterBlock, 1) k_solve_cluster(Dev D) {
  __shared__ double smd[32];
  __shared__ int s_last;
  __shared__ unsigned long long sbm[kSmemBodies * 3];
  Ctl* ctl = D.ctl;
  // an error raised by the contact phase (uniform over the cluster: set by an
  // earlier kernel) skips the sweeps; the finish still runs so the barrier
  // words of k_step_fused are reset and nothing is committed
  const bool ok = !block_should_exit(ctl);
  const Layout L = layout(D, ctl);
  const int G = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  SweepAcc A;
  sweep_acc_init(D, A, sbm, t0);
  for (int s = 0; ok && s < D.S; ++s) {
    if (s > 0) cluster_barrier();
    const float4* Win = (s == 0) ? L.v : D.W[(s - 1) & 1];
    float4* Wout = D.W[s & 1];
    for (int k = t0; k < D.n_own; k += G) sweep_particle(D, k, Win, Wout, A);
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

// Goal-box statistics per env on the committed state (bulldozer_reward,
// GoalBox.contains / .distance, envs.py:39-70): one block per env, fixed-order
// reduction.  reward = sum(inside ? 100/n : -d/n); inside = particles in the box.
__global__ void __launch_bounds__(kBlock) k_env_box(Dev D, double lx, double ly, double lz,
                                                    double hx, double hy, double hz,
                                                    double* __restrict__ reward,
                                                    long long* __restrict__ inside) {
  __shared__ double smd[32];
  __shared__ unsigned long long smu[32];
  const int env = blockIdx.x;
  const float4* X = D.X[D.ctl->cur];
  const double inv_n = 100.0 / static_cast<double>(D.ne);
  const double dn = static_cast<double>(D.ne);
  double acc = 0.0;
  unsigned long long cnt = 0;
  for (int q = threadIdx.x; q < D.ne; q += blockDim.x) {
    const float4 p = X[static_cast<long long>(env) * D.ne + q];
    const double px = p.x, py = p.y, pz = p.z;
    const bool in = px >= lx && py >= ly && pz >= lz && px <= hx && py <= hy && pz <= hz;
    if (in) {
      acc += inv_n;
      ++cnt;
    } else {
      const double dx = nmax(nmax(__dsub_rn(lx, px), __dsub_rn(px, hx)), 0.0);
      const double dy = nmax(nmax(__dsub_rn(ly, py), __dsub_rn(py, hy)), 0.0);
      const double dz = nmax(nmax(__dsub_rn(lz, pz), __dsub_rn(pz, hz)), 0.0);
      acc += -__ddiv_rn(norm3(dx, dy, dz), dn);
    }
  }
  const double r = block_reduce<0>(acc, smd);
  const unsigned long long c = block_sum_u64(cnt, smu);
  if (threadIdx.x == 0) {
    if (reward) reward[env] = r;
    if (inside) inside[env] = static_cast<long long>(c);
  }
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
