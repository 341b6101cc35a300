// gg_abi.cu — context, buffers, the step schedule (CUDA graph) and the
// extern "C" entry points declared in include/granusim_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gg_kernels.cuh"
#include "gg_slab.cuh"
#include "gg_render.cuh"
#include "gg_bake.cuh"
#include "gg_l1.cuh"
#include "gg_drive.cuh"

using namespace gg;

struct gg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  gg_params P{};
  long long n = 0, n_h = 0;  // n = E * ne particles; n_h buckets per env
  int E = 1;                 // independent environments (segments)
  long long ne = 0;          // particles per env
  int K = 16;
  int max_bodies = 0;
  int nblocks = 0;
  int ntiles = 0;
  Dev D{};
  std::string err;
  long long launches = 0;

  // batch buffers
  int batch_cap = 0;
  gg_body* d_bodies = nullptr;
  gg_body* h_bodies = nullptr;  // pinned staging
  gg_report* d_reports = nullptr;
  double* d_bm = nullptr;
  Ctl* h_ctl = nullptr;  // pinned
  int last_batch = 0;
  int last_nb = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  // grids
  std::vector<DevGrid> grids;
  DevGrid* d_grids = nullptr;
  int d_grids_cap = 0;
  double* d_gvals = nullptr;
  long long gvals_cap = 0, gvals_used = 0;

  // staging for f64 state / taps
  double* d_stage = nullptr;  // 6n doubles

  // contact taps read UID[cur ^ 1] after gg_detect (uncommitted sort)
  bool tap_uncommitted = false;

  // bench helpers
  void* flush_buf = nullptr;
  long long flush_bytes = 0;
  std::vector<cudaEvent_t> evpool;

  // graphs of one step: [0] plain, [1] re-sort first
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  bool graph_dirty = true;
  int solve_grid = 0;      // co-resident blocks of k_solve
  int resort_every = 32;   // physical re-sort period (steps; particles move << a cell per step)
  int solve_mode = 0;      // 0 auto, 1 coop solve, 2 plain persistent solve, 3 per-sweep, 4 fused step
  int pipeline = 0;        // PipelineMode of the captured graphs (GG_MODE_*)
  int fused_grid = 0;      // co-resident blocks of k_step_fused
  int staged_grid = 0;     // co-resident blocks of k_solve_staged (one per SM)
  int nflags = 1;          // length of D.bflags
  size_t staged_smem = 0;  // its dynamic shared memory per block
  bool cluster_ok = false; // a 16-CTA cluster of k_solve_cluster can be resident
  long long since_resort = 1 << 30;  // force a re-sort after upload

  std::vector<void*> owned;  // fixed-size allocations freed at destroy

  // slab mode (gg_slab_*): owned particles [0, n_own), ghosts [n_own, n_cur)
  bool slab_on = false;
  SlabCfg slab{};
  long long n_own = 0, n_cur = 0;
  long long ghost_in[2] = {0, 0};   // ghosts received from lo / hi
  long long ghost_out[2] = {0, 0};  // boundary particles sent to lo / hi
  unsigned long long* d_scnt = nullptr;  // [4] slab counters
  unsigned long long* d_x = nullptr;     // [kXCount] device-side exchange counts
  unsigned long long* h_x = nullptr;     // pinned mirror
  int* d_n = nullptr;                    // [2] {n, n_own} of a graph-replayed slab step
  unsigned long long* d_step = nullptr;  // slab steps replayed (the mailbox sequence numbers)
  // slab step graphs: [batched][re-sort] (batched: without the per-step
  // batch reset, replayed K times after one k_batch_begin)
  cudaGraphExec_t sgexec[4] = {nullptr, nullptr, nullptr, nullptr};
  unsigned long long sgkey = 0;          // what the slab graphs were built for
  unsigned long long pgen = 0;           // bumped by every parameter / schedule change
  unsigned long long* h_scnt = nullptr;  // pinned mirror
  int* d_holes = nullptr;
  int* d_movers = nullptr;
  int* d_map[2] = {nullptr, nullptr};
  // peer-memory halo (gg_slab_mailbox / gg_slab_connect / gg_slab_halo_p2p)
  Mailbox* mbox = nullptr;
  long long mbox_cap = 0;
  Mailbox* peer[2] = {nullptr, nullptr};
  bool peer_ipc[2] = {false, false};  // opened with cudaIpcOpenMemHandle

  // device-resident body drivers (gg_drive_*), one per body slot
  struct DriveSlot {
    int kind = 0;  // 0 none, 1 fixed, 2 track, 3 chain
    gg_body* d_fixed = nullptr;
    double* d_state = nullptr;  // track: [3][E] x, y, theta; chain: [E][J] q
    double* d_action = nullptr; // track: [E][2]; chain: [E][J] joint rate commands
    DriveTrack P{};
    DriveChain C{};
  };
  std::vector<DriveSlot> drive;
};

namespace {

#define GG_STR2(x) #x
#define GG_STR(x) GG_STR2(x)
const char* kBuildInfo = "granusim_b200 sm_100a nvcc " GG_STR(__CUDACC_VER_MAJOR__) "." GG_STR(__CUDACC_VER_MINOR__);

int fail(gg_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(gg_ctx* c, cudaError_t e, const char* where) {
  return fail(c, GG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                              \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr);  \
  } while (0)

template <typename T>
cudaError_t dalloc(gg_ctx* ctx, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e == cudaSuccess) {
    *p = static_cast<T*>(q);
    ctx->owned.push_back(q);
  }
  return e;
}

void dfree(gg_ctx* ctx, void* p) {
  if (!p) return;
  auto it = std::find(ctx->owned.begin(), ctx->owned.end(), p);
  if (it != ctx->owned.end()) ctx->owned.erase(it);
  cudaFree(p);
}

int blocks_for(long long n) { return static_cast<int>((n + kBlock - 1) / kBlock); }
#ifndef GG_SORT_BLOCK
#define GG_SORT_BLOCK 256
#endif
constexpr int kSortBlock = GG_SORT_BLOCK;  // count / scatter / fill / resort block size
static_assert(kBlock % kSortBlock == 0, "sort blocks tile the kBlock grid");
// up to this many scan tiles (2048 buckets each) k_scan_apply sums its
// predecessor tiles itself and k_scan_top is not launched
#ifndef GG_SCAN_TOP_FREE
#define GG_SCAN_TOP_FREE 2048
#endif
constexpr int kScanTopFree = GG_SCAN_TOP_FREE;
#ifndef GG_SWEEP_BLOCK
#define GG_SWEEP_BLOCK 32
#endif
constexpr int kSweepBlock = GG_SWEEP_BLOCK;  // k_sweep block size (<= kBlock)
#ifndef GG_FINISH_BLOCK
#define GG_FINISH_BLOCK 256
#endif
constexpr int kFinishBlockFin = GG_FINISH_BLOCK;
int sweep_grid(long long n) { return static_cast<int>((n + kSweepBlock - 1) / kSweepBlock); }
// one per-particle sweep launch over particles [0, n): record-major by default
#ifndef GG_SWEEP_FIN
#define GG_SWEEP_FIN 0  // measured slower; bitwise equal either way
#endif
// the last record-major sweep integrates too (no k_finish launch): one bed
// (E == 1), not the slab graph's device-count variant
bool sweep_fin(const Dev& D) {
  return GG_SWEEP_RM && GG_SWEEP_FIN && kFinishBlockFin == kFinGroup && D.E == 1 && !D.dn &&
         D.S >= 1 && D.pipeline != GG_MODE_ONE_LOOP;
}
// fin: the caller launches no k_finish after the last sweep (sweep_fin(D))
void launch_sweep(const Dev& D, int it, long long n, cudaStream_t s, bool fin = false) {
#if GG_SWEEP_RM
  if (fin && it == D.S - 1)
    k_sweep_rm<false, true><<<sweep_grid(n), kSweepBlock, 0, s>>>(D, it);
  else if (D.dn)
    k_sweep_rm<true><<<sweep_grid(n), kSweepBlock, 0, s>>>(D, it);
  else
    k_sweep_rm<false><<<sweep_grid(n), kSweepBlock, 0, s>>>(D, it);
#else
  if (D.dn)
    k_sweep<true><<<sweep_grid(n), kSweepBlock, 0, s>>>(D, it);
  else
    k_sweep<false><<<sweep_grid(n), kSweepBlock, 0, s>>>(D, it);
#endif
}
#ifndef GG_FINISH_BLOCK
#define GG_FINISH_BLOCK 256
#endif
constexpr int kFinishBlock = GG_FINISH_BLOCK;  // k_finish block size (<= kBlock)
int finish_grid(long long n) { return static_cast<int>((n + kFinishBlock - 1) / kFinishBlock); }
int narrow_blocks(long long n) { return static_cast<int>((n + kNarrowBlock - 1) / kNarrowBlock); }

int validate_params(gg_ctx* ctx, const gg_params* p) {
  if (!p) return fail(ctx, GG_EINVAL, "params is NULL");
  if (!(p->radius > 0)) return fail(ctx, GG_EINVAL, "radius must be > 0");
  if (!(p->particle_mass > 0)) return fail(ctx, GG_EINVAL, "particle_mass must be > 0");
  if (!(p->friction >= 0)) return fail(ctx, GG_EINVAL, "friction must be >= 0");
  if (!(p->timestep > 0)) return fail(ctx, GG_EINVAL, "timestep must be > 0");
  if (p->solver_iterations < 1) return fail(ctx, GG_EINVAL, "solver_iterations must be >= 1");
  if (p->has_boundary && !(p->z_min < p->z_max))
    return fail(ctx, GG_EINVAL, "cyclic boundary requires z_min < z_max");
  return GG_OK;
}

void fill_params(gg_ctx* ctx) {
  const gg_params& P = ctx->P;
  Dev& D = ctx->D;
  D.r = P.radius;
  D.two_r = 2.0 * P.radius;
  D.contact_d2 = P.contact_d2;
  D.coinc_d2 = P.coincident_d2;
  D.mass = P.particle_mass;
  D.mu = P.friction;
  D.alpha = P.baumgarte_alpha;
  D.dt = P.timestep;
  D.gamma = P.gamma;
  D.bias_coef = P.baumgarte_alpha / P.timestep;
  {
    // conservative float32 reject threshold (see k_narrow)
    const double t = P.contact_d2 * (1.0 + 1e-5);
    float f = static_cast<float>(t);
    if (static_cast<double>(f) < t) f = nextafterf(f, INFINITY);
    D.reject_d2f = f;
  }
  D.gdt0 = P.gdt[0];
  D.gdt1 = P.gdt[1];
  D.gdt2 = P.gdt[2];
  D.S = P.solver_iterations;
  D.has_boundary = P.has_boundary;
  D.z_min = P.z_min;
  D.band = P.z_max - P.z_min;
}

int alloc_slots(gg_ctx* ctx, int K) {
  Dev& D = ctx->D;
  dfree(ctx, D.cgeo);
  dfree(ctx, D.coth);
  dfree(ctx, D.cvb);
  D.cgeo = nullptr;
  D.coth = nullptr;
  D.cvb = nullptr;
  // K records per particle on average: record 0 of particle k at index k,
  // then one region of 32 x (K - 1) records per warp of 32 particles (a
  // warp's owners share it: per-owner counts are not limited by K)
  K = std::max(K, kFixedSlots + 1);
  const long long n1 = std::max<long long>(ctx->n, 1);
  const long long wcap = 32ll * (K - kFixedSlots);
  // regions for every warp of a kBlock-rounded grid: a sweep warp past the
  // last particle still requests its region's first records (speculatively,
  // with the heads) and must stay inside the allocation
  const long long nwarps = ((n1 + kBlock - 1) / kBlock) * (kBlock / 32);
  const size_t slots = static_cast<size_t>(kFixedSlots * n1 + nwarps * wcap);
  CK(dalloc(ctx, &D.cgeo, slots));
  CK(dalloc(ctx, &D.coth, slots));
  CK(dalloc(ctx, &D.cvb, slots));
  // defined contents: the sweeps load a particle's slot-0 record together
  // with its count, before knowing whether it has one
  CK(cudaMemset(D.cgeo, 0, sizeof(float4) * slots));
  CK(cudaMemset(D.coth, 0, sizeof(int) * slots));
  CK(cudaMemset(D.cvb, 0, sizeof(float4) * slots));
  ctx->K = K;
  D.K = K;
  D.cap_tot = static_cast<long long>(slots);
  D.nrec0 = static_cast<long long>(kFixedSlots) * n1;
  D.wcap = wcap;
  ctx->graph_dirty = true;
  return GG_OK;
}

int ensure_batch(gg_ctx* ctx, int steps, int nb) {
  const int need = std::max(steps, 1);
  const int nbx = std::max(nb, 1);
  if (need <= ctx->batch_cap && nbx <= std::max(ctx->max_bodies, 1)) return GG_OK;
  if (nb > ctx->max_bodies) {
    // grow the body capacity: the fallback momentum accumulators depend on it
    ctx->max_bodies = nb;
    dfree(ctx, ctx->D.bm_fix);
    ctx->D.bm_fix = nullptr;
    CK(dalloc(ctx, &ctx->D.bm_fix, static_cast<size_t>(nb) * 3 * ctx->E));
    CK(cudaMemset(ctx->D.bm_fix, 0, sizeof(unsigned long long) * nb * 3 * ctx->E));
  }
  int cap = std::max(ctx->batch_cap, 1);
  while (cap < need) cap *= 2;
  dfree(ctx, ctx->d_bodies);
  dfree(ctx, ctx->d_reports);
  dfree(ctx, ctx->d_bm);
  if (ctx->h_bodies) cudaFreeHost(ctx->h_bodies);
  ctx->d_bodies = nullptr;
  ctx->d_reports = nullptr;
  ctx->d_bm = nullptr;
  ctx->h_bodies = nullptr;
  const size_t mb = static_cast<size_t>(std::max(ctx->max_bodies, 1)) * ctx->E;  // per step
  CK(dalloc(ctx, &ctx->d_bodies, static_cast<size_t>(cap) * mb));
  CK(dalloc(ctx, &ctx->d_reports, static_cast<size_t>(cap) * ctx->E));
  CK(dalloc(ctx, &ctx->d_bm, static_cast<size_t>(cap) * mb * 3));
  CK(cudaMallocHost(&ctx->h_bodies, sizeof(gg_body) * static_cast<size_t>(cap) * mb));
  ctx->batch_cap = cap;
  ctx->graph_dirty = true;
  return GG_OK;
}

// The step schedule.  Optional Morton re-sort (R1-R4), the hash index
// (H1-H4), narrowphase, cooperative solve.  All on ctx->stream.
// every entry point starts with zeroed bucket/tile counts (a failed step may
// leave them dirty; within a batch each scatter re-zeroes them)
int begin_batch(gg_ctx* ctx, cudaStream_t s) {
  CK(cudaMemsetAsync(ctx->D.cnt, 0, sizeof(uint32_t) * static_cast<size_t>(ctx->D.nh_tot), s));  // every env's table
  CK(cudaMemsetAsync(ctx->D.tile, 0, sizeof(uint32_t) * static_cast<size_t>(ctx->ntiles), s));
  CK(cudaMemsetAsync(ctx->D.bflags, 0, sizeof(unsigned) * ctx->nflags, s));
  const long long work = std::max<long long>(ctx->E, static_cast<long long>(ctx->E) * std::max(ctx->max_bodies, 1) * 3);
  k_batch_begin<<<static_cast<int>(std::min<long long>(148, (work + 255) / 256)), 256, 0, s>>>(ctx->D);
  CK(cudaGetLastError());
  return GG_OK;
}

bool use_fused_step(const gg_ctx* ctx) {
  if (ctx->pipeline == GG_MODE_ONE_LOOP) return false;  // per-sweep k_sweep_oneloop launches
  if (ctx->solve_mode == 4 || ctx->solve_mode == 5 || ctx->solve_mode == 6 || ctx->solve_mode == 7)
    return true;
  if (ctx->solve_mode != 0) return false;
  return ctx->n <= static_cast<long long>(ctx->fused_grid) * kBlock;
}

// fused prep (sort + contacts, grid-wide) + cluster solve: auto for small n
bool use_cluster_solve(const gg_ctx* ctx) {
  if (!use_fused_step(ctx) || !ctx->cluster_ok) return false;
  return ctx->solve_mode == 6;
}

// k_solve_staged (mode 8): usable while a block's particles and most of
// its records fit its shared memory
// (opt-in: measured 3.5% slower than the per-sweep kernels per bed1m step
// inside the step graph, although 7% faster as a kernel timed alone)
bool use_staged_solve(const gg_ctx* ctx) {
  if (ctx->pipeline == GG_MODE_ONE_LOOP || ctx->staged_grid < 1 || ctx->D.stage_cap < 0) return false;
  return ctx->solve_mode == 8;
}

bool use_persistent_solve(const gg_ctx* ctx) {
  if (ctx->solve_mode == 3 || ctx->pipeline == GG_MODE_ONE_LOOP) return false;
  if (use_staged_solve(ctx)) return true;
  if (ctx->solve_mode == 0) return false;
  return ctx->n <= static_cast<long long>(ctx->solve_grid) * kBlock;
}

int launch_coop(gg_ctx* ctx, void (*kern)(Dev), int grid, const Dev& D, cudaStream_t s, bool coop,
                size_t smem = 0) {
  // bar_count, done_count, bar_gen are contiguous in Ctl
  // barrier words and sweep flags are zero on entry: begin_batch zeroes them
  // and the last block of every cooperative launch resets them
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kern, D));
  return GG_OK;
}

int launch_cluster_solve(gg_ctx* ctx, const Dev& D, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterCTAs);
  cfg.blockDim = dim3(kClusterBlock);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClusterCTAs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_solve_cluster, D));
  return GG_OK;
}

int env_report_blocks(const gg_ctx* ctx) {
  const long long work = std::max<long long>(ctx->E, static_cast<long long>(ctx->E) * ctx->D.nb * 3);
  return static_cast<int>(std::min<long long>(4 * 148, (work + kBlock - 1) / kBlock));
}

// The contact kernel of a step over particles [0, nn)
void launch_narrow(gg_ctx* ctx, const Dev& D, long long nn, cudaStream_t s) {
  if (D.dn)
    k_narrow<true><<<narrow_blocks(nn), kNarrowBlock, sizeof(NarrowSmemN), s>>>(D);
  else
    k_narrow<false><<<narrow_blocks(nn), kNarrowBlock, sizeof(NarrowSmemN), s>>>(D);
}

int launch_solve(gg_ctx* ctx, const Dev& D0, cudaStream_t s) {
  if (!use_persistent_solve(ctx)) {
    // one thread per particle: S sweep launches + integrate/report
    Dev D = D0;
    D.env_kernel = ctx->E > 1 ? 1 : 0;
    for (int it = 0; it < D.S; ++it) {
      if (D.pipeline == GG_MODE_ONE_LOOP)
        k_sweep_oneloop<<<ctx->nblocks, kBlock, 0, s>>>(D, it);
      else
        launch_sweep(D, it, ctx->n, s, sweep_fin(D));
    }
    if (!sweep_fin(D)) k_finish<false><<<finish_grid(ctx->n), kFinishBlock, 0, s>>>(D);
    k_commit<<<1, kBlock, 0, s>>>(D, finish_grid(ctx->n));
    if (D.env_kernel) k_env_reports<<<env_report_blocks(ctx), kBlock, 0, s>>>(D);
    CK(cudaGetLastError());
    return GG_OK;
  }
  const Dev& D = D0;
  if (use_staged_solve(ctx)) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctx->staged_grid);
    cfg.blockDim = dim3(kStageBlock);
    cfg.dynamicSmemBytes = ctx->staged_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_solve_staged, D));
    return GG_OK;
  }
  return launch_coop(ctx, k_solve, ctx->solve_grid, D, s, ctx->solve_mode != 2);  // modes 1, 2
}

int enqueue_sort_pass(gg_ctx* ctx, const Dev& D, cudaStream_t s) {
  // the per-particle sort kernels in kSortBlock-thread blocks (the same
  // threads as ctx->nblocks x kBlock)
  const int nbn = ctx->nblocks * (kBlock / kSortBlock);
  // bucket/tile counts are zero on entry: the previous scatter zeroed them
  if (D.dn)
    k_count<true><<<nbn, kSortBlock, 0, s>>>(D);
  else
    k_count<false><<<nbn, kSortBlock, 0, s>>>(D);
  k_scan_tiles<<<ctx->ntiles, kBlock, 0, s>>>(D);
  if (ctx->ntiles > kScanTopFree) k_scan_top<<<1, 1024, 0, s>>>(D, ctx->ntiles);
  k_scan_apply<<<ctx->ntiles, kBlock, 0, s>>>(D, ctx->ntiles <= kScanTopFree ? 1 : 0);
  if (D.dn) {
    k_scatter<true><<<nbn, kSortBlock, 0, s>>>(D);
    if (D.key_morton)
      k_resort<true><<<nbn, kSortBlock, 0, s>>>(D);
    else
      k_fill<true><<<nbn, kSortBlock, 0, s>>>(D);
  } else {
    k_scatter<false><<<nbn, kSortBlock, 0, s>>>(D);
    if (D.key_morton)
      k_resort<false><<<nbn, kSortBlock, 0, s>>>(D);
    else
      k_fill<false><<<nbn, kSortBlock, 0, s>>>(D);
  }
  CK(cudaGetLastError());
  return GG_OK;
}

Dev pass_dev(const gg_ctx* ctx, int resort, int morton) {
  Dev D = ctx->D;
  D.resort = resort;
  D.key_morton = morton;
  D.fused_stop = 0;
  D.sweep_barrier = (ctx->solve_mode == 7 || ctx->solve_mode == 0) ? 1 : 0;
  D.env_kernel = 0;
  D.pipeline = ctx->pipeline;
  return D;
}

bool use_cluster_solve(const gg_ctx* ctx);

// the small-n schedule: k_step_fused, then (split mode) k_solve_cluster
int launch_fused(gg_ctx* ctx, int resort, cudaStream_t s) {
  Dev D = pass_dev(ctx, resort, 0);
  const bool split = use_cluster_solve(ctx);
  D.fused_stop = split ? 1 : 0;
  int st = launch_coop(ctx, k_step_fused, ctx->fused_grid, D, s, ctx->solve_mode != 5,
                       sizeof(NarrowSmem));
  if (st != GG_OK || !split) return st;
  D.fused_stop = 0;
  return launch_cluster_solve(ctx, D, s);
}

int enqueue_step(gg_ctx* ctx, int resort) {
  cudaStream_t s = ctx->stream;
  if (use_fused_step(ctx)) return launch_fused(ctx, resort, s);
  int st;
  if (resort) {
    st = enqueue_sort_pass(ctx, pass_dev(ctx, 1, 1), s);
    if (st != GG_OK) return st;
  }
  const Dev D = pass_dev(ctx, resort, 0);
  st = enqueue_sort_pass(ctx, D, s);
  if (st != GG_OK) return st;
  launch_narrow(ctx, D, ctx->n, s);
  CK(cudaGetLastError());
  return launch_solve(ctx, D, s);
}

bool use_persistent_solve(const gg_ctx* ctx);
bool use_fused_step(const gg_ctx* ctx);

bool use_staged_solve(const gg_ctx* ctx);

int kernels_per_step(const gg_ctx* ctx, int resort) {
  if (use_fused_step(ctx)) return use_cluster_solve(ctx) ? 2 : 1;
  const int solve = use_persistent_solve(ctx) ? 1 : ctx->D.S + (sweep_fin(ctx->D) ? 1 : 2);
  const int env_reports = (ctx->E > 1 && !use_persistent_solve(ctx)) ? 1 : 0;
  const int top = ctx->ntiles > kScanTopFree ? 1 : 0;  // k_scan_top per sort pass
  return 6 + top + solve + env_reports + (resort ? 5 + top : 0);
}

// Same schedule as enqueue_step, with an event after every kernel so each
// kernel kind's device time can be attributed (bench roofline pass).
constexpr int kProfKinds = 14;
const char* kProfNames[kProfKinds] = {"(unused)", "k_count", "k_scan_tiles", "k_scan_top",
                                      "k_scan_apply",  "k_scatter", "k_resort",  "k_fill",
                                      "k_narrow",      "k_solve",   "(unused)",  "k_step_fused",
                                      "k_sweep",       "k_finish"};

int ensure_events(gg_ctx* ctx, size_t n) {
  while (ctx->evpool.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->evpool.push_back(e);
  }
  return GG_OK;
}

// Same schedule as enqueue_step with an event after every kernel, so each
// kernel kind's device time can be attributed (bench roofline pass).
int enqueue_step_profiled(gg_ctx* ctx, int resort, cudaEvent_t* ev, int* kind_of_interval) {
  cudaStream_t s = ctx->stream;
  const int nbn = ctx->nblocks;
  int e = 0;
  auto mark = [&](int kind) {
    cudaEventRecord(ev[e + 1], s);
    kind_of_interval[e] = kind;
    ++e;
  };
  cudaEventRecord(ev[0], s);
  if (use_fused_step(ctx)) {
    Dev D = pass_dev(ctx, resort, 0);
    const bool split = use_cluster_solve(ctx);
    D.fused_stop = split ? 1 : 0;
    if (launch_coop(ctx, k_step_fused, ctx->fused_grid, D, s, ctx->solve_mode != 5,
                    sizeof(NarrowSmem)) != GG_OK)
      return -1;
    mark(11);
    if (split) {
      D.fused_stop = 0;
      if (launch_cluster_solve(ctx, D, s) != GG_OK) return -1;
      mark(9);
    }
    return e;
  }
  for (int pass = resort ? 0 : 1; pass < 2; ++pass) {
    const Dev D = pass_dev(ctx, resort, pass == 0 ? 1 : 0);
    k_count<false><<<nbn, kBlock, 0, s>>>(D);
    mark(1);
    k_scan_tiles<<<ctx->ntiles, kBlock, 0, s>>>(D);
    mark(2);
    if (ctx->ntiles > kScanTopFree) k_scan_top<<<1, 1024, 0, s>>>(D, ctx->ntiles);
    mark(3);
    k_scan_apply<<<ctx->ntiles, kBlock, 0, s>>>(D, ctx->ntiles <= kScanTopFree ? 1 : 0);
    mark(4);
    k_scatter<false><<<nbn, kBlock, 0, s>>>(D);
    mark(5);
    if (pass == 0) {
      k_resort<false><<<nbn, kBlock, 0, s>>>(D);
      mark(6);
    } else {
      k_fill<false><<<nbn, kBlock, 0, s>>>(D);
      mark(7);
    }
  }
  const Dev D = pass_dev(ctx, resort, 0);
  launch_narrow(ctx, D, ctx->n, s);
  mark(8);
  if (use_persistent_solve(ctx)) {
    if (launch_solve(ctx, D, s) != GG_OK) return -1;
    mark(9);
  } else {
    for (int it = 0; it < D.S; ++it) {
      if (D.pipeline == GG_MODE_ONE_LOOP)
        k_sweep_oneloop<<<nbn, kBlock, 0, s>>>(D, it);
      else
        launch_sweep(D, it, ctx->n, s, sweep_fin(D));
      mark(12);
    }
    Dev Df = D;
    Df.env_kernel = ctx->E > 1 ? 1 : 0;
    if (!sweep_fin(D)) k_finish<false><<<finish_grid(ctx->n), kFinishBlock, 0, s>>>(Df);
    k_commit<<<1, kBlock, 0, s>>>(Df, finish_grid(ctx->n));
    if (Df.env_kernel) k_env_reports<<<env_report_blocks(ctx), kBlock, 0, s>>>(Df);
    mark(13);
  }
  if (cudaGetLastError() != cudaSuccess) return -1;
  return e;
}

int refresh_dev(gg_ctx* ctx) {
  Dev& D = ctx->D;
  D.bodies = ctx->d_bodies;
  D.grids = ctx->d_grids;
  D.gvals = ctx->d_gvals;
  D.reports = ctx->d_reports;
  D.bm_out = ctx->d_bm;
  return GG_OK;
}

int build_graph(gg_ctx* ctx) {
  refresh_dev(ctx);
  for (int g = 0; g < 2; ++g) {
    if (ctx->gexec[g]) {
      cudaGraphExecDestroy(ctx->gexec[g]);
      ctx->gexec[g] = nullptr;
    }
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    int st = enqueue_step(ctx, g);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (st != GG_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&ctx->gexec[g], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
  }
  ctx->graph_dirty = false;
  return GG_OK;
}

// launch one step's graph, re-sorting the physical order every resort_every
int launch_step(gg_ctx* ctx) {
  const int resort = ctx->since_resort >= ctx->resort_every ? 1 : 0;
  CK(cudaGraphLaunch(ctx->gexec[resort], ctx->stream));
  ctx->since_resort = resort ? 1 : ctx->since_resort + 1;
  ctx->launches += kernels_per_step(ctx, resort);
  return GG_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int now = -1;
    cudaGetDevice(&now);
    if (prev >= 0 && now != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

const char* gg_build_info(void) { return kBuildInfo; }

int64_t gg_kernel_launches(const gg_ctx* ctx) { return ctx ? ctx->launches : 0; }

// context-free entry points (gg_bake_mesh_sdf) report here
thread_local std::string g_free_err = "null context";

const char* gg_last_error(const gg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_free_err.c_str(); }

int gg_bake_mesh_sdf(int32_t device, const double* tri, int64_t n_tri, const double* points,
                     int64_t n_points, const double origin[3], const double spacing[3],
                     const int64_t dims[3], double* out, float* kernel_ms) {
  auto ferr = [](int code, const std::string& m) {
    g_free_err = m;
    return code;
  };
  if (!tri || n_tri < 1 || !out) return ferr(GG_EINVAL, "bake: need at least one triangle and an output");
  long long n = n_points;
  if (!points) {
    if (!origin || !spacing || !dims) return ferr(GG_EINVAL, "bake: grid mode needs origin, spacing, dims");
    n = 1;
    for (int a = 0; a < 3; ++a) {
      if (dims[a] < 1) return ferr(GG_EINVAL, "bake: dims must be positive");
      n *= dims[a];
    }
  }
  if (n < 1) return ferr(GG_EINVAL, "bake: no points");
  int prev = -1;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  double *d_tri = nullptr, *d_pts = nullptr, *d_out = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto step = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
    return e == cudaSuccess;
  };
  const size_t tb = static_cast<size_t>(n_tri) * kTriDoubles * sizeof(double);
  if (step(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) && step(cudaEventCreate(&e0)) &&
      step(cudaEventCreate(&e1)) && step(cudaMalloc(&d_tri, tb)) &&
      step(cudaMalloc(&d_out, static_cast<size_t>(n) * sizeof(double))) &&
      (!points || step(cudaMalloc(&d_pts, static_cast<size_t>(n) * 3 * sizeof(double)))) &&
      step(cudaMemcpyAsync(d_tri, tri, tb, cudaMemcpyHostToDevice, st)) &&
      (!points || step(cudaMemcpyAsync(d_pts, points, static_cast<size_t>(n) * 3 * sizeof(double),
                                       cudaMemcpyHostToDevice, st)))) {
    BakeArgs A{};
    A.tri = d_tri;
    A.T = n_tri;
    A.pts = d_pts;
    for (int a = 0; a < 3; ++a) {
      A.origin[a] = points ? 0.0 : origin[a];
      A.spacing[a] = points ? 0.0 : spacing[a];
      A.dims[a] = points ? 1 : dims[a];
    }
    A.n = n;
    A.out = d_out;
    const long long blocks = (n + 255) / 256;
    step(cudaEventRecord(e0, st));
    k_bake_sdf<<<static_cast<unsigned>(blocks), 256, 0, st>>>(A);
    step(cudaGetLastError());
    step(cudaEventRecord(e1, st));
    step(cudaMemcpyAsync(out, d_out, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (step(cudaStreamSynchronize(st)) && kernel_ms) step(cudaEventElapsedTime(kernel_ms, e0, e1));
  }
  cudaFree(d_tri);
  cudaFree(d_pts);
  cudaFree(d_out);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) return ferr(GG_ECUDA, std::string("bake: ") + cudaGetErrorString(e));
  return GG_OK;
}

int gg_create(int device, const gg_params* params, int64_t n, int64_t n_h, int32_t max_bodies,
              int32_t max_contacts, gg_ctx** out) {
  return gg_create_batched(device, params, 1, n, n_h, max_bodies, max_contacts, out);
}

int gg_create_batched(int device, const gg_params* params, int32_t n_envs, int64_t n_per_env,
                      int64_t n_h, int32_t max_bodies, int32_t max_contacts, gg_ctx** out) {
  if (!out) return GG_EINVAL;
  *out = nullptr;
  gg_ctx* ctx = new gg_ctx();
  int st = validate_params(ctx, params);
  if (st != GG_OK) {
    // keep the context so the caller can read the message
    *out = ctx;
    return st;
  }
  const long long E = n_envs;
  const long long n = E * n_per_env;
  if (E < 1 || n_per_env < 1 || n >= (1ll << 31) || n_h < 1 || E * n_h >= (1ll << 31)) {
    *out = ctx;
    return fail(ctx, GG_EINVAL,
                "need n_envs >= 1, n_per_env >= 1, n_envs * n_per_env < 2^31 and "
                "1 <= n_envs * n_h < 2^31");
  }
  *out = ctx;
  ctx->device = device;
  DeviceGuard guard(device);
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&ctx->ev0));
  CK(cudaEventCreate(&ctx->ev1));
  ctx->P = *params;
  ctx->n = n;
  ctx->n_h = n_h;
  ctx->E = static_cast<int>(E);
  ctx->ne = n_per_env;
  ctx->max_bodies = std::max(max_bodies, 0);
  ctx->nblocks = blocks_for(n);
  ctx->ntiles = static_cast<int>((E * n_h + kScanTile - 1) / kScanTile);
  Dev& D = ctx->D;
  D.n = static_cast<int>(n);
  D.n_own = static_cast<int>(n);
  D.E = static_cast<int>(E);
  D.ne = static_cast<int>(n_per_env);
  D.nh_tot = E * n_h;
  D.nblocks = ctx->nblocks;
  D.H.n_h = n_h;
  D.H.pow2 = (n_h & (n_h - 1)) == 0 ? 1 : 0;
  D.H.mask = static_cast<uint32_t>(n_h - 1);
  {
    long long p2 = 1;
    while (p2 * 2 <= n_h) p2 *= 2;
    D.mmask = static_cast<uint32_t>(p2 - 1);
    D.mspan = static_cast<uint32_t>(p2);
    int bits = 0;
    while (bits < 10 && (1ll << (3 * (bits + 1))) <= p2) ++bits;
    D.mbits = bits;
    // until a state is uploaded: the window centred on the origin, wrapping
    D.mlo[0] = D.mlo[1] = D.mlo[2] = -(1 << bits) / 2;
    D.msh[0] = D.msh[1] = D.msh[2] = 0;
    D.mclamp = 0;
  }
  fill_params(ctx);
  D.nb = 0;
  for (int b = 0; b < 2; ++b) {
    CK(dalloc(ctx, &D.X[b], n));
    CK(dalloc(ctx, &D.V[b], n));
    CK(dalloc(ctx, &D.UID[b], n));
    CK(dalloc(ctx, &D.W[b], n));
  }
  CK(dalloc(ctx, &D.key, n));
  CK(dalloc(ctx, &D.arrive, n));
  CK(dalloc(ctx, &D.tmp, n));
  CK(dalloc(ctx, &D.cnt, E * n_h));
  CK(dalloc(ctx, &D.start, E * n_h + 1));
  CK(dalloc(ctx, &D.tile, ctx->ntiles));
  CK(dalloc(ctx, &D.Xs, n));
  CK(dalloc(ctx, &D.V0, n));
  CK(dalloc(ctx, &D.cinfo, n));
  CK(cudaMemset(D.cinfo, 0, sizeof(int2) * n));
  CK(dalloc(ctx, &D.bad, n));
  CK(cudaMemset(D.bad, 0, sizeof(int) * n));
  CK(cudaFuncSetAttribute(k_narrow<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(sizeof(NarrowSmemN))));
  CK(cudaFuncSetAttribute(k_narrow<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(sizeof(NarrowSmemN))));
  CK(cudaFuncSetAttribute(k_step_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(sizeof(NarrowSmem))));
#ifndef GG_SWEEP_CARVE
#define GG_SWEEP_CARVE -1
#endif
#ifndef GG_NARROW_CARVE
#define GG_NARROW_CARVE -1
#endif
  // shared-memory carve-out preference (percent of the unified L1/shared
  // array; -1 leaves the driver's choice)
  if (GG_SWEEP_CARVE >= 0) {
    CK(cudaFuncSetAttribute(k_sweep_rm<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            GG_SWEEP_CARVE));
    CK(cudaFuncSetAttribute(k_sweep_rm<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            GG_SWEEP_CARVE));
    CK(cudaFuncSetAttribute(k_finish<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            GG_SWEEP_CARVE));
  }
  if (GG_NARROW_CARVE >= 0)
    CK(cudaFuncSetAttribute(k_narrow<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            GG_NARROW_CARVE));
  CK(dalloc(ctx, &D.acc, E));
  D.ke_fix = nullptr;
  if (E > 1) {
    CK(dalloc(ctx, &D.ke_fix, E));
    CK(cudaMemset(D.ke_fix, 0, sizeof(unsigned long long) * E));
  }
  // co-resident grid of the cooperative solve kernel
  {
    int per_sm = 0, sms = 0, per_sm_f = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, kBlock, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_f, k_step_fused, kBlock,
                                                     sizeof(NarrowSmem)));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    ctx->solve_grid = std::max(1, std::min(ctx->nblocks, per_sm * sms));
    // n / kBlock blocks (packed) when they fit: measured faster than spreading
    // the particles thinly over every co-resident block (hero50k 0.117 vs
    // 0.130 ms/step); the kernel spreads particles evenly over its grid
    ctx->fused_grid = std::max(1, std::min(ctx->nblocks, per_sm_f * sms));
    // k_solve_staged: one block of kStageBlock threads per SM with (nearly)
    // all of the SM's shared memory for the staged contact records
    {
      int optin = 0;
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
      cudaFuncAttributes fa{};
      CK(cudaFuncGetAttributes(&fa, k_solve_staged));
      const long long dyn = static_cast<long long>(optin) - static_cast<long long>(fa.sharedSizeBytes) - 1024;
      int per_sm_s = 0;
      if (dyn > 0 &&
          cudaFuncSetAttribute(k_solve_staged, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(dyn)) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, k_solve_staged, kStageBlock,
                                                        static_cast<size_t>(dyn)) == cudaSuccess &&
          per_sm_s > 0) {
        ctx->staged_grid = per_sm_s * sms;
        ctx->staged_smem = static_cast<size_t>(dyn);
        // average particles per block; blocks size their ranges by work at run time
        const long long pb = (n + ctx->staged_grid - 1) / ctx->staged_grid;
        D.stage_pb = static_cast<int>(pb);
        D.stage_smem = dyn;
        // shared-memory staging pays while a block's counts and most of its
        // records fit: beyond ~16k particles per block the per-sweep kernels win
        D.stage_cap = (pb <= 16384 && ctx->staged_grid <= kStageMaxGrid) ? 1 : -1;
      } else {
        ctx->staged_grid = 0;
        D.stage_cap = -1;
      }
      cudaGetLastError();
    }
    // can one 16-CTA cluster of k_solve_cluster be resident?
    if (cudaFuncSetAttribute(k_solve_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
        cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kClusterCTAs);
      cfg.blockDim = dim3(kClusterBlock);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kClusterCTAs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      ctx->cluster_ok = cudaOccupancyMaxActiveClusters(&nclusters, k_solve_cluster, &cfg) == cudaSuccess &&
                        nclusters >= 1;
    }
    cudaGetLastError();  // a refused query only disables the cluster path
  }
  // kXhPad entries past the end: the candidate loop's sentinel bucket may read
  // up to GG_KDEPTH - 1 entries beyond a bucket that ends at the last entry
  // (values never tested); zeroed so every read is of initialised memory
  CK(dalloc(ctx, &D.Xh, n + kXhPad));
  CK(cudaMemset(D.Xh, 0, sizeof(float4) * (n + kXhPad)));
  {  // far padding after the particles: the contact kernel's list sentinel
     // reads it, and nothing there ever passes the prefilter
    float4 far[kXhPad];
    const int none = -1;  // (w: no particle)
    float wn;
    std::memcpy(&wn, &none, sizeof(wn));
    for (int i = 0; i < kXhPad; ++i) far[i] = make_float4(1e30f, 1e30f, 1e30f, wn);
    CK(cudaMemcpy(D.Xh + n, far, sizeof(far), cudaMemcpyHostToDevice));
    D.xh_pad = static_cast<int>(n);
  }
  // one flag per block of any persistent launch (the commit of each resets
  // its grid's flags)
  ctx->nflags = std::max({ctx->fused_grid, ctx->solve_grid, ctx->staged_grid, kClusterCTAs, 1});
  CK(dalloc(ctx, &D.bflags, static_cast<size_t>(ctx->nflags)));
  CK(dalloc(ctx, &D.part, static_cast<size_t>(std::max({ctx->solve_grid, ctx->fused_grid, ctx->nblocks,
                                                          finish_grid(n), kClusterCTAs,
                                                          ctx->staged_grid}))));
  CK(dalloc(ctx, &D.wpart, static_cast<size_t>(sweep_grid(n) * (kSweepBlock / 32))));
  CK(dalloc(ctx, &D.gcnt, static_cast<size_t>(finish_grid(n))));
  CK(cudaMemset(D.gcnt, 0, sizeof(unsigned) * finish_grid(n)));
  CK(dalloc(ctx, &D.bm_fix, static_cast<size_t>(std::max(ctx->max_bodies, 1)) * 3 * E));
  CK(dalloc(ctx, &D.stage_seg, static_cast<size_t>(std::max(ctx->staged_grid, 1))));
  CK(cudaMemset(D.bm_fix, 0, sizeof(unsigned long long) * std::max(ctx->max_bodies, 1) * 3 * E));
  CK(dalloc(ctx, &D.ctl, 1));
  CK(cudaMallocHost(&ctx->h_ctl, sizeof(Ctl)));
  st = alloc_slots(ctx, max_contacts > 0 ? max_contacts : 16);
  if (st != GG_OK) return st;
  // start[E * n_h] = n never changes for a context
  const uint32_t nn = static_cast<uint32_t>(n);
  CK(cudaMemcpy(D.start + E * n_h, &nn, sizeof(uint32_t), cudaMemcpyHostToDevice));
  CK(cudaMemset(D.ctl, 0, sizeof(Ctl)));
  CK(cudaMemset(D.UID[0], 0, sizeof(int) * n));
  st = ensure_batch(ctx, 1, ctx->max_bodies);
  if (st != GG_OK) return st;
  // zero-state until the caller uploads
  CK(cudaMemset(D.X[0], 0, sizeof(float4) * n));
  CK(cudaMemset(D.V[0], 0, sizeof(float4) * n));
  CK(cudaDeviceSynchronize());
  return GG_OK;
}

int gg_destroy(gg_ctx* ctx) {
  if (!ctx) return GG_OK;
  {
    DeviceGuard guard(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (int g = 0; g < 2; ++g)
      if (ctx->gexec[g]) cudaGraphExecDestroy(ctx->gexec[g]);
    for (int g = 0; g < 4; ++g)
      if (ctx->sgexec[g]) cudaGraphExecDestroy(ctx->sgexec[g]);
    for (cudaEvent_t e : ctx->evpool) cudaEventDestroy(e);
    for (int side = 0; side < 2; ++side)
      if (ctx->peer_ipc[side] && ctx->peer[side]) cudaIpcCloseMemHandle(ctx->peer[side]);
    for (void* p : ctx->owned) cudaFree(p);
    ctx->owned.clear();
    if (ctx->h_bodies) cudaFreeHost(ctx->h_bodies);
    if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
    if (ctx->h_scnt) cudaFreeHost(ctx->h_scnt);
    if (ctx->h_x) cudaFreeHost(ctx->h_x);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
  return GG_OK;
}

int gg_set_params(gg_ctx* ctx, const gg_params* params) {
  if (!ctx) return GG_EINVAL;
  int st = validate_params(ctx, params);
  if (st != GG_OK) return st;
  ctx->P = *params;
  fill_params(ctx);
  ctx->graph_dirty = true;
  ++ctx->pgen;
  return GG_OK;
}

int gg_set_max_contacts(gg_ctx* ctx, int32_t K) {
  if (!ctx || K < 1) return fail(ctx, GG_EINVAL, "max_contacts must be >= 1");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  return alloc_slots(ctx, K);
}

int gg_max_contacts(const gg_ctx* ctx) { return ctx ? ctx->K : 0; }

int gg_set_solve_mode(gg_ctx* ctx, int32_t mode) {
  if (!ctx || mode < 0 || mode > 8) return fail(ctx, GG_EINVAL, "solve mode must be 0..8");
  ctx->solve_mode = mode;
  ctx->graph_dirty = true;
  ++ctx->pgen;
  return GG_OK;
}

int gg_phase_timer(gg_ctx* ctx, int32_t on, uint64_t* stamps, int32_t cap) {
  if (!ctx) return GG_EINVAL;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  if (stamps && ctx->D.tstamp && cap > 0)
    CK(cudaMemcpy(stamps, ctx->D.tstamp, sizeof(uint64_t) * std::min(cap, 64),
                  cudaMemcpyDeviceToHost));
  if (on && !ctx->D.tstamp) {
    unsigned long long* t = nullptr;
    CK(dalloc(ctx, &t, 64));
    CK(cudaMemset(t, 0, sizeof(unsigned long long) * 64));
    ctx->D.tstamp = t;
    ctx->graph_dirty = true;
  } else if (!on && ctx->D.tstamp) {
    dfree(ctx, ctx->D.tstamp);
    ctx->D.tstamp = nullptr;
    ctx->graph_dirty = true;
  }
  return GG_OK;
}

int gg_set_resort_every(gg_ctx* ctx, int32_t steps) {
  if (!ctx || steps < 1) return fail(ctx, GG_EINVAL, "resort_every must be >= 1");
  ctx->resort_every = steps;
  return GG_OK;
}

static int ensure_stage(gg_ctx* ctx) {
  if (ctx->d_stage) return GG_OK;
  CK(dalloc(ctx, &ctx->d_stage, static_cast<size_t>(ctx->n) * 6));
  static_assert(sizeof(double) == sizeof(long long), "stage reuse");
  return GG_OK;
}

// The Morton window (Dev::mlo, msh) of a state with positions x (row stride
// `stride` values, n rows): per axis the 0.05% .. 99.95% cell quantiles,
// shifted right until they fit the key's bits per axis.  Only the physical
// order (locality) depends on it, never a result.  Marks the graphs dirty
// when it changes.
void set_morton_window(gg_ctx* ctx, const float* xf, const double* xd, long long n, int stride) {
  if (n <= 0) return;
  const int bits = ctx->D.mbits;
  const long long sample = std::min<long long>(n, 1 << 15);  // quantiles of a 32k sample: ~1 ms per upload
  const long long stepi = std::max<long long>(1, n / sample);
  std::vector<long long> c;
  c.reserve(static_cast<size_t>(sample) + 1);
  int lo[3], sh[3];
  for (int a = 0; a < 3; ++a) {
    c.clear();
    for (long long i = 0; i < n; i += stepi) {
      const double q = (xf ? static_cast<double>(xf[i * stride + a]) : xd[i * stride + a]) / ctx->D.two_r;
      if (!std::isfinite(q) || std::fabs(q) > 1e9) continue;
      c.push_back(static_cast<long long>(std::copysign(std::floor(std::fabs(q) + 0.5), q)));
    }
    if (c.empty()) {
      lo[a] = 0;
      sh[a] = 0;
      continue;
    }
    const size_t m = c.size();
    const size_t klo = m / 2000, khi = m - 1 - m / 2000;
    std::nth_element(c.begin(), c.begin() + klo, c.end());
    const long long qlo = c[klo];
    std::nth_element(c.begin(), c.begin() + khi, c.end());
    const long long qhi = c[khi];
    const long long ext = qhi - qlo + 3;  // + the halo cells either side
    int s = 0;
    while ((ext >> s) >= (1ll << bits) && s < 20) ++s;
    lo[a] = static_cast<int>(qlo - 1);
    sh[a] = s;
  }
  bool changed = ctx->D.mclamp != 1;
  ctx->D.mclamp = 1;
  for (int a = 0; a < 3; ++a) {
    changed |= ctx->D.mlo[a] != lo[a] || ctx->D.msh[a] != sh[a];
    ctx->D.mlo[a] = lo[a];
    ctx->D.msh[a] = sh[a];
  }
  if (changed) ctx->graph_dirty = true;
}

int gg_set_state_f64(gg_ctx* ctx, const double* x, const double* v) {
  if (!ctx || !x || !v) return fail(ctx, GG_EINVAL, "null argument");
  DeviceGuard guard(ctx->device);
  int st = ensure_stage(ctx);
  if (st != GG_OK) return st;
  const size_t bytes = sizeof(double) * 3 * static_cast<size_t>(ctx->n);
  CK(cudaMemcpyAsync(ctx->d_stage, x, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_stage + 3 * ctx->n, v, bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (!ctx->slab_on) set_morton_window(ctx, nullptr, x, ctx->n, 3);
  ctx->since_resort = 1 << 30;
  k_load_f64<<<ctx->nblocks, kBlock, 0, ctx->stream>>>(ctx->D, ctx->d_stage,
                                                        ctx->d_stage + 3 * ctx->n);
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return GG_OK;
}

int gg_get_state_f64(gg_ctx* ctx, double* x, double* v) {
  if (!ctx || !x || !v) return fail(ctx, GG_EINVAL, "null argument");
  DeviceGuard guard(ctx->device);
  int st = ensure_stage(ctx);
  if (st != GG_OK) return st;
  const size_t bytes = sizeof(double) * 3 * static_cast<size_t>(ctx->n);
  k_store_f64<<<ctx->nblocks, kBlock, 0, ctx->stream>>>(ctx->D, ctx->d_stage,
                                                         ctx->d_stage + 3 * ctx->n);
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(x, ctx->d_stage, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(v, ctx->d_stage + 3 * ctx->n, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return GG_OK;
}

int gg_set_state_f32x4_dev(gg_ctx* ctx, const void* x4, const void* v4) {
  if (!ctx || !x4 || !v4) return fail(ctx, GG_EINVAL, "null argument");
  DeviceGuard guard(ctx->device);
  if (!ctx->slab_on && ctx->n > 0) {
    std::vector<float> hx(4 * static_cast<size_t>(ctx->n));
    CK(cudaMemcpyAsync(hx.data(), x4, sizeof(float) * hx.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    set_morton_window(ctx, hx.data(), nullptr, ctx->n, 4);
  }
  ctx->since_resort = 1 << 30;
  k_load_f4<<<ctx->nblocks, kBlock, 0, ctx->stream>>>(ctx->D, static_cast<const float4*>(x4),
                                                       static_cast<const float4*>(v4));
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return GG_OK;
}

int gg_get_state_f32x4_dev(gg_ctx* ctx, void* x4, void* v4) {
  if (!ctx || !x4 || !v4) return fail(ctx, GG_EINVAL, "null argument");
  DeviceGuard guard(ctx->device);
  k_store_f4<<<ctx->nblocks, kBlock, 0, ctx->stream>>>(ctx->D, static_cast<float4*>(x4),
                                                        static_cast<float4*>(v4));
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return GG_OK;
}

int gg_upload_grid(gg_ctx* ctx, const double* values, const int32_t dims[3],
                   const double origin[3], const double spacing[3], int32_t* grid_id) {
  if (!ctx || !values || !dims || !origin || !spacing || !grid_id)
    return fail(ctx, GG_EINVAL, "null argument");
  for (int a = 0; a < 3; ++a)
    if (dims[a] < 2) return fail(ctx, GG_EINVAL, "grid dims must be >= 2 on every axis");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const long long count = static_cast<long long>(dims[0]) * dims[1] * dims[2];
  if (ctx->gvals_used + count > ctx->gvals_cap) {
    long long cap = std::max<long long>(ctx->gvals_cap * 2, ctx->gvals_used + count);
    double* nv = nullptr;
    CK(dalloc(ctx, &nv, static_cast<size_t>(cap)));
    if (ctx->gvals_used)
      CK(cudaMemcpy(nv, ctx->d_gvals, sizeof(double) * ctx->gvals_used, cudaMemcpyDeviceToDevice));
    dfree(ctx, ctx->d_gvals);
    ctx->d_gvals = nv;
    ctx->gvals_cap = cap;
  }
  CK(cudaMemcpy(ctx->d_gvals + ctx->gvals_used, values, sizeof(double) * count,
                cudaMemcpyHostToDevice));
  DevGrid G{};
  for (int a = 0; a < 3; ++a) {
    G.origin[a] = origin[a];
    G.spacing[a] = spacing[a];
    G.dims[a] = dims[a];
    G.upper[a] = origin[a] + static_cast<double>(dims[a] - 1) * spacing[a];
  }
  G.offset = ctx->gvals_used;
  ctx->gvals_used += count;
  ctx->grids.push_back(G);
  if (static_cast<int>(ctx->grids.size()) > ctx->d_grids_cap) {
    dfree(ctx, ctx->d_grids);
    ctx->d_grids = nullptr;
    ctx->d_grids_cap = std::max<int>(8, 2 * static_cast<int>(ctx->grids.size()));
    CK(dalloc(ctx, &ctx->d_grids, ctx->d_grids_cap));
  }
  CK(cudaMemcpy(ctx->d_grids, ctx->grids.data(), sizeof(DevGrid) * ctx->grids.size(),
                cudaMemcpyHostToDevice));
  *grid_id = static_cast<int32_t>(ctx->grids.size() - 1);
  ctx->graph_dirty = true;
  return GG_OK;
}

int gg_step(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies, int32_t mode) {
  if (!ctx) return GG_EINVAL;
  if (n_steps < 0) return fail(ctx, GG_EINVAL, "n_steps must be >= 0");
  if (n_bodies < 0) return fail(ctx, GG_EINVAL, "bad bodies");
  const bool driven = n_bodies > 0 && !bodies;  // rows from the device drivers
  if (driven)
    for (int b = 0; b < n_bodies; ++b)
      if (b >= static_cast<int>(ctx->drive.size()) || ctx->drive[b].kind == 0)
        return fail(ctx, GG_EINVAL, "bodies == NULL needs a device driver on every body slot");
  if (mode < 0 || mode > 2) return fail(ctx, GG_EINVAL, "unknown pipeline mode");
  if (mode != ctx->pipeline) {
    ctx->pipeline = mode;
    ctx->graph_dirty = true;
  }
  for (long long i = 0; !driven && i < static_cast<long long>(n_steps) * ctx->E * n_bodies; ++i) {
    const gg_body& b = bodies[i];
    if (b.kind < GG_GEOM_SPHERE || b.kind > GG_GEOM_GRID)
      return fail(ctx, GG_EINVAL, "unknown geometry kind");
    if (b.kind == GG_GEOM_GRID && (b.grid_id < 0 || b.grid_id >= (int)ctx->grids.size()))
      return fail(ctx, GG_EINVAL, "unknown grid id");
  }
  DeviceGuard guard(ctx->device);
  // the pinned staging buffer is reused: the previous batch must be done
  CK(cudaStreamSynchronize(ctx->stream));
  int st = ensure_batch(ctx, n_steps, n_bodies);
  if (st != GG_OK) return st;
  if (ctx->D.nb != n_bodies) {
    ctx->D.nb = n_bodies;
    ctx->graph_dirty = true;
  }
  if (driven) {
    const int E = ctx->E;
    const unsigned g = static_cast<unsigned>((E + 127) / 128);
    for (int b = 0; b < n_bodies; ++b) {
      gg_ctx::DriveSlot& ds = ctx->drive[b];
      if (ds.kind == 1) {
        k_drive_fixed<<<g, 128, 0, ctx->stream>>>(ctx->d_bodies, ds.d_fixed, n_steps, E, n_bodies, b);
      } else if (ds.kind == 3) {
        DriveChain C = ds.C;
        C.dt = ctx->P.timestep;
        k_drive_chain<<<g, 128, 0, ctx->stream>>>(ctx->d_bodies, C, n_steps, E, n_bodies, b);
      } else {
        DriveTrack P = ds.P;
        P.dt = ctx->P.timestep;
        k_drive_track<<<g, 128, 0, ctx->stream>>>(ctx->d_bodies, P, n_steps, E, n_bodies, b);
      }
      ctx->launches += 1;
    }
    CK(cudaGetLastError());
  } else if (n_bodies > 0) {
    const size_t bytes = sizeof(gg_body) * static_cast<size_t>(n_steps) * ctx->E * n_bodies;
    std::memcpy(ctx->h_bodies, bodies, bytes);
    CK(cudaMemcpyAsync(ctx->d_bodies, ctx->h_bodies, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ctx->graph_dirty) {
    st = build_graph(ctx);
    if (st != GG_OK) return st;
  }
  refresh_dev(ctx);
  st = begin_batch(ctx, ctx->stream);
  if (st != GG_OK) return st;
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  for (int i = 0; i < n_steps; ++i) {
    int st2 = launch_step(ctx);
    if (st2 != GG_OK) return st2;
  }
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->launches += 1;
  ctx->last_batch = n_steps;
  ctx->last_nb = n_bodies;
  ctx->tap_uncommitted = false;
  return GG_OK;
}

int gg_detect(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, gg_report* out) {
  if (!ctx) return GG_EINVAL;
  if (n_bodies < 0 || (n_bodies > 0 && !bodies)) return fail(ctx, GG_EINVAL, "bad bodies");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  int st = ensure_batch(ctx, 1, n_bodies);
  if (st != GG_OK) return st;
  if (ctx->D.nb != n_bodies) {
    ctx->D.nb = n_bodies;
    ctx->graph_dirty = true;
  }
  if (n_bodies > 0)
    CK(cudaMemcpy(ctx->d_bodies, bodies, sizeof(gg_body) * n_bodies * ctx->E,
                  cudaMemcpyHostToDevice));
  refresh_dev(ctx);
  const Dev D = pass_dev(ctx, 0, 0);
  cudaStream_t s = ctx->stream;
  st = begin_batch(ctx, s);
  if (st != GG_OK) return st;
  st = enqueue_sort_pass(ctx, D, s);
  if (st != GG_OK) return st;
  k_narrow<false><<<narrow_blocks(ctx->n), kNarrowBlock, sizeof(NarrowSmemN), s>>>(D);
  ctx->launches += 9;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  ctx->tap_uncommitted = true;
  CK(cudaMemcpy(ctx->h_ctl, D.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  if (ctx->h_ctl->err == GG_EPOSITIONS) return fail(ctx, GG_EPOSITIONS, "positions must be finite");
  if (ctx->h_ctl->err == GG_EBUCKET)
    return fail(ctx, GG_EINVAL, "hash table too small: the neighbour buckets of a particle hold more "
                                "than 27 x 65534 particles (raise hashmap_size)");
  if (ctx->h_ctl->err == GG_ECAPACITY) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "contact capacity exceeded: an owner has %d contacts > %d slots",
                  ctx->h_ctl->cap_needed, ctx->K);
    return fail(ctx, GG_ECAPACITY, buf);
  }
  if (out) {
    std::vector<Acc> acc(ctx->E);
    CK(cudaMemcpy(acc.data(), D.acc, sizeof(Acc) * ctx->E, cudaMemcpyDeviceToHost));
    for (int e = 0; e < ctx->E; ++e) {
      const Acc& a = acc[e];
      gg_report* o = out + e;
      std::memset(o, 0, sizeof(gg_report));
      o->n_contacts = static_cast<int64_t>(a.n_pp);
      o->n_candidates = static_cast<int64_t>(a.n_cand);
      o->n_body_contacts = static_cast<int64_t>(a.n_body);
      o->n_coincident = static_cast<int64_t>(a.n_coinc);
      o->n_degenerate = static_cast<int64_t>(a.n_deg);
      double mp;
      std::memcpy(&mp, &a.max_psi_bits, sizeof(double));
      o->max_penetration = mp;
    }
  }
  return GG_OK;
}

static int stage_bodies(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies) {
  CK(cudaStreamSynchronize(ctx->stream));
  int st = ensure_batch(ctx, n_steps, n_bodies);
  if (st != GG_OK) return st;
  if (ctx->D.nb != n_bodies) {
    ctx->D.nb = n_bodies;
    ctx->graph_dirty = true;
  }
  if (n_bodies > 0) {
    const size_t bytes = sizeof(gg_body) * static_cast<size_t>(n_steps) * ctx->E * n_bodies;
    std::memcpy(ctx->h_bodies, bodies, bytes);
    CK(cudaMemcpyAsync(ctx->d_bodies, ctx->h_bodies, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ctx->graph_dirty) {
    st = build_graph(ctx);
    if (st != GG_OK) return st;
  }
  refresh_dev(ctx);
  return GG_OK;
}

int gg_bench_steps(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies,
                   int64_t flush_bytes, float* step_ms) {
  if (!ctx || n_steps < 1 || !step_ms) return fail(ctx, GG_EINVAL, "bad bench arguments");
  DeviceGuard guard(ctx->device);
  int st = stage_bodies(ctx, n_steps, bodies, n_bodies);
  if (st != GG_OK) return st;
  if (flush_bytes > ctx->flush_bytes) {
    dfree(ctx, ctx->flush_buf);
    ctx->flush_buf = nullptr;
    char* fb = nullptr;
    CK(dalloc(ctx, &fb, static_cast<size_t>(flush_bytes)));
    ctx->flush_buf = fb;
    ctx->flush_bytes = flush_bytes;
  }
  st = ensure_events(ctx, 2 * static_cast<size_t>(n_steps));
  if (st != GG_OK) return st;
  st = begin_batch(ctx, ctx->stream);
  if (st != GG_OK) return st;
  for (int i = 0; i < n_steps; ++i) {
    if (flush_bytes > 0)
      CK(cudaMemsetAsync(ctx->flush_buf, i & 0xff, static_cast<size_t>(flush_bytes), ctx->stream));
    CK(cudaEventRecord(ctx->evpool[2 * i], ctx->stream));
    st = launch_step(ctx);
    if (st != GG_OK) return st;
    CK(cudaEventRecord(ctx->evpool[2 * i + 1], ctx->stream));
  }
  ctx->launches += 1;
  ctx->last_batch = n_steps;
  ctx->last_nb = n_bodies;
  ctx->tap_uncommitted = false;
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n_steps; ++i)
    CK(cudaEventElapsedTime(&step_ms[i], ctx->evpool[2 * i], ctx->evpool[2 * i + 1]));
  return GG_OK;
}

int gg_profile_steps(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies,
                     float* kind_ms, int32_t* kind_launches) {
  if (!ctx || n_steps < 1 || !kind_ms) return fail(ctx, GG_EINVAL, "bad profile arguments");
  DeviceGuard guard(ctx->device);
  int st = stage_bodies(ctx, n_steps, bodies, n_bodies);
  if (st != GG_OK) return st;
  const int per = 40;
  st = ensure_events(ctx, static_cast<size_t>(per + 1));
  if (st != GG_OK) return st;
  for (int k = 0; k < kProfKinds; ++k) {
    kind_ms[k] = 0.f;
    if (kind_launches) kind_launches[k] = 0;
  }
  std::vector<int> kinds(per + 1);
  st = begin_batch(ctx, ctx->stream);
  if (st != GG_OK) return st;
  for (int i = 0; i < n_steps; ++i) {
    const int resort = ctx->since_resort >= ctx->resort_every ? 1 : 0;
    ctx->since_resort = resort ? 1 : ctx->since_resort + 1;
    ctx->launches += kernels_per_step(ctx, resort);
    const int m = enqueue_step_profiled(ctx, resort, ctx->evpool.data(), kinds.data());
    if (m < 0) return fail(ctx, GG_ECUDA, "profiled launch failed");
    CK(cudaStreamSynchronize(ctx->stream));
    for (int e = 0; e < m; ++e) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ctx->evpool[e], ctx->evpool[e + 1]));
      kind_ms[kinds[e]] += t;
      if (kind_launches && kinds[e] > 0) kind_launches[kinds[e]] += 1;
    }
  }
  ctx->launches += 1;
  ctx->last_batch = n_steps;
  ctx->last_nb = n_bodies;
  ctx->tap_uncommitted = false;
  return GG_OK;
}

const char* gg_profile_kind_name(int32_t k) {
  return (k >= 0 && k < kProfKinds) ? kProfNames[k] : "";
}

int gg_last_batch_ms(gg_ctx* ctx, float* ms) {
  if (!ctx || !ms) return GG_EINVAL;
  DeviceGuard guard(ctx->device);
  CK(cudaEventSynchronize(ctx->ev1));
  CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  return GG_OK;
}

}  // extern "C"
namespace {
std::string nonfinite_message(gg_ctx* ctx, int err_step, std::vector<int> bad);
}
extern "C" {

int gg_sync(gg_ctx* ctx, gg_report* reports, double* body_momentum, int32_t cap,
            int32_t* n_done, int32_t* err_step) {
  if (!ctx) return GG_EINVAL;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(ctx->h_ctl, ctx->D.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  const Ctl& c = *ctx->h_ctl;
  const int done = std::min(c.step, ctx->last_batch);
  if (n_done) *n_done = done;
  if (err_step) *err_step = c.err ? c.err_step : -1;
  const int ncopy = std::min(done, cap);
  if (reports && ncopy > 0)
    CK(cudaMemcpy(reports, ctx->d_reports, sizeof(gg_report) * ncopy * ctx->E,
                  cudaMemcpyDeviceToHost));
  if (body_momentum && ncopy > 0 && ctx->last_nb > 0)
    CK(cudaMemcpy(body_momentum, ctx->d_bm, sizeof(double) * 3 * ctx->last_nb * ctx->E * ncopy,
                  cudaMemcpyDeviceToHost));
  if (!c.err) return GG_OK;
  char buf[512];
  switch (c.err) {
    case GG_EPOSITIONS:
      return fail(ctx, GG_EPOSITIONS, "positions must be finite");
    case GG_ENONFINITE: {
      // every particle whose correction is non-finite (D.bad: uid + 1 per
      // physical index, written only on failure), then cleared
      std::vector<int> flags(ctx->n);
      CK(cudaMemcpy(flags.data(), ctx->D.bad, sizeof(int) * ctx->n, cudaMemcpyDeviceToHost));
      CK(cudaMemset(ctx->D.bad, 0, sizeof(int) * ctx->n));
      std::vector<int> bad;
      for (int f : flags)
        if (f) bad.push_back(f - 1);
      if (bad.empty()) bad.assign(c.bad_uid, c.bad_uid + std::min(c.n_bad, kMaxBad));
      const int es = c.err_step;
      return fail(ctx, GG_ENONFINITE, nonfinite_message(ctx, es, bad));
    }
    case GG_ECAPACITY:
      std::snprintf(buf, sizeof(buf),
                    "contact capacity exceeded: an owner has %d contacts > %d slots",
                    c.cap_needed, ctx->K);
      return fail(ctx, GG_ECAPACITY, buf);
    case GG_EBUCKET:
      return fail(ctx, GG_EINVAL,
                  "hash table too small: the neighbour buckets of a particle hold more than "
                  "27 x 65534 particles (raise hashmap_size)");
    default:
      return fail(ctx, c.err, "device error");
  }
}

int gg_required_contacts(gg_ctx* ctx) {
  return ctx && ctx->h_ctl ? ctx->h_ctl->cap_needed : 0;
}

static int drive_slot(gg_ctx* ctx, int32_t slot, gg_ctx::DriveSlot** out) {
  if (slot < 0 || slot >= std::max(ctx->max_bodies, 1)) return fail(ctx, GG_EINVAL, "body slot out of range");
  if (static_cast<int>(ctx->drive.size()) <= slot) ctx->drive.resize(slot + 1);
  *out = &ctx->drive[slot];
  return GG_OK;
}

int gg_drive_fixed(gg_ctx* ctx, int32_t slot, const gg_body* rows) {
  if (!ctx || !rows) return GG_EINVAL;
  gg_ctx::DriveSlot* ds = nullptr;
  int st = drive_slot(ctx, slot, &ds);
  if (st != GG_OK) return st;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  if (!ds->d_fixed) CK(dalloc(ctx, &ds->d_fixed, ctx->E));
  CK(cudaMemcpy(ds->d_fixed, rows, sizeof(gg_body) * ctx->E, cudaMemcpyHostToDevice));
  ds->kind = 1;
  return GG_OK;
}

int gg_drive_track(gg_ctx* ctx, int32_t slot, const gg_body* tmpl, const double lo[3], const double hi[3],
                   const double* x, const double* y, const double* theta, double z, double scale_v,
                   double scale_omega, const double base_pose[16]) {
  if (!ctx || !tmpl || !x || !y || !theta || !base_pose) return GG_EINVAL;
  if (tmpl->bounded && (!lo || !hi)) return fail(ctx, GG_EINVAL, "bounded template needs local bounds");
  gg_ctx::DriveSlot* ds = nullptr;
  int st = drive_slot(ctx, slot, &ds);
  if (st != GG_OK) return st;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const int E = ctx->E;
  if (!ds->d_state) CK(dalloc(ctx, &ds->d_state, 3 * static_cast<size_t>(E)));
  if (!ds->d_action) CK(dalloc(ctx, &ds->d_action, 2 * static_cast<size_t>(E)));
  CK(cudaMemcpy(ds->d_state, x, sizeof(double) * E, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds->d_state + E, y, sizeof(double) * E, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds->d_state + 2 * E, theta, sizeof(double) * E, cudaMemcpyHostToDevice));
  CK(cudaMemset(ds->d_action, 0, sizeof(double) * 2 * E));
  DriveTrack& P = ds->P;
  P = DriveTrack{};
  P.x = ds->d_state;
  P.y = ds->d_state + E;
  P.theta = ds->d_state + 2 * E;
  P.action = ds->d_action;
  P.z = z;
  P.scale_v = scale_v;
  P.scale_omega = scale_omega;
  for (int i = 0; i < 16; ++i) P.base[i] = base_pose[i];
  for (int a = 0; a < 3; ++a) {
    P.lo[a] = lo ? lo[a] : 0.0;
    P.hi[a] = hi ? hi[a] : 0.0;
  }
  P.tmpl = *tmpl;
  ds->kind = 2;
  return GG_OK;
}

int gg_drive_chain(gg_ctx* ctx, int32_t slot, const gg_body* tmpl, const double lo[3], const double hi[3],
                   int32_t n_links, int32_t link_index, const int32_t* parents, const int32_t* prismatic,
                   const double* origins, const double* axes, const double* limits,
                   const double base_pose[16], const double* q) {
  if (!ctx || !tmpl || !parents || !prismatic || !origins || !axes || !limits || !base_pose || !q)
    return GG_EINVAL;
  if (n_links < 1 || n_links > kChainMax || link_index < 0 || link_index >= n_links)
    return fail(ctx, GG_EINVAL, "chain: 1..16 links and a link index among them");
  for (int i = 0; i < n_links; ++i)
    if (parents[i] >= i) return fail(ctx, GG_EINVAL, "chain: links must follow their parents");
  if (tmpl->bounded && (!lo || !hi)) return fail(ctx, GG_EINVAL, "bounded template needs local bounds");
  gg_ctx::DriveSlot* ds = nullptr;
  int st = drive_slot(ctx, slot, &ds);
  if (st != GG_OK) return st;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const size_t EJ = static_cast<size_t>(ctx->E) * n_links;
  if (ds->d_state) dfree(ctx, ds->d_state);
  if (ds->d_action) dfree(ctx, ds->d_action);
  ds->d_state = nullptr;
  ds->d_action = nullptr;
  CK(dalloc(ctx, &ds->d_state, EJ));
  CK(dalloc(ctx, &ds->d_action, EJ));
  CK(cudaMemcpy(ds->d_state, q, sizeof(double) * EJ, cudaMemcpyHostToDevice));
  CK(cudaMemset(ds->d_action, 0, sizeof(double) * EJ));
  DriveChain& C = ds->C;
  C = DriveChain{};
  C.q = ds->d_state;
  C.cmd = ds->d_action;
  C.J = n_links;
  C.link = link_index;
  for (int i = 0; i < n_links; ++i) {
    C.parent[i] = parents[i];
    C.prismatic[i] = prismatic[i];
    for (int r = 0; r < 12; ++r) C.origin[i][r] = origins[16 * i + r];
    for (int a = 0; a < 3; ++a) C.axis[i][a] = axes[3 * i + a];
    C.limit[i] = limits[i];
  }
  for (int r = 0; r < 12; ++r) C.base[r] = base_pose[r];
  for (int a = 0; a < 3; ++a) {
    C.lo[a] = lo ? lo[a] : 0.0;
    C.hi[a] = hi ? hi[a] : 0.0;
  }
  C.tmpl = *tmpl;
  ds->kind = 3;
  return GG_OK;
}

int gg_drive_command(gg_ctx* ctx, int32_t slot, const double* actions) {
  if (!ctx || !actions) return GG_EINVAL;
  if (slot < 0 || slot >= static_cast<int>(ctx->drive.size()) || ctx->drive[slot].kind < 2)
    return fail(ctx, GG_EINVAL, "no track or chain driver on this body slot");
  DeviceGuard guard(ctx->device);
  const int E = ctx->E;
  gg_ctx::DriveSlot& ds = ctx->drive[slot];
  const size_t m = static_cast<size_t>(E) * (ds.kind == 2 ? 2 : ds.C.J);
  std::vector<double> a(actions, actions + m);
  if (ds.kind == 2)
    for (double& u : a) u = u < -1.0 ? -1.0 : (u > 1.0 ? 1.0 : u);  // TrackSteeringDriver.command clip
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(ds.d_action, a.data(), sizeof(double) * m, cudaMemcpyHostToDevice));
  return GG_OK;
}

int gg_drive_chain_state(gg_ctx* ctx, int32_t slot, double* q) {
  if (!ctx || !q) return GG_EINVAL;
  if (slot < 0 || slot >= static_cast<int>(ctx->drive.size()) || ctx->drive[slot].kind != 3)
    return fail(ctx, GG_EINVAL, "no chain driver on this body slot");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const gg_ctx::DriveSlot& ds = ctx->drive[slot];
  CK(cudaMemcpy(q, ds.d_state, sizeof(double) * ctx->E * ds.C.J, cudaMemcpyDeviceToHost));
  return GG_OK;
}

int gg_drive_state(gg_ctx* ctx, int32_t slot, double* x, double* y, double* theta) {
  if (!ctx) return GG_EINVAL;
  if (slot < 0 || slot >= static_cast<int>(ctx->drive.size()) || ctx->drive[slot].kind != 2)
    return fail(ctx, GG_EINVAL, "no track driver on this body slot");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const int E = ctx->E;
  const double* d = ctx->drive[slot].d_state;
  if (x) CK(cudaMemcpy(x, d, sizeof(double) * E, cudaMemcpyDeviceToHost));
  if (y) CK(cudaMemcpy(y, d + E, sizeof(double) * E, cudaMemcpyDeviceToHost));
  if (theta) CK(cudaMemcpy(theta, d + 2 * E, sizeof(double) * E, cudaMemcpyDeviceToHost));
  return GG_OK;
}

int gg_step_resume(gg_ctx* ctx, int32_t first, int32_t n_steps, int32_t mode) {
  if (!ctx) return GG_EINVAL;
  if (first < 0 || n_steps < 1 || first + n_steps > ctx->batch_cap || ctx->D.nb < 1)
    return fail(ctx, GG_EINVAL, "gg_step_resume: rows outside the last batch");
  if (mode != ctx->pipeline) return fail(ctx, GG_EINVAL, "gg_step_resume: pipeline mode changed");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const size_t per = static_cast<size_t>(ctx->E) * ctx->D.nb;
  if (first > 0) {
    // the remaining rows to the front (a temporary: the ranges may overlap)
    gg_body* tmp = nullptr;
    CK(cudaMalloc(&tmp, sizeof(gg_body) * per * n_steps));
    CK(cudaMemcpy(tmp, ctx->d_bodies + per * first, sizeof(gg_body) * per * n_steps, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(ctx->d_bodies, tmp, sizeof(gg_body) * per * n_steps, cudaMemcpyDeviceToDevice));
    cudaFree(tmp);
  }
  int st;
  if (ctx->graph_dirty) {
    st = build_graph(ctx);
    if (st != GG_OK) return st;
  }
  refresh_dev(ctx);
  st = begin_batch(ctx, ctx->stream);
  if (st != GG_OK) return st;
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  for (int i = 0; i < n_steps; ++i) {
    st = launch_step(ctx);
    if (st != GG_OK) return st;
  }
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->launches += 1;
  ctx->last_batch = n_steps;
  ctx->tap_uncommitted = false;
  return GG_OK;
}

int gg_batch_reports(gg_ctx* ctx, int32_t first, int32_t count, gg_report* reports, double* body_momentum) {
  if (!ctx) return GG_EINVAL;
  if (first < 0 || count < 0 || first + count > ctx->last_batch)
    return fail(ctx, GG_EINVAL, "report range outside the last batch");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const size_t E = static_cast<size_t>(ctx->E);
  if (reports && count > 0)
    CK(cudaMemcpy(reports, ctx->d_reports + first * E, sizeof(gg_report) * count * E, cudaMemcpyDeviceToHost));
  if (body_momentum && count > 0 && ctx->last_nb > 0) {
    const size_t per = 3 * static_cast<size_t>(ctx->last_nb) * E;
    CK(cudaMemcpy(body_momentum, ctx->d_bm + first * per, sizeof(double) * count * per, cudaMemcpyDeviceToHost));
  }
  return GG_OK;
}

int gg_tap_hash(gg_ctx* ctx, int64_t* cells, int64_t* hashes, int64_t* order) {
  if (!ctx) return GG_EINVAL;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  int st = ensure_stage(ctx);
  if (st != GG_OK) return st;
  const long long n = ctx->n;
  refresh_dev(ctx);
  const Dev D = pass_dev(ctx, 0, 0);
  cudaStream_t s = ctx->stream;
  st = begin_batch(ctx, s);
  if (st != GG_OK) return st;
  st = enqueue_sort_pass(ctx, D, s);
  if (st != GG_OK) return st;
  long long* tmp = reinterpret_cast<long long*>(ctx->d_stage);  // 6n doubles = room for 5n i64
  k_tap_cells<<<ctx->nblocks, kBlock, 0, s>>>(D, tmp, tmp + 3 * n);
  k_tap_order<<<ctx->nblocks, kBlock, 0, s>>>(D, tmp + 4 * n);
  ctx->launches += 10;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(ctx->h_ctl, D.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  if (ctx->h_ctl->err == GG_EPOSITIONS) return fail(ctx, GG_EPOSITIONS, "positions must be finite");
  if (cells) CK(cudaMemcpy(cells, tmp, sizeof(long long) * 3 * n, cudaMemcpyDeviceToHost));
  if (hashes) CK(cudaMemcpy(hashes, tmp + 3 * n, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  if (order) CK(cudaMemcpy(order, tmp + 4 * n, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  return GG_OK;
}

}  // extern "C"

namespace {

// One detected contact as the reference's ContactSet row (contact.py:244-300).
struct TapRec {
  int owner, other, kind;
  long long key;  // pp: partner's position in bucket order; body: 0
  float4 geo, vb;
};

// Contacts recorded by the last detection (step or gg_detect), in the
// reference's ContactSet order: particle contacts by owner, within an owner
// in candidate order — buckets by ascending hash, a bucket's particles in
// stable order, i.e. ascending position in the bucket-ordered array Xh
// (broadphase.py:149-182) — then body contacts body by body, each body's by
// owner (contact.py:274-298).
int collect_contacts(gg_ctx* ctx, std::vector<TapRec>& out) {
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const long long n = ctx->n;
  const long long cap = ctx->D.cap_tot;
  std::vector<int2> ci(n);
  std::vector<int> uid(n), oth(cap);
  std::vector<float4> geo(cap), vb(cap), xh(n);
  int ucur = 0;
  CK(cudaMemcpy(&ucur, &ctx->D.ctl->ucur, sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ci.data(), ctx->D.cinfo, sizeof(int2) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(uid.data(), ctx->D.UID[ucur], sizeof(int) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(oth.data(), ctx->D.coth, sizeof(int) * cap, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(geo.data(), ctx->D.cgeo, sizeof(float4) * cap, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(vb.data(), ctx->D.cvb, sizeof(float4) * cap, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(xh.data(), ctx->D.Xh, sizeof(float4) * n, cudaMemcpyDeviceToHost));
  std::vector<long long> pos(n, 0);  // physical index -> position in bucket order
  for (long long m = 0; m < n; ++m) {
    int q;
    std::memcpy(&q, &xh[m].w, sizeof(int));
    if (q >= 0 && q < n) pos[q] = m;
  }
  out.clear();
  for (long long k = 0; k < n; ++k) {
    for (int s = 0; s < ci[k].y; ++s) {
      const size_t idx = s < kFixedSlots ? static_cast<size_t>(s) * n + k
                                         : static_cast<size_t>(ci[k].x) + s - kFixedSlots;
      const int j = oth[idx];
      if (j == kNullContact) continue;  // a prefilter pass that is no contact
      TapRec r;
      r.owner = uid[k];
      r.kind = j >= 0 ? 0 : 1;
      r.other = j >= 0 ? uid[j] : -(j + 1);
      r.key = j >= 0 ? pos[j] : 0;
      r.geo = geo[idx];
      r.vb = j >= 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : vb[idx];
      out.push_back(r);
    }
  }
  std::sort(out.begin(), out.end(), [](const TapRec& a, const TapRec& b) {
    if (a.kind != b.kind) return a.kind < b.kind;
    if (a.kind == 0) return a.owner != b.owner ? a.owner < b.owner : a.key < b.key;
    return a.other != b.other ? a.other < b.other : a.owner < b.owner;
  });
  return GG_OK;
}

// The reference's SolverError text (contact.py:503-509): the first five
// particles whose correction is non-finite and the first five indices of
// their contacts in ContactSet order.  The contacts are those of the failing
// step's input state (the state is not committed on failure), detected again
// with that step's body rows.
std::string nonfinite_message(gg_ctx* ctx, int err_step, std::vector<int> bad) {
  std::sort(bad.begin(), bad.end());
  bad.erase(std::unique(bad.begin(), bad.end()), bad.end());
  std::string s = "non-finite velocity correction for particles [";
  for (size_t i = 0; i < bad.size() && i < 5; ++i) {
    if (i) s += ", ";
    s += std::to_string(bad[i]);
  }
  s += "] (contacts [";
  std::vector<TapRec> recs;
  bool ok = ctx->E == 1 && err_step >= 0;
  if (ok) {
    refresh_dev(ctx);
    Dev D = pass_dev(ctx, 0, 0);
    D.bodies = ctx->d_bodies + static_cast<long long>(err_step) * ctx->E * D.nb;
    cudaStream_t st = ctx->stream;
    ok = begin_batch(ctx, st) == GG_OK && enqueue_sort_pass(ctx, D, st) == GG_OK;
    if (ok) {
      k_narrow<false><<<narrow_blocks(ctx->n), kNarrowBlock, sizeof(NarrowSmemN), st>>>(D);
      ctx->launches += 9;
      ok = cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess &&
           collect_contacts(ctx, recs) == GG_OK;
    }
  }
  int shown = 0;
  for (size_t c = 0; ok && c < recs.size() && shown < 5; ++c)
    if (std::binary_search(bad.begin(), bad.end(), recs[c].owner)) {
      if (shown++) s += ", ";
      s += std::to_string(c);
    }
  s += "])";
  return s;
}

// RAII device scratch for the context-level entry points below
struct DevScratch {
  std::vector<void*> ptrs;
  template <typename T>
  cudaError_t get(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) {
      ptrs.push_back(q);
      *p = static_cast<T*>(q);
    }
    return e;
  }
  ~DevScratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

extern "C" {

int gg_tap_contacts(gg_ctx* ctx, int64_t cap_out, int64_t* count, int32_t* owner, int32_t* other,
                    int32_t* kind, double* psi, double* e1, double* vj) {
  if (!ctx || !count) return GG_EINVAL;
  std::vector<TapRec> recs;
  int st = collect_contacts(ctx, recs);
  if (st != GG_OK) return st;
  const long long m = static_cast<long long>(recs.size());
  for (long long o = 0; o < m && o < cap_out; ++o) {
    const TapRec& r = recs[o];
    if (owner) owner[o] = r.owner;
    if (other) other[o] = r.other;
    if (kind) kind[o] = r.kind;
    if (psi) psi[o] = r.geo.w;
    if (e1) {
      e1[3 * o] = r.geo.x;
      e1[3 * o + 1] = r.geo.y;
      e1[3 * o + 2] = r.geo.z;
    }
    if (vj) {
      vj[3 * o] = r.vb.x;
      vj[3 * o + 1] = r.vb.y;
      vj[3 * o + 2] = r.vb.z;
    }
  }
  *count = m;
  return GG_OK;
}

int gg_position_cells(gg_ctx* ctx, const double* x, int64_t n, double radius, int64_t* cells) {
  if (!ctx) return GG_EINVAL;
  if (n < 0 || (n > 0 && (!x || !cells))) return fail(ctx, GG_EINVAL, "position_cells: bad arguments");
  if (n == 0) return GG_OK;
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  CK(cudaStreamSynchronize(s));
  DevScratch tmp;
  double* d_x = nullptr;
  long long* d_c = nullptr;
  int* d_bad = nullptr;
  CK(tmp.get(&d_x, 3 * n));
  CK(tmp.get(&d_c, 3 * n));
  CK(tmp.get(&d_bad, 1));
  CK(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
  CK(cudaMemcpyAsync(d_x, x, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  k_cells_f64<<<static_cast<unsigned>((n + kBlock - 1) / kBlock), kBlock, 0, s>>>(d_x, n, 2.0 * radius,
                                                                                 d_c, d_bad);
  ctx->launches += 1;
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(cells, d_c, sizeof(long long) * 3 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad) return fail(ctx, GG_EPOSITIONS, "positions must be finite");
  return GG_OK;
}

int gg_tap_candidates(gg_ctx* ctx, int64_t cap_out, int64_t* count, int64_t* ci, int64_t* cj) {
  if (!ctx || !count) return GG_EINVAL;
  if (ctx->E != 1) return fail(ctx, GG_EINVAL, "gg_tap_candidates: single-scene contexts only");
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  const long long n = ctx->n;
  refresh_dev(ctx);
  const Dev D = pass_dev(ctx, 0, 0);
  cudaStream_t s = ctx->stream;
  int st = begin_batch(ctx, s);
  if (st != GG_OK) return st;
  st = enqueue_sort_pass(ctx, D, s);
  if (st != GG_OK) return st;
  DevScratch tmp;
  long long *d_cnt = nullptr, *d_off = nullptr;
  CK(tmp.get(&d_cnt, n));
  CK(tmp.get(&d_off, n));
  k_cand_count<<<ctx->nblocks, kBlock, 0, s>>>(D, d_cnt);
  ctx->launches += 8;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(ctx->h_ctl, D.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  if (ctx->h_ctl->err == GG_EPOSITIONS) return fail(ctx, GG_EPOSITIONS, "positions must be finite");
  std::vector<long long> cnt(n), off(n);
  CK(cudaMemcpy(cnt.data(), d_cnt, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  long long total = 0;
  for (long long i = 0; i < n; ++i) {
    off[i] = total;
    total += cnt[i];
  }
  *count = total;
  if (!ci || !cj || cap_out < total || total == 0) return GG_OK;
  long long *d_ci = nullptr, *d_cj = nullptr;
  CK(tmp.get(&d_ci, total));
  CK(tmp.get(&d_cj, total));
  CK(cudaMemcpyAsync(d_off, off.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, s));
  k_cand_fill<<<ctx->nblocks, kBlock, 0, s>>>(D, d_off, d_ci, d_cj);
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ci, d_ci, sizeof(long long) * total, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(cj, d_cj, sizeof(long long) * total, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return GG_OK;
}

int gg_narrow_pairs(gg_ctx* ctx, const double* x, int64_t n, const int64_t* ci, const int64_t* cj,
                    int64_t m, double radius, const gg_body* bodies, int32_t n_bodies,
                    double* pp_e1, double* pp_psi, uint8_t* pp_colliding, int64_t* n_coincident,
                    uint8_t* b_near, uint8_t* b_hit, double* b_psi, double* b_normal, double* b_vj,
                    int64_t* n_degenerate) {
  if (!ctx) return GG_EINVAL;
  if (n < 0 || m < 0 || (n > 0 && !x) || (m > 0 && (!ci || !cj || !pp_e1 || !pp_psi || !pp_colliding)))
    return fail(ctx, GG_EINVAL, "narrowphase_candidates: bad arguments");
  if (n_bodies < 0 || (n_bodies > 0 && (!bodies || !b_near || !b_hit || !b_psi || !b_normal || !b_vj)))
    return fail(ctx, GG_EINVAL, "narrowphase_candidates: bad body arguments");
  if (!(radius > 0.0)) return fail(ctx, GG_EINVAL, "particle radius must be positive");
  for (long long t = 0; t < m; ++t)
    if (ci[t] < 0 || ci[t] >= n || cj[t] < 0 || cj[t] >= n)
      return fail(ctx, GG_EINVAL, "candidate index out of range");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  CK(cudaStreamSynchronize(s));
  DevScratch tmp;
  double *d_x = nullptr, *d_e1 = nullptr, *d_psi = nullptr, *d_bpsi = nullptr, *d_bn = nullptr,
         *d_bvj = nullptr;
  long long *d_ci = nullptr, *d_cj = nullptr;
  unsigned char *d_col = nullptr, *d_near = nullptr, *d_hit = nullptr;
  unsigned long long* d_cnt = nullptr;
  gg_body* d_bodies = nullptr;
  CK(tmp.get(&d_x, 3 * n));
  CK(tmp.get(&d_cnt, 2));
  CK(cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned long long), s));
  if (n > 0) CK(cudaMemcpyAsync(d_x, x, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  if (m > 0) {
    CK(tmp.get(&d_ci, m));
    CK(tmp.get(&d_cj, m));
    CK(tmp.get(&d_e1, 3 * m));
    CK(tmp.get(&d_psi, m));
    CK(tmp.get(&d_col, m));
    CK(cudaMemcpyAsync(d_ci, ci, sizeof(long long) * m, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_cj, cj, sizeof(long long) * m, cudaMemcpyHostToDevice, s));
    const double two_r = 2.0 * radius;
    k_pairs_pp<<<static_cast<unsigned>((m + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        d_x, d_ci, d_cj, m, two_r, two_r * two_r, 1e-12 * 1e-12, d_e1, d_psi, d_col, d_cnt);
    ctx->launches += 1;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(pp_e1, d_e1, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(pp_psi, d_psi, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(pp_colliding, d_col, m, cudaMemcpyDeviceToHost, s));
  }
  if (n_bodies > 0 && n > 0) {
    refresh_dev(ctx);
    const long long nb = n_bodies;
    CK(tmp.get(&d_bodies, nb));
    CK(tmp.get(&d_near, nb * n));
    CK(tmp.get(&d_hit, nb * n));
    CK(tmp.get(&d_bpsi, nb * n));
    CK(tmp.get(&d_bn, 3 * nb * n));
    CK(tmp.get(&d_bvj, 3 * nb * n));
    CK(cudaMemcpyAsync(d_bodies, bodies, sizeof(gg_body) * nb, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(d_hit, 0, nb * n, s));
    CK(cudaMemsetAsync(d_bpsi, 0, sizeof(double) * nb * n, s));
    CK(cudaMemsetAsync(d_bn, 0, sizeof(double) * 3 * nb * n, s));
    CK(cudaMemsetAsync(d_bvj, 0, sizeof(double) * 3 * nb * n, s));
    k_pairs_body<<<dim3(static_cast<unsigned>((n + kBlock - 1) / kBlock), static_cast<unsigned>(nb)),
                   kBlock, 0, s>>>(d_bodies, ctx->d_grids, ctx->d_gvals, d_x, n, radius, d_near,
                                   d_hit, d_bpsi, d_bn, d_bvj, d_cnt + 1);
    ctx->launches += 1;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(b_near, d_near, nb * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(b_hit, d_hit, nb * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(b_psi, d_bpsi, sizeof(double) * nb * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(b_normal, d_bn, sizeof(double) * 3 * nb * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(b_vj, d_bvj, sizeof(double) * 3 * nb * n, cudaMemcpyDeviceToHost, s));
  }
  unsigned long long cnt[2] = {0, 0};
  CK(cudaMemcpyAsync(cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (n_coincident) *n_coincident = static_cast<int64_t>(cnt[0]);
  if (n_degenerate) *n_degenerate = static_cast<int64_t>(cnt[1]);
  return GG_OK;
}

int gg_solve_contacts(gg_ctx* ctx, const gg_contact_list* c, int64_t n, const double* v,
                      const gg_params* p, int32_t n_bodies, int32_t first_sweep, int32_t n_sweeps,
                      double* dv, double* body_momentum, double* diag, int64_t* n_live) {
  if (!ctx) return GG_EINVAL;
  if (!c || !p || n < 0 || c->m < 0 || (n > 0 && (!v || !dv)) || n_bodies < 0 || first_sweep < 0 ||
      n_sweeps < 0 || (n_bodies > 0 && !body_momentum) || !diag)
    return fail(ctx, GG_EINVAL, "solve_contacts_pja: bad arguments");
  const long long m = c->m;
  if (m > 0 && (!c->owner || !c->kind || !c->other || !c->e1 || !c->psi || !c->vj))
    return fail(ctx, GG_EINVAL, "solve_contacts_pja: contact arrays missing");
  if (n >= (1ll << 31) || m >= (1ll << 31))
    return fail(ctx, GG_EINVAL, "solve_contacts_pja: at most 2^31 - 1 particles and contacts");
  // CSR of the contacts by owner, contact order kept (a stable counting sort)
  std::vector<int> rowptr(n + 1, 0), cidx(m);
  long long live = 0;
  for (long long k = 0; k < m; ++k) {
    const long long o = c->owner[k];
    if (o < 0 || o >= n) return fail(ctx, GG_EINVAL, "contact owner out of range");
    if (c->kind[k] == 0 && (c->other[k] < 0 || c->other[k] >= n))
      return fail(ctx, GG_EINVAL, "contact partner out of range");
    rowptr[o + 1] += 1;
    live += (!c->colliding || c->colliding[k]) ? 1 : 0;
  }
  if (n_live) *n_live = live;
  for (long long i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
  {
    std::vector<int> fillp(rowptr.begin(), rowptr.end() - 1);
    for (long long k = 0; k < m; ++k) cidx[fillp[c->owner[k]]++] = static_cast<int>(k);
  }
  if (n == 0 || m == 0 || n_sweeps == 0) return GG_OK;  // dv stays as given (zeros)
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  CK(cudaStreamSynchronize(s));
  DevScratch tmp;
  int *d_row = nullptr, *d_cidx = nullptr;
  long long *d_kind = nullptr, *d_other = nullptr;
  unsigned char* d_mask = nullptr;
  double *d_e1 = nullptr, *d_e2 = nullptr, *d_e3 = nullptr, *d_psi = nullptr, *d_vj = nullptr,
         *d_v = nullptr, *d_dv[2] = {nullptr, nullptr};
  unsigned long long *d_bm = nullptr, *d_diag = nullptr;
  CK(tmp.get(&d_row, n + 1));
  CK(tmp.get(&d_cidx, m));
  CK(tmp.get(&d_kind, m));
  CK(tmp.get(&d_other, m));
  CK(tmp.get(&d_e1, 3 * m));
  CK(tmp.get(&d_e2, 3 * m));
  CK(tmp.get(&d_e3, 3 * m));
  CK(tmp.get(&d_psi, m));
  CK(tmp.get(&d_vj, 3 * m));
  CK(tmp.get(&d_v, 3 * n));
  CK(tmp.get(&d_dv[0], 3 * n));
  CK(tmp.get(&d_dv[1], 3 * n));
  CK(tmp.get(&d_bm, 3 * std::max(n_bodies, 1)));
  CK(tmp.get(&d_diag, 2));
  if (c->colliding) {
    CK(tmp.get(&d_mask, m));
    CK(cudaMemcpyAsync(d_mask, c->colliding, m, cudaMemcpyHostToDevice, s));
  }
  // vj0: body surface velocity, or velocities[other] for particle contacts
  // (contact.py:440-443) — gathered on the host while the copies run
  std::vector<double> vj0(c->vj, c->vj + 3 * m);
  for (long long k = 0; k < m; ++k)
    if (c->kind[k] == 0)
      for (int a = 0; a < 3; ++a) vj0[3 * k + a] = v[3 * c->other[k] + a];
  CK(cudaMemcpyAsync(d_row, rowptr.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_cidx, cidx.data(), sizeof(int) * m, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_kind, c->kind, sizeof(long long) * m, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_other, c->other, sizeof(long long) * m, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_e1, c->e1, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_psi, c->psi, sizeof(double) * m, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_vj, vj0.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_v, v, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_dv[0], dv, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(d_bm, 0, sizeof(unsigned long long) * 3 * std::max(n_bodies, 1), s));
  unsigned long long dg[2];
  std::memcpy(&dg[0], &diag[0], sizeof(double));
  std::memcpy(&dg[1], &diag[1], sizeof(double));
  if (!(diag[0] > 0.0)) dg[0] = 0ull;
  if (!(diag[1] >= 0.0)) dg[1] = 0x7ff0000000000000ull;
  CK(cudaMemcpyAsync(d_diag, dg, sizeof(dg), cudaMemcpyHostToDevice, s));
  const unsigned mb = static_cast<unsigned>((m + kBlock - 1) / kBlock);
  k_l1_frames<<<mb, kBlock, 0, s>>>(m, d_e1, d_mask, d_e2, d_e3);
  L1Solve L{};
  L.n = static_cast<int>(n);
  L.m = m;
  L.rowptr = d_row;
  L.cidx = d_cidx;
  L.kind = d_kind;
  L.other = d_other;
  L.mask = d_mask;
  L.e1 = d_e1;
  L.e2 = d_e2;
  L.e3 = d_e3;
  L.psi = d_psi;
  L.vj0 = d_vj;
  L.v = d_v;
  L.gamma = p->gamma;
  L.mu = p->friction;
  L.alpha = p->baumgarte_alpha;
  L.dt = p->timestep;
  L.mass = p->particle_mass;
  L.gdt0 = p->gdt[0];
  L.gdt1 = p->gdt[1];
  L.gdt2 = p->gdt[2];
  L.nb = n_bodies;
  L.bm_fix = d_bm;
  L.diag = d_diag;
  const unsigned nbk = static_cast<unsigned>((n + kBlock - 1) / kBlock);
  for (int it = 0; it < n_sweeps; ++it)
    k_l1_sweep<<<nbk, kBlock, 0, s>>>(L, d_dv[it & 1], d_dv[(it + 1) & 1]);
  ctx->launches += 1 + n_sweeps;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(dv, d_dv[n_sweeps & 1], sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
  std::vector<unsigned long long> bm(3 * std::max(n_bodies, 1));
  CK(cudaMemcpyAsync(bm.data(), d_bm, sizeof(unsigned long long) * bm.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(dg, d_diag, sizeof(dg), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < 3 * n_bodies; ++i)
    body_momentum[i] += static_cast<double>(static_cast<long long>(bm[i])) / kMomScale;
  std::memcpy(&diag[0], &dg[0], sizeof(double));
  std::memcpy(&diag[1], &dg[1], sizeof(double));
  // SolverError after the last sweep (contact.py:503-509)
  if (first_sweep + n_sweeps >= p->solver_iterations) {
    std::vector<int> bad;
    for (long long i = 0; i < n; ++i)
      if (!std::isfinite(dv[3 * i]) || !std::isfinite(dv[3 * i + 1]) || !std::isfinite(dv[3 * i + 2]))
        bad.push_back(static_cast<int>(i));
    if (!bad.empty()) {
      std::string msg = "non-finite velocity correction for particles [";
      for (size_t i = 0; i < bad.size() && i < 5; ++i) msg += (i ? ", " : "") + std::to_string(bad[i]);
      msg += "] (contacts [";
      int shown = 0;
      for (long long k = 0; k < m && shown < 5; ++k)
        if (std::binary_search(bad.begin(), bad.end(), static_cast<int>(c->owner[k])))
          msg += (shown++ ? ", " : "") + std::to_string(k);
      msg += "])";
      return fail(ctx, GG_ENONFINITE, msg);
    }
  }
  return GG_OK;
}

int gg_project_cone(gg_ctx* ctx, double* b, int64_t k, const double* psi, int32_t psi_scalar,
                    double mu, double alpha, double dt) {
  if (!ctx) return GG_EINVAL;
  if (mu < 0 || !(dt > 0)) return fail(ctx, GG_EINVAL, "require mu >= 0 and dt > 0");
  if (k < 0 || (k > 0 && (!b || !psi))) return fail(ctx, GG_EINVAL, "project_friction_cone: bad arguments");
  if (k == 0) return GG_OK;
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  CK(cudaStreamSynchronize(s));
  DevScratch tmp;
  double *d_b = nullptr, *d_psi = nullptr;
  const long long np_ = psi_scalar ? 1 : k;
  CK(tmp.get(&d_b, 3 * k));
  CK(tmp.get(&d_psi, np_));
  CK(cudaMemcpyAsync(d_b, b, sizeof(double) * 3 * k, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_psi, psi, sizeof(double) * np_, cudaMemcpyHostToDevice, s));
  k_cone<<<static_cast<unsigned>((k + kBlock - 1) / kBlock), kBlock, 0, s>>>(d_b, d_psi, k, psi_scalar,
                                                                             mu, alpha, dt);
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(b, d_b, sizeof(double) * 3 * k, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return GG_OK;
}

int gg_penetration(gg_ctx* ctx, const gg_body* body, const double* points, int64_t n,
                   double radius, double* psi, double* normal, int32_t* hit,
                   int64_t* n_degenerate) {
  if (!ctx || !body || (n > 0 && (!points || !psi || !normal || !hit)))
    return fail(ctx, GG_EINVAL, "null argument");
  if (!(radius > 0)) return fail(ctx, GG_EINVAL, "particle radius must be positive");
  if (body->kind == GG_GEOM_GRID && (body->grid_id < 0 || body->grid_id >= (int)ctx->grids.size()))
    return fail(ctx, GG_EINVAL, "unknown grid id");
  if (n_degenerate) *n_degenerate = 0;
  if (n == 0) return GG_OK;
  DeviceGuard guard(ctx->device);
  double* d = nullptr;
  unsigned long long* deg = nullptr;
  CK(cudaMalloc(&d, sizeof(double) * 7 * n + sizeof(int) * n));
  CK(cudaMalloc(&deg, sizeof(unsigned long long)));
  CK(cudaMemset(deg, 0, sizeof(unsigned long long)));
  CK(cudaMemcpy(d, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  double* dpsi = d + 3 * n;
  double* dn = d + 4 * n;
  int* dh = reinterpret_cast<int*>(d + 7 * n);
  k_penetration<<<blocks_for(n), kBlock, 0, ctx->stream>>>(*body, ctx->d_grids, ctx->d_gvals, d,
                                                            n, radius, dpsi, dn, dh, deg);
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  unsigned long long nd = 0;
  CK(cudaMemcpy(psi, dpsi, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(normal, dn, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hit, dh, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&nd, deg, sizeof(nd), cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(deg);
  if (n_degenerate) *n_degenerate = static_cast<int64_t>(nd);
  return GG_OK;
}

int gg_spatial_hash(gg_ctx* ctx, const int64_t* cells, int64_t k, int64_t n_h, int64_t* out) {
  if (n_h < 1) return fail(ctx, GG_EINVAL, "hash table size must be >= 1");
  if (k == 0) return GG_OK;
  if (!cells || !out) return fail(ctx, GG_EINVAL, "null argument");
  HashCfg H;
  H.n_h = n_h;
  H.pow2 = ((n_h & (n_h - 1)) == 0 && n_h <= (1ll << 32)) ? 1 : 0;
  H.mask = static_cast<uint32_t>(n_h - 1);
  long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(long long) * 4 * k);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  e = cudaMemcpy(d, cells, sizeof(long long) * 3 * k, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_hash_cells<<<blocks_for(k), kBlock>>>(reinterpret_cast<const long long*>(d), k, H, d + 3 * k);
    if (ctx) ctx->launches += 1;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d + 3 * k, sizeof(long long) * k, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gg_spatial_hash");
  return GG_OK;
}

int gg_host_register(void* ptr, int64_t bytes) {
  return cudaHostRegister(ptr, static_cast<size_t>(bytes), cudaHostRegisterDefault) == cudaSuccess
             ? GG_OK
             : GG_ECUDA;
}

int gg_host_unregister(void* ptr) {
  return cudaHostUnregister(ptr) == cudaSuccess ? GG_OK : GG_ECUDA;
}

void* gg_stream(gg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int gg_num_envs(const gg_ctx* ctx) { return ctx ? ctx->E : 0; }

int gg_env_box_stats(gg_ctx* ctx, const double lo[3], const double hi[3], double* reward,
                     int64_t* inside) {
  if (!ctx || !lo || !hi) return fail(ctx, GG_EINVAL, "null argument");
  for (int a = 0; a < 3; ++a)
    if (!(lo[a] < hi[a])) return fail(ctx, GG_EINVAL, "goal box requires min < max componentwise");
  DeviceGuard guard(ctx->device);
  const int E = ctx->E;
  double* d = nullptr;
  CK(cudaMalloc(&d, sizeof(double) * 2 * E));
  long long* di = reinterpret_cast<long long*>(d + E);
  k_env_box<<<E, kBlock, 0, ctx->stream>>>(ctx->D, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], d, di);
  ctx->launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess && reward) e = cudaMemcpy(reward, d, sizeof(double) * E, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && inside) e = cudaMemcpy(inside, di, sizeof(long long) * E, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gg_env_box_stats");
  return GG_OK;
}

}  // extern "C"

// ===========================================================================
// Slab domain decomposition (gg_slab.cuh).  All calls are on the context
// stream; *_pack calls synchronise (the host needs the counts to size the
// exchange), the others are asynchronous until gg_slab_finish.
// ===========================================================================
namespace {

Dev slab_dev(const gg_ctx* ctx) {
  Dev D = ctx->D;
  D.n = static_cast<int>(ctx->n_cur);
  D.n_own = static_cast<int>(ctx->n_own);
  D.resort = 0;
  D.key_morton = 0;
  return D;
}

int slab_check(gg_ctx* ctx) {
  if (!ctx) return GG_EINVAL;
  if (!ctx->slab_on) return fail(ctx, GG_EINVAL, "gg_slab_setup has not been called");
  return GG_OK;
}

}  // namespace

extern "C" {

int gg_slab_setup(gg_ctx* ctx, int64_t cell_lo, int64_t cell_hi, int32_t has_lo, int32_t has_hi) {
  if (!ctx) return GG_EINVAL;
  if (ctx->E != 1) return fail(ctx, GG_EINVAL, "slab mode needs a single-bed context");
  if (has_lo && has_hi && !(cell_lo < cell_hi)) return fail(ctx, GG_EINVAL, "empty slab");
  DeviceGuard guard(ctx->device);
  if (!ctx->d_scnt) {
    CK(dalloc(ctx, &ctx->d_scnt, 4));
    CK(cudaMallocHost(&ctx->h_scnt, sizeof(unsigned long long) * 4));
    CK(dalloc(ctx, &ctx->d_holes, ctx->n));
    CK(dalloc(ctx, &ctx->d_movers, ctx->n));
    CK(dalloc(ctx, &ctx->d_map[0], ctx->n));
    CK(dalloc(ctx, &ctx->d_map[1], ctx->n));
  }
  ctx->slab = SlabCfg{cell_lo, cell_hi, has_lo ? 1 : 0, has_hi ? 1 : 0};
  ctx->slab_on = true;
  int st = ensure_batch(ctx, 1, std::max(ctx->max_bodies, 1));
  if (st != GG_OK) return st;
  refresh_dev(ctx);
  ctx->n_cur = ctx->n_own;
  return begin_batch(ctx, ctx->stream);  // zero bucket/tile counts once
}

int gg_slab_load(gg_ctx* ctx, const double* x, const double* v, const int32_t* gid, int64_t n_own) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (n_own < 0 || n_own > ctx->n || (n_own > 0 && (!x || !v || !gid)))
    return fail(ctx, GG_EINVAL, "bad slab state (n_own exceeds the context capacity?)");
  DeviceGuard guard(ctx->device);
  st = ensure_stage(ctx);
  if (st != GG_OK) return st;
  ctx->n_own = ctx->n_cur = n_own;
  ctx->ghost_in[0] = ctx->ghost_in[1] = 0;
  if (ctx->d_n) {  // a reload after graph steps: the device counts follow
    const int nn[2] = {static_cast<int>(n_own), static_cast<int>(n_own)};
    CK(cudaMemcpy(ctx->d_n, nn, sizeof(nn), cudaMemcpyHostToDevice));
  }
  if (n_own == 0) return GG_OK;
  set_morton_window(ctx, nullptr, x, n_own, 3);
  const size_t b = sizeof(double) * 3 * static_cast<size_t>(n_own);
  CK(cudaMemcpyAsync(ctx->d_stage, x, b, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_stage + 3 * ctx->n, v, b, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_holes, gid, sizeof(int) * n_own, cudaMemcpyHostToDevice, ctx->stream));
  k_slab_load<<<blocks_for(n_own), kBlock, 0, ctx->stream>>>(slab_dev(ctx), ctx->d_stage,
                                                              ctx->d_stage + 3 * ctx->n, ctx->d_holes);
  ctx->launches += 1;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return GG_OK;
}

int gg_slab_migrate_pack(gg_ctx* ctx, void* send_lo, void* send_hi, int64_t cap, int64_t counts[2]) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (!counts) return fail(ctx, GG_EINVAL, "null counts");
  DeviceGuard guard(ctx->device);
  ctx->n_cur = ctx->n_own;  // ghosts of the previous step are dropped
  cudaStream_t s = ctx->stream;
  CK(cudaMemsetAsync(ctx->d_scnt, 0, sizeof(unsigned long long) * 4, s));
  const Dev D = slab_dev(ctx);
  if (ctx->n_own > 0)
    k_slab_emigrate<<<blocks_for(ctx->n_own), kBlock, 0, s>>>(
        D, ctx->slab, static_cast<SlabRec*>(send_lo), static_cast<SlabRec*>(send_hi), cap, ctx->d_scnt);
  CK(cudaMemcpyAsync(ctx->h_scnt, ctx->d_scnt, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  counts[0] = static_cast<int64_t>(ctx->h_scnt[0]);
  counts[1] = static_cast<int64_t>(ctx->h_scnt[1]);
  if (counts[0] > cap || counts[1] > cap)
    return fail(ctx, GG_ECAPACITY, "slab migration buffer too small");
  const long long n_em = counts[0] + counts[1];
  ctx->launches += 1;
  if (n_em > 0) {
    const int n_stay = static_cast<int>(ctx->n_own - n_em);
    k_slab_holes<<<blocks_for(ctx->n_own), kBlock, 0, s>>>(D, n_stay, ctx->d_holes, ctx->d_movers,
                                                            ctx->d_scnt);
    CK(cudaMemcpyAsync(ctx->h_scnt, ctx->d_scnt, sizeof(unsigned long long) * 4,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int m = static_cast<int>(ctx->h_scnt[2]);
    if (m > 0) k_slab_fill<<<blocks_for(m), kBlock, 0, s>>>(D, ctx->d_holes, ctx->d_movers, m);
    ctx->launches += 2;
    CK(cudaGetLastError());
    ctx->n_own = ctx->n_cur = n_stay;
  }
  return GG_OK;
}

static int slab_append(gg_ctx* ctx, const void* rec, int64_t m, long long at) {
  if (m <= 0) return GG_OK;
  if (!rec) return fail(ctx, GG_EINVAL, "null receive buffer");
  k_slab_append<<<blocks_for(m), kBlock, 0, ctx->stream>>>(slab_dev(ctx), static_cast<const SlabRec*>(rec),
                                                           static_cast<int>(m), static_cast<int>(at));
  ctx->launches += 1;
  CK(cudaGetLastError());
  return GG_OK;
}

int gg_slab_migrate_unpack(gg_ctx* ctx, const void* recv_lo, int64_t n_lo, const void* recv_hi,
                           int64_t n_hi) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (n_lo < 0 || n_hi < 0 || ctx->n_own + n_lo + n_hi > ctx->n)
    return fail(ctx, GG_ECAPACITY, "slab particle capacity exceeded by immigrants");
  DeviceGuard guard(ctx->device);
  st = slab_append(ctx, recv_lo, n_lo, ctx->n_own);
  if (st == GG_OK) st = slab_append(ctx, recv_hi, n_hi, ctx->n_own + n_lo);
  if (st != GG_OK) return st;
  ctx->n_own += n_lo + n_hi;
  ctx->n_cur = ctx->n_own;
  return GG_OK;
}

int gg_slab_resort(gg_ctx* ctx) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (ctx->n_own == 0) return GG_OK;
  DeviceGuard guard(ctx->device);
  ctx->n_cur = ctx->n_own;
  Dev D = slab_dev(ctx);
  D.resort = 1;
  D.key_morton = 1;
  cudaStream_t s = ctx->stream;
  k_slab_set_n<<<1, 1, 0, s>>>(D);
  const int nb_save = ctx->nblocks;
  ctx->nblocks = blocks_for(ctx->n_own);
  st = enqueue_sort_pass(ctx, D, s);
  ctx->nblocks = nb_save;
  if (st != GG_OK) return st;
  k_slab_commit_sorted<<<blocks_for(ctx->n_own), kBlock, 0, s>>>(D);
  ctx->launches += 8;
  CK(cudaGetLastError());
  return GG_OK;
}

int gg_slab_ghost_pack(gg_ctx* ctx, void* send_lo, void* send_hi, int64_t cap, int64_t counts[2]) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (!counts) return fail(ctx, GG_EINVAL, "null counts");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  ctx->n_cur = ctx->n_own;
  CK(cudaMemsetAsync(ctx->d_scnt, 0, sizeof(unsigned long long) * 4, s));
  if (ctx->n_own > 0)
    k_slab_ghosts<<<blocks_for(ctx->n_own), kBlock, 0, s>>>(
        slab_dev(ctx), ctx->slab, static_cast<SlabRec*>(send_lo), static_cast<SlabRec*>(send_hi),
        ctx->d_map[0], ctx->d_map[1], std::min<long long>(cap, ctx->n), ctx->d_scnt);
  ctx->launches += 1;
  CK(cudaMemcpyAsync(ctx->h_scnt, ctx->d_scnt, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  counts[0] = static_cast<int64_t>(ctx->h_scnt[0]);
  counts[1] = static_cast<int64_t>(ctx->h_scnt[1]);
  if (counts[0] > cap || counts[1] > cap) return fail(ctx, GG_ECAPACITY, "slab ghost buffer too small");
  ctx->ghost_out[0] = counts[0];
  ctx->ghost_out[1] = counts[1];
  return GG_OK;
}

int gg_slab_ghost_unpack(gg_ctx* ctx, const void* recv_lo, int64_t n_lo, const void* recv_hi,
                         int64_t n_hi) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (n_lo < 0 || n_hi < 0 || ctx->n_own + n_lo + n_hi > ctx->n)
    return fail(ctx, GG_ECAPACITY, "slab particle capacity exceeded by ghosts");
  DeviceGuard guard(ctx->device);
  st = slab_append(ctx, recv_lo, n_lo, ctx->n_own);
  if (st == GG_OK) st = slab_append(ctx, recv_hi, n_hi, ctx->n_own + n_lo);
  if (st != GG_OK) return st;
  ctx->ghost_in[0] = n_lo;
  ctx->ghost_in[1] = n_hi;
  ctx->n_cur = ctx->n_own + n_lo + n_hi;
  return GG_OK;
}

int gg_slab_detect(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (n_bodies < 0 || (n_bodies > 0 && !bodies)) return fail(ctx, GG_EINVAL, "bad bodies");
  for (int b = 0; b < n_bodies; ++b)
    if (bodies[b].kind < GG_GEOM_SPHERE || bodies[b].kind > GG_GEOM_GRID ||
        (bodies[b].kind == GG_GEOM_GRID && (bodies[b].grid_id < 0 || bodies[b].grid_id >= (int)ctx->grids.size())))
      return fail(ctx, GG_EINVAL, "bad body");
  DeviceGuard guard(ctx->device);
  st = stage_bodies(ctx, 1, bodies, n_bodies);
  if (st != GG_OK) return st;
  cudaStream_t s = ctx->stream;
  const Dev D = slab_dev(ctx);
  k_batch_begin<<<1, 256, 0, s>>>(D);  // step / error / accumulators (bucket counts stay zero)
  k_slab_set_n<<<1, 1, 0, s>>>(D);
  if (ctx->n_cur > 0) {
    const int nb_save = ctx->nblocks;
    ctx->nblocks = blocks_for(ctx->n_cur);
    st = enqueue_sort_pass(ctx, D, s);
    ctx->nblocks = nb_save;
    if (st != GG_OK) return st;
    launch_narrow(ctx, D, ctx->n_cur, s);
  }
  ctx->launches += 9;
  ctx->last_batch = 1;
  ctx->last_nb = n_bodies;
  CK(cudaGetLastError());
  return GG_OK;
}

int gg_slab_sweep(gg_ctx* ctx, int32_t sweep) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (sweep < 0 || sweep >= ctx->D.S) return fail(ctx, GG_EINVAL, "sweep index out of range");
  DeviceGuard guard(ctx->device);
  if (ctx->n_own > 0)
    launch_sweep(slab_dev(ctx), sweep, ctx->n_own, ctx->stream);
  ctx->launches += 1;
  CK(cudaGetLastError());
  return GG_OK;
}

int gg_slab_halo_pack(gg_ctx* ctx, int32_t sweep, void* out_lo, void* out_hi) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  DeviceGuard guard(ctx->device);
  const Dev D = slab_dev(ctx);
  for (int side = 0; side < 2; ++side) {
    const long long m = ctx->ghost_out[side];
    void* out = side ? out_hi : out_lo;
    if (m <= 0) continue;
    if (!out) return fail(ctx, GG_EINVAL, "null halo buffer");
    k_slab_halo_pack<<<blocks_for(m), kBlock, 0, ctx->stream>>>(D, sweep, ctx->d_map[side],
                                                                 static_cast<int>(m), static_cast<float4*>(out));
    ctx->launches += 1;
  }
  CK(cudaGetLastError());
  return GG_OK;
}

int gg_slab_halo_unpack(gg_ctx* ctx, int32_t sweep, const void* in_lo, const void* in_hi) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  DeviceGuard guard(ctx->device);
  const Dev D = slab_dev(ctx);
  long long at = ctx->n_own;
  for (int side = 0; side < 2; ++side) {
    const long long m = ctx->ghost_in[side];
    const void* in = side ? in_hi : in_lo;
    if (m > 0) {
      if (!in) return fail(ctx, GG_EINVAL, "null halo buffer");
      k_slab_halo_unpack<<<blocks_for(m), kBlock, 0, ctx->stream>>>(
          D, sweep, static_cast<const float4*>(in), static_cast<int>(m), static_cast<int>(at));
      ctx->launches += 1;
    }
    at += m;
  }
  CK(cudaGetLastError());
  return GG_OK;
}

int gg_slab_finish(gg_ctx* ctx, gg_report* report, double* body_momentum) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  k_finish<false><<<finish_grid(std::max<long long>(ctx->n_own, 1)), kFinishBlock, 0, s>>>(slab_dev(ctx));
  k_commit<<<1, kBlock, 0, s>>>(slab_dev(ctx), finish_grid(std::max<long long>(ctx->n_own, 1)));
  ctx->launches += 2;
  CK(cudaGetLastError());
  int32_t nd = 0, es = -1;
  st = gg_sync(ctx, report, body_momentum, 1, &nd, &es);
  ctx->n_cur = ctx->n_own;  // ghosts are dropped after the commit
  ctx->ghost_in[0] = ctx->ghost_in[1] = 0;
  if (st == GG_OK && nd != 1) return fail(ctx, GG_ECUDA, "slab step did not commit");
  return st;
}

int64_t gg_slab_owned(const gg_ctx* ctx) { return ctx ? ctx->n_own : 0; }

int gg_slab_get(gg_ctx* ctx, double* x, double* v, int32_t* gid, int64_t cap, int64_t* n_own) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (!n_own) return fail(ctx, GG_EINVAL, "null n_own");
  *n_own = ctx->n_own;
  if (cap < ctx->n_own) return fail(ctx, GG_EINVAL, "output capacity below the owned count");
  if (ctx->n_own == 0) return GG_OK;
  DeviceGuard guard(ctx->device);
  st = ensure_stage(ctx);
  if (st != GG_OK) return st;
  cudaStream_t s = ctx->stream;
  k_slab_store<<<blocks_for(ctx->n_own), kBlock, 0, s>>>(slab_dev(ctx), ctx->d_stage,
                                                          ctx->d_stage + 3 * ctx->n, ctx->d_holes);
  ctx->launches += 1;
  const size_t b = sizeof(double) * 3 * static_cast<size_t>(ctx->n_own);
  if (x) CK(cudaMemcpyAsync(x, ctx->d_stage, b, cudaMemcpyDeviceToHost, s));
  if (v) CK(cudaMemcpyAsync(v, ctx->d_stage + 3 * ctx->n, b, cudaMemcpyDeviceToHost, s));
  if (gid) CK(cudaMemcpyAsync(gid, ctx->d_holes, sizeof(int) * ctx->n_own, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return GG_OK;
}

}  // extern "C"

// 0 every pixel tests every particle of its env, tiled through shared memory
// (default: measured 61 ms for 4096 envs x (36x36 + 72x36)); 1 splat every
// particle into the pixels it can cover (100+ ms there: the 64-bit atomicMin
// traffic on small images outweighs the saved tests).  Bitwise equal images.
static int g_render_mode = 1;  // internal: 0 splat, 1 brute force

extern "C" int gg_set_render_mode(int32_t mode) {
  if (mode != 0 && mode != 1) return GG_EINVAL;
  g_render_mode = mode ? 0 : 1;  // internal: 0 splat, 1 brute force
  return GG_OK;
}

extern "C" int gg_render_depth(gg_ctx* ctx, const gg_camera* cams, int32_t n_cams, int32_t per_env,
                               const gg_body* bodies, int32_t n_bodies, float* out) {
  if (!ctx || !cams || !out || n_cams < 1 || n_bodies < 0 || (n_bodies > 0 && !bodies))
    return fail(ctx, GG_EINVAL, "bad render arguments");
  const int E = ctx->E;
  const int ncam_tot = per_env ? E * n_cams : n_cams;
  std::vector<long long> off(n_cams + 1, 0);
  int max_pix = 0;
  for (int c = 0; c < n_cams; ++c) {
    const gg_camera& C = cams[c];
    if (C.width < 1 || C.height < 1 || !(C.far > 0) || (C.kind != 0 && C.kind != 1))
      return fail(ctx, GG_EINVAL, "bad camera (size >= 1x1, far > 0, kind 0/1)");
    off[c + 1] = off[c] + static_cast<long long>(C.width) * C.height;
    max_pix = std::max(max_pix, C.width * C.height);
  }
  if (per_env)
    for (int e = 1; e < E; ++e)
      for (int c = 0; c < n_cams; ++c)
        if (cams[e * n_cams + c].width != cams[c].width || cams[e * n_cams + c].height != cams[c].height ||
            cams[e * n_cams + c].kind != cams[c].kind || cams[e * n_cams + c].fov != cams[c].fov ||
            cams[e * n_cams + c].extent[0] != cams[c].extent[0] ||
            cams[e * n_cams + c].extent[1] != cams[c].extent[1])
          return fail(ctx, GG_EINVAL, "camera c must have the same intrinsics in every env");
  for (long long i = 0; i < static_cast<long long>(E) * n_bodies; ++i)
    if (bodies[i].kind == GG_GEOM_GRID && (bodies[i].grid_id < 0 || bodies[i].grid_id >= (int)ctx->grids.size()))
      return fail(ctx, GG_EINVAL, "unknown grid id");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t cam_b = sizeof(gg_camera) * ncam_tot;
  const size_t body_b = sizeof(gg_body) * static_cast<size_t>(E) * n_bodies;
  const size_t off_b = sizeof(long long) * (n_cams + 1);
  const size_t out_b = sizeof(float) * static_cast<size_t>(E) * off[n_cams];
  const size_t z_b = g_render_mode == 0 ? sizeof(unsigned long long) * static_cast<size_t>(E) * off[n_cams] : 0;
  const size_t loc_b = sizeof(double) * 3 * static_cast<size_t>(off[n_cams]);
  char* buf = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&buf), cam_b + body_b + off_b + out_b + z_b + loc_b + 64, s));
  gg_camera* dc = reinterpret_cast<gg_camera*>(buf);
  gg_body* db = reinterpret_cast<gg_body*>(buf + cam_b);
  long long* doff = reinterpret_cast<long long*>(buf + cam_b + body_b);
  float* dout = reinterpret_cast<float*>(buf + cam_b + body_b + off_b);
  cudaError_t e = cudaMemcpyAsync(dc, cams, cam_b, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && body_b) e = cudaMemcpyAsync(db, bodies, body_b, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(doff, off.data(), off_b, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    // 8-byte aligned z-buffer and local-ray table after the float output
    unsigned long long* zb = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(dout) + out_b + 7) & ~static_cast<uintptr_t>(7));
    double* dloc = reinterpret_cast<double*>(reinterpret_cast<char*>(zb) + z_b);
    RenderArgs A{dc, n_cams, per_env ? 1 : 0, db, n_bodies, doff, dout, dloc};
    dim3 grid((max_pix + kBlock - 1) / kBlock, n_cams, E);
    refresh_dev(ctx);
    // camera-frame rays of camera index c (the intrinsics agree across envs)
    k_render_local<<<dim3((max_pix + kBlock - 1) / kBlock, n_cams), kBlock, 0, s>>>(dc, n_cams, doff, dloc);
    if (g_render_mode == 0) {
      e = cudaMemsetAsync(zb, 0xff, z_b, s);
      if (e == cudaSuccess) {
        k_render_splat<<<dim3((ctx->ne + kBlock - 1) / kBlock, E), kBlock, 0, s>>>(ctx->D, A, zb);
        k_render_bodies<<<grid, kBlock, 0, s>>>(ctx->D, A, zb);
        ctx->launches += 2;
      }
    } else {
      k_render<<<grid, kBlock, 0, s>>>(ctx->D, A);
      ctx->launches += 1;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, out_b, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(buf, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gg_render_depth");
  return GG_OK;
}

// ---------------------------------------------------------------------------
// Peer-memory halo (gg_slab.cuh: Mailbox, k_halo_push, k_halo_pull)
// ---------------------------------------------------------------------------
extern "C" {

int gg_slab_mailbox(gg_ctx* ctx, int64_t cap, void* handle_out) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (cap < 1 || !handle_out) return fail(ctx, GG_EINVAL, "mailbox needs cap >= 1 and a handle buffer");
  DeviceGuard guard(ctx->device);
  if (ctx->mbox && ctx->mbox_cap < cap) {
    dfree(ctx, ctx->mbox);
    ctx->mbox = nullptr;
  }
  const size_t bytes = mailbox_bytes(cap);
  if (!ctx->mbox) {
    // plain cudaMalloc (IPC-exportable), zeroed flags
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    ctx->owned.push_back(p);
    ctx->mbox = static_cast<Mailbox*>(p);
    ctx->mbox_cap = cap;
    CK(cudaMemset(p, 0, bytes));
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->mbox));
  std::memcpy(handle_out, &h, sizeof(h));
  return GG_OK;
}

int gg_slab_connect(gg_ctx* ctx, int32_t side, const void* handle) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (side != 0 && side != 1) return fail(ctx, GG_EINVAL, "side must be 0 (lo) or 1 (hi)");
  DeviceGuard guard(ctx->device);
  if (ctx->peer_ipc[side] && ctx->peer[side]) cudaIpcCloseMemHandle(ctx->peer[side]);
  ctx->peer[side] = nullptr;
  ctx->peer_ipc[side] = false;
  if (!handle) return GG_OK;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ctx->peer[side] = static_cast<Mailbox*>(p);
  ctx->peer_ipc[side] = true;
  return GG_OK;
}

// Migration and ghost exchange through the neighbours' mailboxes, counts on
// the device, one host read-back (gg_slab.cuh, "Device-side exchange").
// Sequence numbers seq (migrants) and seq + 1 (ghosts): the caller advances
// seq by 2 per step, identically on every rank.  resort != 0 re-sorts the
// owned particles first (the physical order never changes a result).
// info[6]: migrants sent lo, hi, received lo, hi; ghosts received lo, hi.
int gg_slab_exchange_p2p(gg_ctx* ctx, uint64_t seq, int32_t resort, int64_t info[6]) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (!ctx->mbox) return fail(ctx, GG_EINVAL, "gg_slab_mailbox has not been called");
  if ((ctx->slab.has_lo && !ctx->peer[0]) || (ctx->slab.has_hi && !ctx->peer[1]))
    return fail(ctx, GG_EINVAL, "slab neighbour mailbox not connected");
  if (resort) {
    st = gg_slab_resort(ctx);
    if (st != GG_OK) return st;
  }
  DeviceGuard guard(ctx->device);
  if (!ctx->d_x) {
    CK(dalloc(ctx, &ctx->d_x, kXCount));
    CK(cudaMallocHost(&ctx->h_x, sizeof(unsigned long long) * kXCount));
  }
  const long long cap = ctx->mbox_cap;
  cudaStream_t s = ctx->stream;
  unsigned long long* X = ctx->d_x;
  ctx->n_cur = ctx->n_own;
  const long long n0 = ctx->n_own;
  const Dev D = slab_dev(ctx);
  Dev Dcap = D;
  Dcap.n = static_cast<int>(ctx->n);  // append bound: the particle capacity
  const int has_lo = ctx->slab.has_lo ? 1 : 0, has_hi = ctx->slab.has_hi ? 1 : 0;
  const unsigned long long tmo = 20000000000ull;  // 20 s
  CK(cudaMemsetAsync(X, 0, sizeof(unsigned long long) * kXCount, s));
  // migrants -> the neighbours' kind-0 boxes (I am my lo neighbour's hi side)
  SlabRec* m_lo = ctx->peer[0] ? mailbox_rec(ctx->peer[0], cap, 0, 1) : nullptr;
  SlabRec* m_hi = ctx->peer[1] ? mailbox_rec(ctx->peer[1], cap, 0, 0) : nullptr;
  if (n0 > 0) k_slab_emigrate<<<blocks_for(n0), kBlock, 0, s>>>(D, ctx->slab, m_lo, m_hi, cap, X);
  k_x_signal<<<1, 32, 0, s>>>(ctx->peer[0], ctx->peer[1], 0, seq, X);
  k_x_wait<<<1, 32, 0, s>>>(D, ctx->mbox, 0, seq, has_lo, has_hi, X, 5, tmo);
  if (n0 > 0) {
    k_x_holes<<<blocks_for(n0), kBlock, 0, s>>>(D, X, ctx->d_holes, ctx->d_movers, X);
    k_x_fill<<<blocks_for(n0), kBlock, 0, s>>>(D, ctx->d_holes, ctx->d_movers, X);
  }
  k_x_append<<<blocks_for(2 * cap), kBlock, 0, s>>>(Dcap, ctx->mbox, cap, 0, X, 4, 5);
  // ghosts: the boundary cells of the new owned set -> kind-1 boxes
  SlabRec* g_lo = ctx->peer[0] ? mailbox_rec(ctx->peer[0], cap, 1, 1) : nullptr;
  SlabRec* g_hi = ctx->peer[1] ? mailbox_rec(ctx->peer[1], cap, 1, 0) : nullptr;
  k_slab_ghosts<<<blocks_for(n0 + 2 * cap), kBlock, 0, s>>>(D, ctx->slab, g_lo, g_hi, ctx->d_map[0],
                                                          ctx->d_map[1], std::min<long long>(cap, ctx->n),
                                                          X + 8, X + 7);
  k_x_signal<<<1, 32, 0, s>>>(ctx->peer[0], ctx->peer[1], 1, seq + 1, X + 8);
  k_x_wait<<<1, 32, 0, s>>>(D, ctx->mbox, 1, seq + 1, has_lo, has_hi, X, 10, tmo);
  k_x_append<<<blocks_for(2 * cap), kBlock, 0, s>>>(Dcap, ctx->mbox, cap, 1, X, 7, 10);
  ctx->launches += 10;
  CK(cudaGetLastError());
  int err = 0;
  CK(cudaMemcpyAsync(ctx->h_x, X, sizeof(unsigned long long) * kXCount, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&err, &ctx->D.ctl->err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const unsigned long long* h = ctx->h_x;
  if (h[0] > static_cast<unsigned long long>(cap) || h[1] > static_cast<unsigned long long>(cap) ||
      h[8] > static_cast<unsigned long long>(cap) || h[9] > static_cast<unsigned long long>(cap))
    return fail(ctx, GG_ECAPACITY, "slab mailbox too small for this step's migrants or ghosts");
  if (err == GG_ECAPACITY) return fail(ctx, GG_ECAPACITY, "slab particle capacity exceeded");
  if (err) return fail(ctx, GG_ECUDA, "slab exchange: a neighbour did not answer (timeout)");
  ctx->n_own = static_cast<long long>(h[7]);
  ctx->ghost_out[0] = static_cast<long long>(h[8]);
  ctx->ghost_out[1] = static_cast<long long>(h[9]);
  ctx->ghost_in[0] = static_cast<long long>(h[10]);
  ctx->ghost_in[1] = static_cast<long long>(h[11]);
  ctx->n_cur = ctx->n_own + ctx->ghost_in[0] + ctx->ghost_in[1];
  if (info) {
    info[0] = static_cast<int64_t>(h[0]);
    info[1] = static_cast<int64_t>(h[1]);
    info[2] = static_cast<int64_t>(h[5]);
    info[3] = static_cast<int64_t>(h[6]);
    info[4] = static_cast<int64_t>(h[10]);
    info[5] = static_cast<int64_t>(h[11]);
  }
  return GG_OK;
}

// ---------------------------------------------------------------------------
// The whole slab step on the peer-memory transport as ONE CUDA graph (one per
// re-sort flag), replayed every step: nothing in it depends on the host.  The
// particle counts live on the device (Dev::dn, grids sized for the
// capacity), the mailbox sequence numbers derive from a device step counter,
// capacity and timeout failures raise the error word.  The host stages the
// body rows, launches the graph and reads the report back: one
// synchronisation per step.
// ---------------------------------------------------------------------------
static unsigned long long slab_graph_key(const gg_ctx* ctx) {
  const Dev& D = ctx->D;
  unsigned long long k = 1469598103934665603ull;
  auto mix = [&](unsigned long long v) { k = (k ^ v) * 1099511628211ull; };
  mix(static_cast<unsigned long long>(D.nb));
  mix(reinterpret_cast<uintptr_t>(D.bodies));
  mix(reinterpret_cast<uintptr_t>(D.grids));
  mix(reinterpret_cast<uintptr_t>(D.gvals));
  mix(reinterpret_cast<uintptr_t>(D.cgeo));
  mix(reinterpret_cast<uintptr_t>(D.reports));
  mix(reinterpret_cast<uintptr_t>(D.bm_out));
  mix(static_cast<unsigned long long>(D.wcap));
  mix(static_cast<unsigned long long>(D.S));
  mix(static_cast<unsigned long long>(ctx->pipeline));
  mix(reinterpret_cast<uintptr_t>(ctx->mbox));
  mix(static_cast<unsigned long long>(ctx->mbox_cap));
  mix(reinterpret_cast<uintptr_t>(ctx->peer[0]));
  mix(reinterpret_cast<uintptr_t>(ctx->peer[1]));
  mix(ctx->pgen);
  for (int a = 0; a < 3; ++a) mix(static_cast<unsigned long long>(D.mlo[a] * 64 + D.msh[a]));
  return k;
}

static int enqueue_slab_step(gg_ctx* ctx, int resort, cudaStream_t s, bool begin) {
  const long long cap = ctx->mbox_cap;
  const long long ncap = ctx->n;  // particle capacity
  Dev D = ctx->D;
  D.n = D.n_own = static_cast<int>(ncap);
  D.dn = ctx->d_n;
  D.resort = 0;
  D.key_morton = 0;
  D.pipeline = ctx->pipeline;
  unsigned long long* X = ctx->d_x;
  const unsigned long long* dstep = ctx->d_step;
  const int has_lo = ctx->slab.has_lo ? 1 : 0, has_hi = ctx->slab.has_hi ? 1 : 0;
  const unsigned long long tmo = 20000000000ull;  // 20 s
  if (begin) k_batch_begin<<<1, 256, 0, s>>>(D);
  k_x_prep<<<1, 32, 0, s>>>(X, ctx->d_n);
  if (resort) {  // (results never depend on the physical order)
    Dev R = D;
    R.resort = 1;
    R.key_morton = 1;
    k_slab_set_n<<<1, 1, 0, s>>>(R);
    int st = enqueue_sort_pass(ctx, R, s);
    if (st != GG_OK) return st;
    k_slab_commit_sorted<<<blocks_for(ncap), kBlock, 0, s>>>(R);
  }
  const bool alone = !has_lo && !has_hi;  // one rank: nothing to exchange
  // migrants, then ghosts, through the neighbours' mailboxes
  if (!alone) {
  SlabRec* m_lo = ctx->peer[0] ? mailbox_rec(ctx->peer[0], cap, 0, 1) : nullptr;
  SlabRec* m_hi = ctx->peer[1] ? mailbox_rec(ctx->peer[1], cap, 0, 0) : nullptr;
  k_slab_emigrate<<<blocks_for(ncap), kBlock, 0, s>>>(D, ctx->slab, m_lo, m_hi, cap, X);
  k_x_signal<<<1, 32, 0, s>>>(ctx->peer[0], ctx->peer[1], 0, 1, X, dstep, ctx->D.ctl, cap);
  k_x_wait<<<1, 32, 0, s>>>(D, ctx->mbox, 0, 1, has_lo, has_hi, X, 5, tmo, dstep);
  k_x_holes<<<blocks_for(ncap), kBlock, 0, s>>>(D, X, ctx->d_holes, ctx->d_movers, X);
  k_x_fill<<<blocks_for(ncap), kBlock, 0, s>>>(D, ctx->d_holes, ctx->d_movers, X);
  k_x_append<<<blocks_for(2 * cap), kBlock, 0, s>>>(D, ctx->mbox, cap, 0, X, 4, 5);
  SlabRec* g_lo = ctx->peer[0] ? mailbox_rec(ctx->peer[0], cap, 1, 1) : nullptr;
  SlabRec* g_hi = ctx->peer[1] ? mailbox_rec(ctx->peer[1], cap, 1, 0) : nullptr;
  k_slab_ghosts<<<blocks_for(ncap), kBlock, 0, s>>>(D, ctx->slab, g_lo, g_hi, ctx->d_map[0], ctx->d_map[1],
                                                    std::min<long long>(cap, ncap), X + 8, X + 7);
  k_x_signal<<<1, 32, 0, s>>>(ctx->peer[0], ctx->peer[1], 1, 2, X + 8, dstep, ctx->D.ctl, cap);
  k_x_wait<<<1, 32, 0, s>>>(D, ctx->mbox, 1, 2, has_lo, has_hi, X, 10, tmo, dstep);
  k_x_append<<<blocks_for(2 * cap), kBlock, 0, s>>>(D, ctx->mbox, cap, 1, X, 7, 10);
  k_x_counts<<<1, 32, 0, s>>>(X, ctx->d_n);
  }
  // contacts, sweeps with the per-sweep halo, integration and commit
  k_slab_set_n<<<1, 1, 0, s>>>(D);
  int st = enqueue_sort_pass(ctx, D, s);
  if (st != GG_OK) return st;
  launch_narrow(ctx, D, ncap, s);
  const int S = D.S;
  for (int sweep = 0; sweep < S; ++sweep) {
    launch_sweep(D, sweep, ncap, s);
    if (sweep < S - 1 && !alone) {
      const unsigned long long seq = static_cast<unsigned long long>(sweep) + 1;
      k_halo_push<<<2, 1024, 0, s>>>(D, sweep, seq, ctx->peer[0], ctx->peer[1], cap, ctx->d_map[0],
                                     ctx->d_map[1], 0, 0, X, dstep, static_cast<unsigned long long>(S - 1));
      k_halo_pull<<<2, 1024, 0, s>>>(D, sweep, seq, ctx->mbox, cap, 0, 0, has_lo, has_hi, tmo, X, dstep,
                                     static_cast<unsigned long long>(S - 1));
    }
  }
  k_finish<true><<<finish_grid(ncap), kFinishBlock, 0, s>>>(D);
  k_commit<<<1, kBlock, 0, s>>>(D, finish_grid(ncap));
  k_x_done<<<1, 32, 0, s>>>(ctx->d_step, X);
  CK(cudaGetLastError());
  return GG_OK;
}

static int build_slab_graphs(gg_ctx* ctx) {
  for (int g = 0; g < 4; ++g) {
    if (ctx->sgexec[g]) {
      cudaGraphExecDestroy(ctx->sgexec[g]);
      ctx->sgexec[g] = nullptr;
    }
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    int st = enqueue_slab_step(ctx, g & 1, ctx->stream, g < 2);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (st != GG_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture (slab step)");
    e = cudaGraphInstantiate(&ctx->sgexec[g], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate (slab step)");
  }
  ctx->sgkey = slab_graph_key(ctx);
  return GG_OK;
}

// One slab step on the peer-memory transport (replaces exchange_p2p +
// detect + solve_p2p + finish): bodies for this step, re-sort flag; the
// rank's StepReport (its owned particles) and body momentum; info[6] as
// gg_slab_exchange_p2p's.
// checks, device counters, the staged body rows of n_steps steps and the
// slab graphs (built on first use and whenever what they captured changed)
static int slab_p2p_prepare(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, int32_t n_steps) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (!ctx->mbox) return fail(ctx, GG_EINVAL, "gg_slab_mailbox has not been called");
  if ((ctx->slab.has_lo && !ctx->peer[0]) || (ctx->slab.has_hi && !ctx->peer[1]))
    return fail(ctx, GG_EINVAL, "slab neighbour mailbox not connected");
  if (n_steps < 1) return fail(ctx, GG_EINVAL, "n_steps must be >= 1");
  if (n_bodies < 0 || (n_bodies > 0 && !bodies)) return fail(ctx, GG_EINVAL, "bad bodies");
  for (long long b = 0; b < static_cast<long long>(n_bodies) * n_steps; ++b)
    if (bodies[b].kind < GG_GEOM_SPHERE || bodies[b].kind > GG_GEOM_GRID ||
        (bodies[b].kind == GG_GEOM_GRID && (bodies[b].grid_id < 0 || bodies[b].grid_id >= (int)ctx->grids.size())))
      return fail(ctx, GG_EINVAL, "bad body");
  if (!ctx->d_x) {
    CK(dalloc(ctx, &ctx->d_x, kXCount));
    CK(cudaMallocHost(&ctx->h_x, sizeof(unsigned long long) * kXCount));
  }
  if (!ctx->d_n) {  // first graph step: the device takes over the counts
    CK(dalloc(ctx, &ctx->d_n, 2));
    CK(dalloc(ctx, &ctx->d_step, 2));  // {steps replayed, particles emigrated}
    const int nn[2] = {static_cast<int>(ctx->n_own), static_cast<int>(ctx->n_own)};
    CK(cudaMemcpy(ctx->d_n, nn, sizeof(nn), cudaMemcpyHostToDevice));
    CK(cudaMemset(ctx->d_step, 0, 2 * sizeof(unsigned long long)));
  }
  st = stage_bodies(ctx, n_steps, bodies, n_bodies);
  if (st != GG_OK) return st;
  if (!ctx->sgexec[0] || ctx->sgkey != slab_graph_key(ctx)) {
    st = build_slab_graphs(ctx);
    if (st != GG_OK) return st;
  }
  return GG_OK;
}

int gg_slab_step_p2p(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, int32_t resort,
                     gg_report* report, double* body_momentum, int64_t info[6]) {
  if (!ctx) return GG_EINVAL;
  DeviceGuard guard(ctx->device);
  int st = slab_p2p_prepare(ctx, bodies, n_bodies, 1);
  if (st != GG_OK) return st;
  CK(cudaGraphLaunch(ctx->sgexec[resort ? 1 : 0], ctx->stream));
  ctx->launches += 40 + 3 * ctx->D.S;
  ctx->last_batch = 1;
  ctx->last_nb = n_bodies;
  int dn[2] = {0, 0};
  CK(cudaMemcpyAsync(ctx->h_x, ctx->d_x, sizeof(unsigned long long) * kXCount, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(dn, ctx->d_n, sizeof(dn), cudaMemcpyDeviceToHost, ctx->stream));
  int32_t nd = 0, es = -1;
  st = gg_sync(ctx, report, body_momentum, 1, &nd, &es);  // synchronises the stream
  const unsigned long long* h = ctx->h_x;
  ctx->n_own = ctx->n_cur = dn[1];
  ctx->ghost_out[0] = static_cast<long long>(h[8]);
  ctx->ghost_out[1] = static_cast<long long>(h[9]);
  ctx->ghost_in[0] = ctx->ghost_in[1] = 0;  // dropped after the commit
  if (info) {
    info[0] = static_cast<int64_t>(h[0]);
    info[1] = static_cast<int64_t>(h[1]);
    info[2] = static_cast<int64_t>(h[5]);
    info[3] = static_cast<int64_t>(h[6]);
    info[4] = static_cast<int64_t>(h[10]);
    info[5] = static_cast<int64_t>(h[11]);
  }
  if (st == GG_ECAPACITY && ctx->h_ctl->cap_needed == 0)
    return fail(ctx, GG_ECAPACITY, "slab mailbox or particle capacity exceeded by migrants or ghosts");
  if (st == GG_OK && nd != 1) return fail(ctx, GG_ECUDA, "slab step did not commit");
  return st;
}

// n_steps slab steps on the peer-memory transport, replayed back to back
// (one batch reset, then the batched step graph per step; the host only
// stages the bodies of every step up front and reads the reports once):
// bodies[n_steps][n_bodies], resort[n_steps]; reports[n_steps] and
// body_momentum[n_steps][n_bodies][3] of this rank's particles; info[7]: the
// last step's info (as gg_slab_step_p2p's) and, in info[6], the particles
// this rank sent to its neighbours over the whole batch.
int gg_slab_run_p2p(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, int32_t n_steps,
                    const int32_t* resort, gg_report* reports, double* body_momentum, int64_t info[7]) {
  if (!ctx) return GG_EINVAL;
  if (!resort || !reports) return fail(ctx, GG_EINVAL, "null resort flags or reports");
  DeviceGuard guard(ctx->device);
  int st = slab_p2p_prepare(ctx, bodies, n_bodies, n_steps);  // (synchronises the stream)
  if (st != GG_OK) return st;
  unsigned long long ds0[2] = {0ull, 0ull};
  CK(cudaMemcpy(ds0, ctx->d_step, sizeof(ds0), cudaMemcpyDeviceToHost));
  k_batch_begin<<<1, 256, 0, ctx->stream>>>(ctx->D);
  CK(cudaGetLastError());
  for (int i = 0; i < n_steps; ++i) CK(cudaGraphLaunch(ctx->sgexec[2 + (resort[i] ? 1 : 0)], ctx->stream));
  ctx->launches += 1 + static_cast<long long>(n_steps) * (39 + 3 * ctx->D.S);
  ctx->last_batch = n_steps;
  ctx->last_nb = n_bodies;
  int dn[2] = {0, 0};
  unsigned long long ds1[2] = {0ull, 0ull};
  CK(cudaMemcpyAsync(ctx->h_x, ctx->d_x, sizeof(unsigned long long) * kXCount, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(dn, ctx->d_n, sizeof(dn), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ds1, ctx->d_step, sizeof(ds1), cudaMemcpyDeviceToHost, ctx->stream));
  int32_t nd = 0, es = -1;
  st = gg_sync(ctx, reports, body_momentum, n_steps, &nd, &es);  // synchronises the stream
  const unsigned long long* h = ctx->h_x;
  ctx->n_own = ctx->n_cur = dn[1];
  ctx->ghost_out[0] = static_cast<long long>(h[8]);
  ctx->ghost_out[1] = static_cast<long long>(h[9]);
  ctx->ghost_in[0] = ctx->ghost_in[1] = 0;
  if (info) {
    info[0] = static_cast<int64_t>(h[0]);
    info[1] = static_cast<int64_t>(h[1]);
    info[2] = static_cast<int64_t>(h[5]);
    info[3] = static_cast<int64_t>(h[6]);
    info[4] = static_cast<int64_t>(h[10]);
    info[5] = static_cast<int64_t>(h[11]);
    info[6] = static_cast<int64_t>(ds1[1] - ds0[1]);
  }
  if (st == GG_ECAPACITY && ctx->h_ctl->cap_needed == 0)
    return fail(ctx, GG_ECAPACITY, "slab mailbox or particle capacity exceeded by migrants or ghosts");
  if (st == GG_OK && nd != n_steps) return fail(ctx, GG_ECUDA, "slab batch did not commit every step");
  return st;
}

// The S sweeps of a slab step with the per-sweep peer-memory halo between
// them (gg_slab_sweep / gg_slab_halo_p2p in one call: no host work between
// sweeps).  seq: the halo sequence number before the first sweep; the call
// uses seq + 1 .. seq + S - 1.
int gg_slab_solve_p2p(gg_ctx* ctx, uint64_t seq) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  for (int sweep = 0; sweep < ctx->D.S; ++sweep) {
    st = gg_slab_sweep(ctx, sweep);
    if (st == GG_OK && sweep < ctx->D.S - 1) st = gg_slab_halo_p2p(ctx, sweep, seq + 1 + sweep);
    if (st != GG_OK) return st;
  }
  return GG_OK;
}

int gg_slab_halo_p2p(gg_ctx* ctx, int32_t sweep, uint64_t seq) {
  int st = slab_check(ctx);
  if (st != GG_OK) return st;
  if (!ctx->mbox) return fail(ctx, GG_EINVAL, "gg_slab_mailbox has not been called");
  const long long cap = ctx->mbox_cap;
  for (int side = 0; side < 2; ++side)
    if (ctx->ghost_out[side] > cap || ctx->ghost_in[side] > cap)
      return fail(ctx, GG_ECAPACITY, "slab mailbox too small for this step's halo");
  if ((ctx->slab.has_lo && !ctx->peer[0]) || (ctx->slab.has_hi && !ctx->peer[1]))
    return fail(ctx, GG_EINVAL, "slab neighbour mailbox not connected");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = ctx->stream;
  const Dev D = slab_dev(ctx);
  k_halo_push<<<2, 1024, 0, s>>>(D, sweep, static_cast<unsigned long long>(seq), ctx->peer[0],
                                 ctx->peer[1], cap, ctx->d_map[0], ctx->d_map[1],
                                 static_cast<int>(ctx->ghost_out[0]), static_cast<int>(ctx->ghost_out[1]));
  k_halo_pull<<<2, 1024, 0, s>>>(D, sweep, static_cast<unsigned long long>(seq), ctx->mbox, cap,
                                 static_cast<int>(ctx->ghost_in[0]), static_cast<int>(ctx->ghost_in[1]),
                                 ctx->slab.has_lo ? 1 : 0, ctx->slab.has_hi ? 1 : 0,
                                 20000000000ull /* 20 s */);
  ctx->launches += 2;
  CK(cudaGetLastError());
  return GG_OK;
}

}  // extern "C"
