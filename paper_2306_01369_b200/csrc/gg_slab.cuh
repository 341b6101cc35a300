// gg_slab.cuh — slab domain decomposition of one bed over several GPUs
// (SURVEY.md §8e "single large bed", config 5).  The reference has no
// multi-GPU path; parity is "same answer as one GPU".
//
// The bed is cut along x at cell boundaries (cells are round(x / 2r),
// broadphase.py:33-41, so every contact partner lies within +-1 cell).  A
// rank owns the particles whose cell index cx is in [lo, hi) and, each step,
//   M  migrates owned particles whose cell left [lo, hi) to the neighbour
//      (|v dt| < 2r: at most one cell per step, so only neighbours),
//   G  receives the neighbours' boundary-cell particles (cx == lo - 1 and
//      cx == hi) as ghosts, appended after the owned ones,
//   H  exchanges the ghosts' predicted velocity w after every Jacobi sweep
//      (contact.py:470-472 reads w_j of the previous sweep).
// Ghosts carry their global id as user id, so the stable bucket order, the
// candidate order and therefore every owned particle's contact sequence are
// exactly those of the one-GPU run: the slab step is bitwise identical to it.
//
// Transfer records: SlabRec = (x.xyz, bits(global id)), (v.xyz, 0).
#pragma once

#include "gg_kernels.cuh"

namespace gg {

struct SlabRec {
  float4 x;  // .w = __int_as_float(global id)
  float4 v;
};

struct SlabCfg {
  long long lo, hi;  // owned cell range [lo, hi) along x
  int has_lo, has_hi;  // a neighbour exists below / above
};

// M1: pack emigrants (their slot becomes a hole: UID = -1).  cnt[0] lo,
// cnt[1] hi (atomic slots: the order of the records does not matter — the
// stable sort orders particles by global id).
__global__ void k_slab_emigrate(Dev D, SlabCfg C, SlabRec* __restrict__ send_lo,
                                SlabRec* __restrict__ send_hi, long long cap,
                                unsigned long long* __restrict__ cnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= live_own_rt(D)) return;
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  const float4 x = D.X[cur][k];
  const long long cx = cell_coord(x.x, D.two_r);
  int side = -1;
  if (C.has_lo && cx < C.lo) side = 0;
  if (C.has_hi && cx >= C.hi) side = 1;
  if (side < 0) return;
  const unsigned long long slot = atomicAdd(cnt + side, 1ull);
  if (static_cast<long long>(slot) < cap) {
    SlabRec r;
    r.x = make_float4(x.x, x.y, x.z, __int_as_float(D.UID[u][k]));
    r.v = D.V[cur][k];
    (side ? send_hi : send_lo)[slot] = r;
    __threadfence_system();  // the record may be a peer's mailbox (gg_slab_exchange_p2p)
  }
  D.UID[u][k] = -1;
}

// M2: holes below the new owned count are refilled from the survivors above
// it (O(migrants) work): list the holes below n_stay and the survivors at or
// above it; pair them by slot.  cnt[2] holes, cnt[3] movers.
__global__ void k_slab_holes(Dev D, int n_stay, int* __restrict__ holes, int* __restrict__ movers,
                             unsigned long long* __restrict__ cnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n_own) return;
  const int uid = D.UID[D.ctl->ucur][k];
  if (k < n_stay && uid < 0) holes[atomicAdd(cnt + 2, 1ull)] = k;
  if (k >= n_stay && uid >= 0) movers[atomicAdd(cnt + 3, 1ull)] = k;
}

__global__ void k_slab_fill(Dev D, const int* __restrict__ holes, const int* __restrict__ movers,
                            int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  const int h = holes[i], s = movers[i];
  D.X[cur][h] = D.X[cur][s];
  D.V[cur][h] = D.V[cur][s];
  D.UID[u][h] = D.UID[u][s];
}

// Append records at [at, at + m): immigrants (owned) or ghosts.
__global__ void k_slab_append(Dev D, const SlabRec* __restrict__ in, int m, int at) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  const SlabRec r = in[i];
  D.X[cur][at + i] = make_float4(r.x.x, r.x.y, r.x.z, 0.f);
  D.V[cur][at + i] = make_float4(r.v.x, r.v.y, r.v.z, 0.f);
  D.UID[u][at + i] = __float_as_int(r.x.w);
}

// G1: the owned particles in the boundary cells, packed for the neighbours;
// map_* keeps their physical index for the per-sweep halo (no re-sort
// happens inside a slab step, so the map stays valid for the whole step).
// n_dev: the owned count on the device (after a device-side migration), else D.n_own.
__global__ void k_slab_ghosts(Dev D, SlabCfg C, SlabRec* __restrict__ send_lo,
                              SlabRec* __restrict__ send_hi, int* __restrict__ map_lo,
                              int* __restrict__ map_hi, long long cap,
                              unsigned long long* __restrict__ cnt,
                              const unsigned long long* __restrict__ n_dev = nullptr) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (n_dev ? static_cast<int>(*n_dev) : D.n_own)) return;
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  const float4 x = D.X[cur][k];
  const long long cx = cell_coord(x.x, D.two_r);
  const bool to_lo = C.has_lo && cx == C.lo;
  const bool to_hi = C.has_hi && cx == C.hi - 1;
  if (!to_lo && !to_hi) return;
  SlabRec r;
  r.x = make_float4(x.x, x.y, x.z, __int_as_float(D.UID[u][k]));
  r.v = D.V[cur][k];
  if (to_lo) {
    const unsigned long long s = atomicAdd(cnt + 0, 1ull);
    if (static_cast<long long>(s) < cap) {
      send_lo[s] = r;
      map_lo[s] = k;
    }
  }
  if (to_hi) {
    const unsigned long long s = atomicAdd(cnt + 1, 1ull);
    if (static_cast<long long>(s) < cap) {
      send_hi[s] = r;
      map_hi[s] = k;
    }
  }
  if (n_dev) __threadfence_system();  // peer mailbox records before the signal
}

// H: w of sweep s for the mapped boundary particles -> out; in -> ghosts.
__global__ void k_slab_halo_pack(Dev D, int s, const int* __restrict__ map, int m,
                                 float4* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = D.W[s & 1][map[i]];
}

__global__ void k_slab_halo_unpack(Dev D, int s, const float4* __restrict__ in, int m, int at) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) D.W[s & 1][at + i] = in[i];
}

// start[E * n_h] = n for the current particle count (n varies per step)
__global__ void k_slab_set_n(Dev D) { D.start[D.nh_tot] = static_cast<uint32_t>(live_n_rt(D)); }

// copy a Morton-re-sorted owned set (Xs, V0, UID[u^1]) back to the committed buffers
__global__ void k_slab_commit_sorted(Dev D) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= live_n_rt(D)) return;
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  D.X[cur][k] = D.Xs[k];
  D.V[cur][k] = D.V0[k];
  D.UID[u][k] = D.UID[u ^ 1][k];
}

// owned state in physical order (f64 rows + global ids)
__global__ void k_slab_store(Dev D, double* __restrict__ x, double* __restrict__ v,
                             int* __restrict__ gid) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n_own) return;
  const int cur = D.ctl->cur;
  const float4 p = D.X[cur][k], q = D.V[cur][k];
  x[3 * k] = p.x; x[3 * k + 1] = p.y; x[3 * k + 2] = p.z;
  v[3 * k] = q.x; v[3 * k + 1] = q.y; v[3 * k + 2] = q.z;
  gid[k] = D.UID[D.ctl->ucur][k];
}

__global__ void k_slab_load(Dev D, const double* __restrict__ x, const double* __restrict__ v,
                            const int* __restrict__ gid) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n_own) return;
  const int cur = D.ctl->cur;
  D.X[cur][k] = make_float4(static_cast<float>(x[3 * k]), static_cast<float>(x[3 * k + 1]),
                            static_cast<float>(x[3 * k + 2]), 0.f);
  D.V[cur][k] = make_float4(static_cast<float>(v[3 * k]), static_cast<float>(v[3 * k + 1]),
                            static_cast<float>(v[3 * k + 2]), 0.f);
  D.UID[D.ctl->ucur][k] = gid[k];
}

}  // namespace gg

namespace gg {

// ---------------------------------------------------------------------------
// Peer-memory halo (NVLink P2P through CUDA IPC mappings).  Every rank owns a
// mailbox that its neighbours write into directly; after every sweep a rank
// pushes its boundary particles' w into the two neighbours' mailboxes and
// raises a per-side sequence flag with a system-scope release, then pulls its
// own mailbox once both flags reached this sweep's sequence number.  No host
// work between sweeps.  Data is double-buffered by sweep parity: a sender can
// only get one sweep ahead of its receiver (it waits for the receiver's own
// push of that sweep before sweeping again).
// ---------------------------------------------------------------------------
struct Mailbox {
  unsigned long long flag[2];       // [side]: last halo sequence delivered from the lo / hi neighbour
  unsigned long long xflag[2];      // [side]: last exchange sequence (migrants, then ghosts)
  unsigned long long xcount[2][2];  // [kind][side]: records delivered (kind 0 migrants, 1 ghosts)
  // float4 halo[2 parity][2 side][cap], then SlabRec rec[2 kind][2 side][cap]
};
static_assert(sizeof(Mailbox) == 64, "mailbox header");

__device__ __forceinline__ float4* mailbox_data(Mailbox* m, long long cap, int parity, int side) {
  return reinterpret_cast<float4*>(m + 1) + (static_cast<long long>(parity) * 2 + side) * cap;
}
__host__ __device__ __forceinline__ SlabRec* mailbox_rec(Mailbox* m, long long cap, int kind, int side) {
  return reinterpret_cast<SlabRec*>(reinterpret_cast<float4*>(m + 1) + 4 * cap) +
         (static_cast<long long>(kind) * 2 + side) * cap;
}
__host__ __device__ __forceinline__ size_t mailbox_bytes(long long cap) {
  return sizeof(Mailbox) + (sizeof(float4) + sizeof(SlabRec)) * 4 * static_cast<size_t>(cap);
}

// block 0 -> the lo neighbour (its side 1), block 1 -> the hi neighbour (its side 0)
// X != nullptr (graph-replayed step): the ghost counts are X[8], X[9] and the
// sequence number is dstep * seq_mult + seq (a device step counter)
__global__ void k_halo_push(Dev D, int s, unsigned long long seq, Mailbox* peer_lo, Mailbox* peer_hi,
                            long long cap, const int* __restrict__ map_lo, const int* __restrict__ map_hi,
                            int n_lo, int n_hi, const unsigned long long* __restrict__ X = nullptr,
                            const unsigned long long* __restrict__ dstep = nullptr,
                            unsigned long long seq_mult = 0) {
  const int side = blockIdx.x;  // 0: push to lo, 1: push to hi
  Mailbox* peer = side == 0 ? peer_lo : peer_hi;
  if (dstep) seq += *dstep * seq_mult;
  int m = side == 0 ? n_lo : n_hi;
  if (X) m = static_cast<int>(min(X[8 + side], static_cast<unsigned long long>(cap)));
  if (peer == nullptr) return;  // block-uniform
  const int* map = side == 0 ? map_lo : map_hi;
  float4* dst = mailbox_data(peer, cap, s & 1, side == 0 ? 1 : 0);
  const float4* W = D.W[s & 1];
  for (int i = threadIdx.x; i < m; i += blockDim.x) dst[i] = W[map[i]];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // cumulative: the block's peer stores before the flag
    unsigned long long* f = &peer->flag[side == 0 ? 1 : 0];
    asm volatile("st.release.sys.u64 [%0], %1;" ::"l"(f), "l"(seq) : "memory");
  }
}

// block 0 <- the lo neighbour (my side 0), block 1 <- the hi neighbour (my side 1).
// The flag of an existing neighbour is awaited even when it sends no ghosts
// this step: the neighbour raises it after every sweep regardless, and the
// wait is what keeps it from running more than one sweep ahead of us (and
// overwriting the parity buffer we have not pulled yet) when halos are
// asymmetric.
__global__ void k_halo_pull(Dev D, int s, unsigned long long seq, Mailbox* mine, long long cap,
                            int n_lo, int n_hi, int has_lo, int has_hi,
                            unsigned long long timeout_ns, const unsigned long long* __restrict__ X = nullptr,
                            const unsigned long long* __restrict__ dstep = nullptr,
                            unsigned long long seq_mult = 0) {
  const int side = blockIdx.x;
  if (dstep) seq += *dstep * seq_mult;
  if (X) {
    n_lo = static_cast<int>(min(X[10], static_cast<unsigned long long>(cap)));
    n_hi = static_cast<int>(min(X[11], static_cast<unsigned long long>(cap)));
  }
  const int m = side == 0 ? n_lo : n_hi;
  if (!(side == 0 ? has_lo : has_hi)) return;  // block-uniform: no neighbour on this side
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int ok = 1;
    for (;;) {
      asm volatile("ld.relaxed.sys.u64 %0, [%1];" : "=l"(v) : "l"(&mine->flag[side]) : "memory");
      if (v >= seq) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {  // a neighbour died: fail instead of hanging the GPU
        ok = 0;
        break;
      }
      __nanosleep(200);
    }
    asm volatile("ld.acquire.sys.u64 %0, [%1];" : "=l"(v) : "l"(&mine->flag[side]) : "memory");
    s_ok = ok;
    if (!ok) raise_err(D.ctl, GG_ECUDA);
  }
  __syncthreads();
  if (!s_ok || m == 0) return;
  const float4* src = mailbox_data(mine, cap, s & 1, side);
  const int at = live_own_rt(D) + (side == 0 ? 0 : n_lo);
  float4* W = D.W[s & 1];
  for (int i = threadIdx.x; i < m; i += blockDim.x) W[at + i] = src[i];
}


// ---------------------------------------------------------------------------
// Device-side exchange of migrants and ghosts (gg_slab_exchange_p2p): the
// pack kernels write straight into the neighbours' mailboxes (peer memory),
// then ONE thread per side publishes the count and a system-scope release
// flag; the receiver waits for both flags (bounded) and appends from its own
// mailbox.  Every count lives on the device (X below); the host reads them
// once, after both exchanges.  No host round trip, no NCCL call.
//   X[0], X[1]  migrants sent lo / hi         X[2] holes, X[3] movers
//   X[4]        owned after the departures    X[5], X[6] migrants received lo / hi
//   X[7]        owned after the arrivals      X[8], X[9] ghosts sent lo / hi
//   X[10], X[11] ghosts received lo / hi
// ---------------------------------------------------------------------------
constexpr int kXCount = 12;

// publish this rank's records of `kind` to the neighbours: count, then flag
__global__ void k_x_signal(Mailbox* peer_lo, Mailbox* peer_hi, int kind, unsigned long long seq,
                           const unsigned long long* __restrict__ sent,
                           const unsigned long long* __restrict__ dstep = nullptr, Ctl* ctl = nullptr,
                           long long cap = 0) {
  if (threadIdx.x != 0) return;
  if (dstep) seq += *dstep * 2;
  // records beyond the mailbox were not delivered: the step fails (the host
  // path checks the counts it reads back; a replayed graph reads none)
  if (ctl && (sent[0] > static_cast<unsigned long long>(cap) || sent[1] > static_cast<unsigned long long>(cap)))
    raise_err(ctl, GG_ECAPACITY);
  for (int side = 0; side < 2; ++side) {
    Mailbox* p = side == 0 ? peer_lo : peer_hi;
    if (!p) continue;
    const int their = side == 0 ? 1 : 0;  // I am their hi (resp. lo) neighbour
    volatile unsigned long long* c = &p->xcount[kind][their];
    *c = sent[side];
    __threadfence_system();
    asm volatile("st.release.sys.u64 [%0], %1;" ::"l"(&p->xflag[their]), "l"(seq) : "memory");
  }
}

// wait for the neighbours' flags, read the counts they sent (0 without a
// neighbour) into X[at], X[at + 1]; the departures' survivors count first
__global__ void k_x_wait(Dev D, Mailbox* mine, int kind, unsigned long long seq, int has_lo, int has_hi,
                         unsigned long long* __restrict__ X, int at, unsigned long long timeout_ns,
                         const unsigned long long* __restrict__ dstep = nullptr) {
  if (threadIdx.x != 0) return;
  if (dstep) seq += *dstep * 2;
  for (int side = 0; side < 2; ++side) {
    unsigned long long got = 0;
    if (side == 0 ? has_lo : has_hi) {
      unsigned long long t0, t, v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        asm volatile("ld.relaxed.sys.u64 %0, [%1];" : "=l"(v) : "l"(&mine->xflag[side]) : "memory");
        if (v >= seq) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {  // a neighbour died: fail instead of hanging the GPU
          raise_err(D.ctl, GG_ECUDA);
          break;
        }
        __nanosleep(200);
      }
      asm volatile("ld.acquire.sys.u64 %0, [%1];" : "=l"(v) : "l"(&mine->xflag[side]) : "memory");
      got = *((volatile unsigned long long*)&mine->xcount[kind][side]);
    }
    X[at + side] = got;
  }
  if (kind == 0) X[4] = static_cast<unsigned long long>(live_own_rt(D)) - X[0] - X[1];
}

// holes below the survivors' count and survivors above it (k_slab_holes with
// the device count)
__global__ void k_x_holes(Dev D, const unsigned long long* __restrict__ X, int* __restrict__ holes,
                          int* __restrict__ movers, unsigned long long* __restrict__ cnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= live_own_rt(D)) return;
  const int n_stay = static_cast<int>(X[4]);
  const int uid = D.UID[D.ctl->ucur][k];
  if (k < n_stay && uid < 0) holes[atomicAdd(cnt + 2, 1ull)] = k;
  if (k >= n_stay && uid >= 0) movers[atomicAdd(cnt + 3, 1ull)] = k;
}

__global__ void k_x_fill(Dev D, const int* __restrict__ holes, const int* __restrict__ movers,
                         const unsigned long long* __restrict__ X) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= static_cast<int>(X[2])) return;
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  const int h = holes[i], s = movers[i];
  D.X[cur][h] = D.X[cur][s];
  D.V[cur][h] = D.V[cur][s];
  D.UID[u][h] = D.UID[u][s];
}

// append the mailbox's records of `kind` (lo side first) at X[base];
// kind 0 also sets X[7] = owned after the arrivals.  Grid: 2 * cap threads.
__global__ void k_x_append(Dev D, Mailbox* mine, long long cap, int kind,
                           unsigned long long* __restrict__ X, int base, int in_at) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long m_lo = static_cast<long long>(X[in_at]), m_hi = static_cast<long long>(X[in_at + 1]);
  if (kind == 0 && t == 0) X[7] = X[4] + m_lo + m_hi;
  const int side = t < cap ? 0 : 1;
  const long long i = side == 0 ? t : t - cap;
  if (i >= (side == 0 ? m_lo : m_hi) || i >= cap) return;
  const long long at = static_cast<long long>(X[base]) + (side == 0 ? 0 : m_lo) + i;
  if (at >= D.n) {  // capacity (D.n = the context's particle capacity here)
    raise_err(D.ctl, GG_ECAPACITY);
    return;
  }
  const SlabRec r = mailbox_rec(mine, cap, kind, side)[i];
  const int cur = D.ctl->cur, u = D.ctl->ucur;
  D.X[cur][at] = make_float4(r.x.x, r.x.y, r.x.z, 0.f);
  D.V[cur][at] = make_float4(r.v.x, r.v.y, r.v.z, 0.f);
  D.UID[u][at] = __float_as_int(r.x.w);
}


// Graph-replayed slab step: the step's counts on the device.  k_x_prep:
// exchange counters cleared, ghosts of the previous step dropped
// (n = n_own); k_x_counts: the new counts after both exchanges; k_x_done: the
// device step counter the sequence numbers derive from.
__global__ void k_x_prep(unsigned long long* __restrict__ X, int* __restrict__ dn) {
  const int t = threadIdx.x;
  if (t < kXCount) X[t] = 0ull;
  if (t == 0) dn[0] = dn[1];
}
__global__ void k_x_counts(const unsigned long long* __restrict__ X, int* __restrict__ dn) {
  if (threadIdx.x != 0) return;
  dn[1] = static_cast<int>(X[7]);
  dn[0] = static_cast<int>(X[7] + X[10] + X[11]);
}
__global__ void k_x_done(unsigned long long* __restrict__ dstep, const unsigned long long* __restrict__ X) {
  if (threadIdx.x == 0) {
    dstep[0] += 1;
    dstep[1] += X[0] + X[1];  // emigrants of this step (a running total)
  }
}

}  // namespace gg
