// gg_l1.cuh — the reference's test-facing L1 entry points on the device:
//
//   candidate_pairs        broadphase.py:185-196   k_cand_count / k_cand_fill
//   narrowphase_candidates contact.py:206-223      k_pairs_pp / k_pairs_body
//   solve_contacts_pja     contact.py:393-518      k_l1_frames / k_l1_sweep
//   project_friction_cone  contact.py:59-81        k_cone
//
// These run on caller-supplied float64 arrays (the reference's own data
// layout), not on the resident float32 state, and follow the reference's
// operation order: einsum dot products summed (x + z) + y, numpy's cross
// product and norm, np.add.at accumulation in contact order.  Only the
// body reaction momentum differs in rounding (64-bit fixed point, 2^-36, so
// the sum does not depend on thread order — as in the step kernels).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gg_kernels.cuh"
#include "gg_bake.cuh"

namespace gg {

// ---------------------------------------------------------------------------
// candidate_pairs (broadphase.py:149-196): per particle the 27 neighbour
// buckets sorted by hash with duplicates dropped (_candidate_csr:164-171),
// every particle in those buckets in bucket order, the particle itself
// excluded.  Buckets are visited in ascending hash order by repeated
// "smallest hash above the previous one" selection (27 x 27 hash
// evaluations, no local-memory array).
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void for_sorted_buckets(const Dev& D, long long c0, long long c1,
                                                   long long c2, F&& f) {
  uint32_t tx[3], ty[3], tz[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    tx[d] = hash_term32(c0 + d - 1, kP0);
    ty[d] = hash_term32(c1 + d - 1, kP1);
    tz[d] = hash_term32(c2 + d - 1, kP2);
  }
  long long prev = -1;
  for (int step = 0; step < 27; ++step) {
    long long best = 1ll << 40;
    for (int o = 0; o < 27; ++o) {
      const long long h = nb_hash(D, o, c0, c1, c2, tx, ty, tz);
      if (h > prev && h < best) best = h;
    }
    if (best == (1ll << 40)) break;
    f(static_cast<uint32_t>(best));
    prev = best;
  }
}

// position_cells (broadphase.py:33-41) of float64 positions
__global__ void k_cells_f64(const double* __restrict__ x, long long n, double two_r,
                            long long* __restrict__ cells, int* __restrict__ nonfinite) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double v = x[3 * i + a];
    if (!isfinite(v)) *nonfinite = 1;
    cells[3 * i + a] = cell_coord(v, two_r);
  }
}

// counts[uid] = candidates of particle uid (self excluded)
__global__ void k_cand_count(Dev D, long long* __restrict__ counts) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const float4 p = D.X[D.ctl->cur][k];
  const int uid = D.UID[D.ctl->ucur][k];
  long long total = 0;
  for_sorted_buckets(D, cell_coord(p.x, D.two_r), cell_coord(p.y, D.two_r),
                     cell_coord(p.z, D.two_r),
                     [&](uint32_t h) { total += D.start[h + 1] - D.start[h]; });
  counts[uid] = total - 1;
}

// (ci, cj) rows of particle uid from offs[uid] on, in candidate order
__global__ void k_cand_fill(Dev D, const long long* __restrict__ offs, long long* __restrict__ ci,
                            long long* __restrict__ cj) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= D.n) return;
  const float4 p = D.X[D.ctl->cur][k];
  const int* uid = D.UID[D.ctl->ucur];
  const int me = uid[k];
  long long at = offs[me];
  for_sorted_buckets(D, cell_coord(p.x, D.two_r), cell_coord(p.y, D.two_r),
                     cell_coord(p.z, D.two_r), [&](uint32_t h) {
                       for (uint32_t m = D.start[h]; m < D.start[h + 1]; ++m) {
                         const int q = __float_as_int(D.Xh[m].w);
                         if (q == k) continue;
                         ci[at] = me;
                         cj[at] = uid[q];
                         ++at;
                       }
                     });
}

// ---------------------------------------------------------------------------
// narrowphase_candidates (contact.py:206-223, _assemble_candidates :303-369)
// on explicit pairs of float64 positions.  pp: d = x_i - x_j,
// dist2 = (dx^2 + dz^2) + dy^2 (einsum order), colliding iff
// dist2 < (2r)^2 and not coincident; e1 = d / sqrt(dist2), psi = 2r - dist
// for colliding pairs, zero otherwise.
// ---------------------------------------------------------------------------
__global__ void k_pairs_pp(const double* __restrict__ x, const long long* __restrict__ ci,
                           const long long* __restrict__ cj, long long m, double two_r,
                           double contact_d2, double coinc_d2, double* __restrict__ e1,
                           double* __restrict__ psi, unsigned char* __restrict__ colliding,
                           unsigned long long* __restrict__ n_coinc) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const long long i = ci[t], j = cj[t];
  const double dx = __dsub_rn(x[3 * i], x[3 * j]);
  const double dy = __dsub_rn(x[3 * i + 1], x[3 * j + 1]);
  const double dz = __dsub_rn(x[3 * i + 2], x[3 * j + 2]);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
  const bool coi = d2 < coinc_d2;
  const bool hit = d2 < contact_d2 && !coi;
  if (coi) atomicAdd(n_coinc, 1ull);
  colliding[t] = hit ? 1 : 0;
  if (hit) {
    const double dist = __dsqrt_rn(d2);
    e1[3 * t] = __ddiv_rn(dx, dist);
    e1[3 * t + 1] = __ddiv_rn(dy, dist);
    e1[3 * t + 2] = __ddiv_rn(dz, dist);
    psi[t] = __dsub_rn(two_r, dist);
  } else {
    e1[3 * t] = e1[3 * t + 1] = e1[3 * t + 2] = 0.0;
    psi[t] = 0.0;
  }
}

// Body candidates: for body b and particle i (grid y = body), `_near_body`'s
// inclusive world-AABB test (contact.py:187-203), then penetration_depth and
// RigidBody.velocity_at at the contact point for every near particle
// (contact.py:327-333).  Non-contacts get psi = 0 and a zero normal, so their
// contact point is the centre itself (as in the reference).
__global__ void k_pairs_body(const gg_body* __restrict__ bodies, const DevGrid* __restrict__ grids,
                             const double* __restrict__ gvals, const double* __restrict__ x,
                             long long n, double r, unsigned char* __restrict__ near,
                             unsigned char* __restrict__ hit, double* __restrict__ psi,
                             double* __restrict__ nrm, double* __restrict__ vj,
                             unsigned long long* __restrict__ n_deg) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = blockIdx.y;
  const gg_body& B = bodies[b];
  const long long o = static_cast<long long>(b) * n + i;
  const double px = x[3 * i], py = x[3 * i + 1], pz = x[3 * i + 2];
  const bool in = !B.bounded || (px >= B.aabb_lo[0] && px <= B.aabb_hi[0] && py >= B.aabb_lo[1] &&
                                 py <= B.aabb_hi[1] && pz >= B.aabb_lo[2] && pz <= B.aabb_hi[2]);
  near[o] = in ? 1 : 0;
  if (!in) return;
  double ps = 0.0;
  d3 nv{0.0, 0.0, 0.0};
  int deg = 0;
  const int h = penetrate(B, grids, gvals, px, py, pz, r, &ps, &nv, &deg);
  if (!h) {
    ps = 0.0;
    nv = d3{0.0, 0.0, 0.0};
  }
  const d3 v = body_surface_velocity(B, px, py, pz, nv, r, ps);
  hit[o] = h ? 1 : 0;
  psi[o] = ps;
  nrm[3 * o] = nv.x;
  nrm[3 * o + 1] = nv.y;
  nrm[3 * o + 2] = nv.z;
  vj[3 * o] = v.x;
  vj[3 * o + 1] = v.y;
  vj[3 * o + 2] = v.z;
  if (deg) atomicAdd(n_deg, 1ull);
}

// ---------------------------------------------------------------------------
// solve_contacts_pja (contact.py:393-518) on a caller-supplied contact list.
// ---------------------------------------------------------------------------
struct L1Solve {
  int n;
  long long m;
  const int* rowptr;  // [n + 1]: contacts of owner i are cidx[rowptr[i] .. rowptr[i + 1])
  const int* cidx;    // contact indices grouped by owner, in contact order
  const long long* kind;
  const long long* other;
  const unsigned char* mask;  // CandidateContacts.colliding, or nullptr (all live)
  const double* e1;
  const double* e2;
  const double* e3;
  const double* psi;
  const double* vj0;  // vj with velocities[other] for pp contacts (contact.py:440-443)
  const double* v;
  double gamma, mu, alpha, dt, mass, gdt0, gdt1, gdt2;
  int nb;
  unsigned long long* bm_fix;  // [nb][3], 2^-36 fixed point
  unsigned long long* diag;    // [0] max cone violation bits, [1] min normal impulse bits
};

// edot (gg_bake.cuh): einsum("ij,ij->i") on the reference host, (a0 b0 + a2 b2) + a1 b1

// np.cross for 3-vectors (numpy/core/numeric.py cross: multiply, then subtract)
__device__ __forceinline__ void ncross(double a0, double a1, double a2, double b0, double b1,
                                       double b2, double& c0, double& c1, double& c2) {
  c0 = __dsub_rn(__dmul_rn(a1, b2), __dmul_rn(a2, b1));
  c1 = __dsub_rn(__dmul_rn(a2, b0), __dmul_rn(a0, b2));
  c2 = __dsub_rn(__dmul_rn(a0, b1), __dmul_rn(a1, b0));
}

// contact_frames (contact.py:47-56): axis = argmin |e1| (first on ties),
// e2 = e1 x axis / |e1 x axis|, e3 = e1 x e2.  Masked candidates use
// e1 = (1, 0, 0) for the frame (contact.py:431-432).
__global__ void k_l1_frames(long long m, const double* __restrict__ e1,
                            const unsigned char* __restrict__ mask, double* __restrict__ e2,
                            double* __restrict__ e3) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= m) return;
  double a0 = e1[3 * t], a1 = e1[3 * t + 1], a2 = e1[3 * t + 2];
  if (mask && !mask[t]) {
    a0 = 1.0;
    a1 = 0.0;
    a2 = 0.0;
  }
  int axis = 0;
  double amin = fabs(a0);
  if (fabs(a1) < amin) {
    axis = 1;
    amin = fabs(a1);
  }
  if (fabs(a2) < amin) axis = 2;
  const double p0 = axis == 0 ? 1.0 : 0.0, p1 = axis == 1 ? 1.0 : 0.0, p2 = axis == 2 ? 1.0 : 0.0;
  double c0, c1, c2;
  ncross(a0, a1, a2, p0, p1, p2, c0, c1, c2);
  // np.linalg.norm(axis=1): sqrt((x^2 + y^2) + z^2)
  const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(c0, c0), __dmul_rn(c1, c1)), __dmul_rn(c2, c2)));
  c0 = __ddiv_rn(c0, nn);
  c1 = __ddiv_rn(c1, nn);
  c2 = __ddiv_rn(c2, nn);
  e2[3 * t] = c0;
  e2[3 * t + 1] = c1;
  e2[3 * t + 2] = c2;
  double d0, d1, d2;
  ncross(a0, a1, a2, c0, c1, c2, d0, d1, d2);
  e3[3 * t] = d0;
  e3[3 * t + 1] = d1;
  e3[3 * t + 2] = d2;
}

// np.maximum(x, 0.0): x when x >= 0 or x is NaN
__device__ __forceinline__ double npmax0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }

// One Jacobi sweep (contact.py:463-501): owner i reads dv of the previous
// sweep for itself and its particle partners, accumulates its impulses onto
// dv_i in contact order (np.add.at), writes dv_next_i.
__global__ void k_l1_sweep(L1Solve L, const double* __restrict__ dv, double* __restrict__ dv_next) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.n) return;
  const double vi0 = L.v[3 * i], vi1 = L.v[3 * i + 1], vi2 = L.v[3 * i + 2];
  const double di0 = dv[3 * i], di1 = dv[3 * i + 1], di2 = dv[3 * i + 2];
  double a0 = di0, a1 = di1, a2 = di2;
  double maxviol = 0.0, minb1 = __longlong_as_double(0x7ff0000000000000ll);
  for (int r = L.rowptr[i]; r < L.rowptr[i + 1]; ++r) {
    const int c = L.cidx[r];
    if (L.mask && !L.mask[c]) continue;  // masked to zero impulse (contact.py:481-484)
    const bool pp = L.kind[c] == 0;
    double vj0 = L.vj0[3 * c], vj1 = L.vj0[3 * c + 1], vj2 = L.vj0[3 * c + 2];
    if (pp) {
      const long long j = L.other[c];
      vj0 = __dadd_rn(vj0, dv[3 * j]);
      vj1 = __dadd_rn(vj1, dv[3 * j + 1]);
      vj2 = __dadd_rn(vj2, dv[3 * j + 2]);
    }
    // u = velocities[own] - gamma * vj + gdt + dv[own]
    const double u0 = __dadd_rn(__dadd_rn(__dsub_rn(vi0, __dmul_rn(L.gamma, vj0)), L.gdt0), di0);
    const double u1 = __dadd_rn(__dadd_rn(__dsub_rn(vi1, __dmul_rn(L.gamma, vj1)), L.gdt1), di1);
    const double u2 = __dadd_rn(__dadd_rn(__dsub_rn(vi2, __dmul_rn(L.gamma, vj2)), L.gdt2), di2);
    const double* E1 = L.e1 + 3 * c;
    const double* E2 = L.e2 + 3 * c;
    const double* E3 = L.e3 + 3 * c;
    const double bias = __ddiv_rn(__dmul_rn(L.alpha, L.psi[c]), L.dt);
    const double b1 = npmax0(__dadd_rn(-edot(u0, u1, u2, E1[0], E1[1], E1[2]), bias));
    double b2 = -edot(u0, u1, u2, E2[0], E2[1], E2[2]);
    double b3 = -edot(u0, u1, u2, E3[0], E3[1], E3[2]);
    const double tn = hypot(b2, b3);
    const double lim = __dmul_rn(L.mu, b1);
    if (tn > lim) {
      const double den = (tn >= 1e-300 || tn != tn) ? tn : 1e-300;
      const double sc = __ddiv_rn(lim, den);
      b2 = __dmul_rn(b2, sc);
      b3 = __dmul_rn(b3, sc);
    }
    const double eff = pp ? 0.5 : 1.0;
    const double i0 = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(E1[0], b1), __dmul_rn(E2[0], b2)), __dmul_rn(E3[0], b3)), eff);
    const double i1 = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(E1[1], b1), __dmul_rn(E2[1], b2)), __dmul_rn(E3[1], b3)), eff);
    const double i2 = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(E1[2], b1), __dmul_rn(E2[2], b2)), __dmul_rn(E3[2], b3)), eff);
    a0 = __dadd_rn(a0, i0);
    a1 = __dadd_rn(a1, i1);
    a2 = __dadd_rn(a2, i2);
    if (!pp && L.nb > 0) {  // reaction momentum on the body (contact.py:489-495)
      const long long b = L.other[c];
      if (b >= 0 && b < L.nb) {
        atomicAdd(L.bm_fix + 3 * b, to_fix(-L.mass * i0));
        atomicAdd(L.bm_fix + 3 * b + 1, to_fix(-L.mass * i1));
        atomicAdd(L.bm_fix + 3 * b + 2, to_fix(-L.mass * i2));
      }
    }
    const double viol = __dsub_rn(hypot(b2, b3), lim);
    if (viol > maxviol) maxviol = viol;
    if (b1 < minb1) minb1 = b1;
  }
  dv_next[3 * i] = a0;
  dv_next[3 * i + 1] = a1;
  dv_next[3 * i + 2] = a2;
  if (maxviol > 0.0) atomicMax(L.diag, dbits(maxviol));
  if (minb1 >= 0.0 && minb1 < __longlong_as_double(0x7ff0000000000000ll)) atomicMin(L.diag + 1, dbits(minb1));
}

// project_friction_cone (contact.py:59-81) on k impulses b (k, 3)
__global__ void k_cone(double* __restrict__ b, const double* __restrict__ psi, long long k,
                       int psi_scalar, double mu, double alpha, double dt) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const double ps = psi[psi_scalar ? 0 : t];
  // b[:, 0] = max(b[:, 0] + alpha * psi / dt, 0)
  const double b0 = npmax0(__dadd_rn(b[3 * t], __ddiv_rn(__dmul_rn(alpha, ps), dt)));
  double b1 = b[3 * t + 1], b2 = b[3 * t + 2];
  const double tn = hypot(b1, b2);
  const double lim = __dmul_rn(mu, b0);
  if (tn > lim) {
    const double den = (tn >= 1e-300 || tn != tn) ? tn : 1e-300;
    const double sc = __ddiv_rn(lim, den);
    b1 = __dmul_rn(b1, sc);
    b2 = __dmul_rn(b2, sc);
  }
  b[3 * t] = b0;
  b[3 * t + 1] = b1;
  b[3 * t + 2] = b2;
}

}  // namespace gg
