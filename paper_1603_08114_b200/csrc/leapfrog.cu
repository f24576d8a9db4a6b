// leapfrog.cu -- the fused HMC trajectory and its Metropolis test on sm_100a.
//
// Replaces (paths relative to the reference's pkg/src/rsvhmc/):
//   integrator.py:149-179 integrate_trajectory and :139-146 elementary_step
//     (kernels 1-3, _kernels.py:37-54, force _kernels.py:23-34),
//   model.py:134-182 log_posterior / hamiltonian (H_old, H_new),
//   sampler.py:155-167 (dH, divergence sentinel, Metropolis),
//   the sums inside sampler.py:170-272 (theta sufficient statistics).
//
// traj_kernel: one CTA owns a tile of `core` consecutive sites plus a halo
// of n_steps + 1 sites on each side; each thread keeps 8 consecutive sites
// (d = h - mu, p, and the per-site force constants) in registers for the
// whole trajectory.  Neighbour values move by warp shuffles and, across
// warps, through shared memory with one barrier per step.  Because the
// stencil is nearest-neighbour, L steps on a tile with an L-site halo give
// the core sites exactly the values a global step-by-step sweep gives, so
// the whole trajectory is one launch with no grid-wide synchronisation.
// HBM traffic per trajectory is ~40 B/site, the FP64 pipe is the bound
// ("Roofline").
#include <math.h>

#include "exp_table.h"
#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

__device__ const double g_exp_tab[64] = RSV_EXP_TAB_INIT;

constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52

// exp(-d) for the model's range: n = rint(-64 d / ln2), r = -d - n ln2/64,
// e^r - 1 by a degree-5 polynomial (|r| <= ln2/128), 2^(n/64) by table +
// exponent add.  10 FP64 instructions; <= ~1.5 ulp.  `t` is returned so the
// caller can range-check n (divergence test) with integer ops only.
__device__ __forceinline__ double exp_neg(double d, const double *tab, double &t) {
  t = fma(-d, RSV_INV_LN2_64, MAGIC);
  const double nd = t - MAGIC;
  double r = fma(nd, -RSV_LN2_64_HI, -d);
  r = fma(nd, -RSV_LN2_64_LO, r);
  double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const int n = __double2loint(t);
  const double T = tab[n & 63];
  const double e = fma(T, q, T);
  return __hiloint2double(__double2hiint(e) + ((n >> 6) << 20), __double2loint(e));
}

// |h| <= 50 (and not NaN) <=> n within [n_lo, n_hi] and t a sane magic sum
__device__ __forceinline__ bool in_range(double t, int n_lo, int n_span) {
  const int n = __double2loint(t);
  const unsigned hw = (unsigned)__double2hiint(t) - 0x4337FFFFu;
  return ((unsigned)(n - n_lo) <= (unsigned)n_span) & (hw <= 1u);
}

struct TrajScalars {
  double mu, phi, c_half, c_full, dt, bphi, g_int, g_end, adt, half_dt, alpha, emu, xm;
  double inv2su, inv2se, one_m_phi2;
  int n_lo, n_span;
};

__device__ __forceinline__ TrajScalars traj_scalars(const DevParams &P, double dt) {
  TrajScalars s;
  s.mu = P.mu;
  s.phi = P.phi;
  s.dt = dt;
  s.c_half = 0.5 * dt;
  s.c_full = dt;
  const double inv_su2 = 1.0 / P.su2, inv_se2 = 1.0 / P.se2;
  s.alpha = dt * inv_su2;
  const double beta = dt * inv_se2;
  s.bphi = beta * P.phi;
  s.g_int = s.alpha + beta * (1.0 + P.phi * P.phi);
  s.g_end = s.alpha + beta;
  s.emu = exp(-P.mu);
  s.adt = dt * s.emu;
  s.half_dt = 0.5 * dt;
  s.xm = P.xi + P.mu;
  s.inv2su = 0.5 * inv_su2;
  s.inv2se = 0.5 * inv_se2;
  s.one_m_phi2 = 1.0 - P.phi * P.phi;
  // n = rint(-d * 64/ln2) with d = h - mu; |h| <= 50  <=>  n in [n_lo, n_hi]
  s.n_lo = (int)floor((P.mu - 50.0) * RSV_INV_LN2_64);
  s.n_span = (int)ceil((P.mu + 50.0) * RSV_INV_LN2_64) - s.n_lo;
  return s;
}

// Variable part of H at one site (the theta-only constants are added by the
// accept kernel): 0.5 p^2 + 0.5 d + a e^{-mu} e^{-d} + (q - d)^2 / 2su2 + AR.
__device__ __forceinline__ double site_energy(double d, double dprev, double p, double ae, double q, bool first,
                                              const TrajScalars &s, const double *tab) {
  double t;
  const double E = exp_neg(d, tab, t);
  const double r = q - d;
  const double tr = d - s.phi * dprev;
  const double ar = first ? s.one_m_phi2 * d * d * s.inv2se : tr * tr * s.inv2se;
  return 0.5 * p * p + 0.5 * d + ae * E + r * r * s.inv2su + ar;
}

// Exchange the first / last register site with the neighbouring threads.
__device__ __forceinline__ void exchange(double first, double last, double &left, double &right, double *s_first,
                                         double *s_last, int lane, int warp) {
  left = __shfl_up_sync(0xffffffffu, last, 1);
  right = __shfl_down_sync(0xffffffffu, first, 1);
  if (lane == 31) s_last[warp] = last;
  if (lane == 0) s_first[warp] = first;
  __syncthreads();
  if (lane == 0) left = warp > 0 ? s_last[warp - 1] : 0.0;
  if (lane == 31) right = warp < TR_NW - 1 ? s_first[warp + 1] : 0.0;
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*s_red)[NV], int lane, int warp) {
#pragma unroll
  for (int k = 0; k < NV; k++) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; k++) s_red[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; k++) {
      double acc = s_red[0][k];
      for (int w = 1; w < TR_NW; w++) acc += s_red[w][k];
      v[k] = acc;
    }
  }
}

// One kick p -= dt * dU/dh for the thread's R sites (d-space), see DESIGN.md:
//   p <- p - Cd - G d + beta phi (d_{i-1} + d_{i+1}) + Ad e^{-d}
template <bool EDGE>
__device__ __forceinline__ void kick(double (&d)[TR_R], double (&p)[TR_R], const double (&Ad)[TR_R],
                                     const double (&Cd)[TR_R], double dl, double dr, const TrajScalars &s,
                                     const double *tab, uint32_t live, uint32_t endm, uint32_t core, int &bad) {
#pragma unroll
  for (int r = 0; r < TR_R; r++) {
    const double dm = r ? d[r - 1] : dl;
    const double dp = r < TR_R - 1 ? d[r + 1] : dr;
    double t;
    const double E = exp_neg(d[r], tab, t);
    if (!in_range(t, s.n_lo, s.n_span) && ((core >> r) & 1)) bad = 1;
    const double G = EDGE && ((endm >> r) & 1) ? s.g_end : s.g_int;
    double pp = p[r] - Cd[r];
    pp = fma(-G, d[r], pp);
    pp = fma(s.bphi, dm + dp, pp);
    pp = fma(Ad[r], E, pp);
    p[r] = (EDGE && !((live >> r) & 1)) ? 0.0 : pp;
  }
}

__device__ __forceinline__ void drift(double (&d)[TR_R], const double (&p)[TR_R], double c) {
#pragma unroll
  for (int r = 0; r < TR_R; r++) d[r] = fma(c, p[r], d[r]);
}

template <bool FUSE>
__global__ void __launch_bounds__(TR_NT, 2) traj_kernel(TrajArgs A) {
  __shared__ double s_tab[64];
  __shared__ double s_first[2][TR_NW], s_last[2][TR_NW];
  __shared__ double s_red[TR_NW][TR_NV];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 64) s_tab[tid] = g_exp_tab[tid];

  const DevParams P = *A.prm;
  const TrajScalars s = traj_scalars(P, A.dt);
  const double *hsrc;
  double *hdst;
  if (A.h_src) {
    hsrc = A.h_src;
    hdst = A.h_dst;
  } else {
    const int cur = A.ctrl->cur;
    hsrc = cur ? A.hbuf1 : A.hbuf0;
    hdst = cur ? A.hbuf0 : A.hbuf1;
  }
  const int64_t T = A.T;
  const int H = A.g.halo;
  const int64_t t0 = (int64_t)blockIdx.x * A.g.core;
  const int64_t t1 = min(t0 + A.g.core, T);
  const int64_t lo_live = max((int64_t)0, t0 - H), hi_live = min(T, t1 + H);
  const int64_t g0 = t0 - H + (int64_t)tid * TR_R;

  uint32_t live = 0, core = 0, endm = 0;
  double d[TR_R], p[TR_R], Ad[TR_R], Cd[TR_R];
  double hold = 0.0, so[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int r = 0; r < TR_R; r++) {
    const int64_t gi = g0 + r;
    d[r] = 0.0; p[r] = 0.0; Ad[r] = 0.0; Cd[r] = 0.0;
    if (gi >= lo_live && gi < hi_live) {
      live |= 1u << r;
      if (gi >= t0 && gi < t1) core |= 1u << r;
      if (gi == 0 || gi == T - 1) endm |= 1u << r;
      d[r] = hsrc[gi] - s.mu;
      p[r] = A.p_in[gi];
      const double ae = s.emu * A.a[gi];
      const double q = A.lrv[gi] - s.xm;
      Ad[r] = s.dt * ae;
      Cd[r] = fma(-s.alpha, q, s.half_dt);
    }
  }
  const bool edge = (live != (1u << TR_R) - 1) || endm;
  const bool warp_live = __any_sync(0xffffffffu, live != 0);
  __syncthreads();  // s_tab

  // ---- H_old and statistics of the current path (core sites) ----
  {
    double dl, dr;
    exchange(d[0], d[TR_R - 1], dl, dr, s_first[0], s_last[0], lane, warp);
    double v[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < TR_R; r++) {
      if ((core >> r) & 1) {
        const int64_t gi = g0 + r;
        const double dprev = r ? d[r - 1] : dl;
        const double ae = s.emu * A.a[gi];
        const double q = A.lrv[gi] - s.xm;
        const double e = q - d[r];
        hold += site_energy(d[r], dprev, p[r], ae, q, gi == 0, s, s_tab);
        so[0] += d[r];
        so[1] += d[r] * d[r];
        if (gi > 0) so[2] += d[r] * dprev;
        so[3] += e;
        so[4] += e * e;
        if (!A.h_src) {
          if (gi == 0) A.ctrl->ends_old[0] = d[r];
          if (gi == T - 1) A.ctrl->ends_old[1] = d[r];
        }
      }
    }
    v[0] = hold; v[1] = so[0]; v[2] = so[1]; v[3] = so[2]; v[4] = so[3]; v[5] = so[4];
    block_sum<6>(v, reinterpret_cast<double(*)[6]>(&s_red[0][0]), lane, warp);
    if (tid == 0) {
      TilePart *tp = A.parts + blockIdx.x;
      tp->hold = v[0];
      for (int k = 0; k < 5; k++) tp->so[k] = v[k + 1];
    }
  }

  // ---- the trajectory ----
  int bad = 0;
  const int L = A.n_steps;
  if (FUSE) {
    if (warp_live) drift(d, p, s.c_half);
  }
  for (int step = 0; step < L; step++) {
    const int b = (step + 1) & 1;
    if (!FUSE && warp_live) drift(d, p, s.c_half);
    double dl, dr;
    exchange(d[0], d[TR_R - 1], dl, dr, s_first[b], s_last[b], lane, warp);
    if (warp_live) {
      if (edge) kick<true>(d, p, Ad, Cd, dl, dr, s, s_tab, live, endm, core, bad);
      else kick<false>(d, p, Ad, Cd, dl, dr, s, s_tab, live, endm, core, bad);
      if (FUSE) drift(d, p, step < L - 1 ? s.c_full : s.c_half);
      else drift(d, p, s.c_half);
    }
  }

  // ---- H_new, statistics of the proposal, write-back ----
  {
    double dl, dr;
    exchange(d[0], d[TR_R - 1], dl, dr, s_first[(L + 1) & 1], s_last[(L + 1) & 1], lane, warp);
    double hnew = 0.0, sn[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < TR_R; r++) {
      if ((core >> r) & 1) {
        const int64_t gi = g0 + r;
        const double dprev = r ? d[r - 1] : dl;
        const double ae = s.emu * A.a[gi];
        const double q = A.lrv[gi] - s.xm;
        const double e = q - d[r];
        hnew += site_energy(d[r], dprev, p[r], ae, q, gi == 0, s, s_tab);
        sn[0] += d[r];
        sn[1] += d[r] * d[r];
        if (gi > 0) sn[2] += d[r] * dprev;
        sn[3] += e;
        sn[4] += e * e;
        hdst[gi] = d[r] + s.mu;
        if (A.p_out) A.p_out[gi] = p[r];
        if (!A.h_src) {
          if (gi == 0) A.ctrl->ends_new[0] = d[r];
          if (gi == T - 1) A.ctrl->ends_new[1] = d[r];
        }
      }
    }
    double v[8] = {hnew - hold, hnew, sn[0], sn[1], sn[2], sn[3], sn[4], (double)bad};
    __syncthreads();  // s_red reuse
    block_sum<8>(v, reinterpret_cast<double(*)[8]>(&s_red[0][0]), lane, warp);
    if (tid == 0) {
      TilePart *tp = A.parts + blockIdx.x;
      tp->dh = v[0];
      tp->hnew = v[1];
      for (int k = 0; k < 5; k++) tp->sn[k] = v[k + 2];
      tp->flag = v[7];
    }
  }
}

TrajGeom traj_geometry(int64_t T, int n_steps, int sm_count) {
  TrajGeom g;
  g.halo = n_steps + 1;
  const int64_t core_max = TR_W - 2 * (int64_t)g.halo;
  g.ok = core_max >= TR_W / 4;
  if (!g.ok) { g.core = 0; g.n_tiles = 0; return g; }
  int64_t n = (T + core_max - 1) / core_max;
  const int64_t slots = 2LL * sm_count;
  if (n > slots / 2) n = (n + slots - 1) / slots * slots;
  g.core = (T + n - 1) / n;
  g.n_tiles = (int)((T + g.core - 1) / g.core);
  return g;
}

int launch_trajectory(const TrajArgs &a, cudaStream_t s, int *launches) {
  if (a.fuse) traj_kernel<true><<<a.g.n_tiles, TR_NT, 0, s>>>(a);
  else traj_kernel<false><<<a.g.n_tiles, TR_NT, 0, s>>>(a);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------
// Metropolis (sampler.py:155-167) on the reduced tile partials.
constexpr int AC_NT = 256;
__global__ void __launch_bounds__(AC_NT) accept_kernel(AcceptArgs A) {
  __shared__ double s_v[AC_NT][TR_NV];
  double v[TR_NV];
#pragma unroll
  for (int k = 0; k < TR_NV; k++) v[k] = 0.0;
  for (int i = threadIdx.x; i < A.n_tiles; i += AC_NT) {
    const TilePart &tp = A.parts[i];
    v[0] += tp.dh; v[1] += tp.hold; v[2] += tp.hnew;
#pragma unroll
    for (int k = 0; k < 5; k++) { v[3 + k] += tp.so[k]; v[8 + k] += tp.sn[k]; }
    v[13] += tp.flag;
  }
#pragma unroll
  for (int k = 0; k < TR_NV; k++) s_v[threadIdx.x][k] = v[k];
  __syncthreads();
  for (int w = AC_NT / 2; w >= 1; w >>= 1) {
    if (threadIdx.x < w) {
#pragma unroll
      for (int k = 0; k < TR_NV; k++) s_v[threadIdx.x][k] += s_v[threadIdx.x + w][k];
    }
    __syncthreads();
  }
  if (threadIdx.x) return;
  const DevParams P = *A.prm;
  DevControl *C = A.ctrl;
  const double Td = (double)A.T;
  const double cst = 0.5 * Td * P.mu + 0.5 * Td * log(P.su2) + 0.5 * log(P.se2 / (1.0 - P.phi * P.phi)) +
                     0.5 * (Td - 1.0) * log(P.se2);
  const double *tot = s_v[0];
  DevResult r;
  r.h_old = tot[1] + cst;
  r.h_new = tot[2] + cst;
  r.accept = 0;
  r.u = __longlong_as_double(0x7ff8000000000000LL);
  r.words_used = 0;
  const bool flagged = tot[13] > 0.0;
  if (A.integrate_only) {
    r.diverged = flagged;
    r.delta_h = tot[0];
    C->res = r;
    if (A.res_out) *A.res_out = r;
    return;
  }
  uint64_t used = C->zig_used;
  bool drew = false;
  if (flagged) {
    r.diverged = 1;
    r.delta_h = __longlong_as_double(0x7ff0000000000000LL);
  } else {
    const double dh = tot[0];
    if (!isfinite(dh) || fabs(dh) > 1000.0) {
      r.diverged = 1;
      r.delta_h = __longlong_as_double(0x7ff0000000000000LL);
    } else {
      r.diverged = 0;
      r.delta_h = dh;
      const uint64_t w = C->stream.kind == PRNG_SFC64 ? A.sfc_words[used] : word_at(C->stream, C->stream.pos + used);
      r.u = u01(w);
      drew = true;
      r.accept = (dh <= 0.0) || (r.u < exp(-dh));
    }
  }
  const uint64_t consumed = used + (drew ? 1 : 0);
  r.words_used = consumed;
  if (C->stream.kind == PRNG_SFC64) {
    const uint64_t *q = A.sfc_snaps + 4 * (consumed / SFC_SNAP);
    uint64_t st[4] = {q[0], q[1], q[2], q[3]};
    for (uint64_t i = 0; i < consumed % SFC_SNAP; i++) sfc64_next(st);
    for (int i = 0; i < 4; i++) C->stream.s[i] = st[i];
  }
  C->stream.pos += consumed;
  if (r.accept) C->cur ^= 1;
  // statistics of the kept path, shifted by (mu, xi) of the params used
  const double *sm = r.accept ? tot + 8 : tot + 3;
  C->stats[0] = r.accept ? C->ends_new[0] : C->ends_old[0];
  C->stats[1] = r.accept ? C->ends_new[1] : C->ends_old[1];
  for (int k = 0; k < 5; k++) C->stats[2 + k] = sm[k];
  C->res = r;
  if (A.res_out) *A.res_out = r;
}

int launch_accept(const AcceptArgs &a, cudaStream_t s, int *launches) {
  accept_kernel<<<1, AC_NT, 0, s>>>(a);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------
// Reference-order scalars (model.py:185-199 scalar_pack).
struct RefScal {
  double half, phi, mu, xi, inv_su2, inv_se2, one_m_phi2;
};
__device__ __forceinline__ RefScal ref_scal(const DevParams &P) {
  RefScal s;
  s.half = 0.5;
  s.phi = P.phi;
  s.mu = P.mu;
  s.xi = P.xi;
  s.inv_su2 = __ddiv_rn(1.0, P.su2);
  s.inv_se2 = __ddiv_rn(1.0, P.se2);
  s.one_m_phi2 = __dsub_rn(1.0, __dmul_rn(P.phi, P.phi));
  return s;
}

// _kernels.py:23-34 _grad_site in the reference's evaluation order with no
// contraction; yy = (half * y) * y precomputed or computed by the caller.
__device__ __forceinline__ double grad_site_ref(double v, double vm, double vp, bool has_m, bool has_p, double yy,
                                                double lrv, const RefScal &s) {
  double g = __dadd_rn(__dsub_rn(s.half, __dmul_rn(yy, exp(-v))),
                       __dmul_rn(__dsub_rn(__dadd_rn(s.xi, v), lrv), s.inv_su2));
  if (!has_m) g = __dadd_rn(g, __dmul_rn(__dmul_rn(s.one_m_phi2, __dsub_rn(v, s.mu)), s.inv_se2));
  else g = __dadd_rn(g, __dmul_rn(__dsub_rn(__dsub_rn(v, s.mu), __dmul_rn(s.phi, __dsub_rn(vm, s.mu))), s.inv_se2));
  if (has_p)
    g = __dsub_rn(g, __dmul_rn(__dmul_rn(s.phi, __dsub_rn(__dsub_rn(vp, s.mu), __dmul_rn(s.phi, __dsub_rn(v, s.mu)))),
                               s.inv_se2));
  return g;
}

__device__ __forceinline__ bool h_bad(double v) { return !(-50.0 <= v && v <= 50.0); }

// One elementary step (K1 -> K2 -> K3, integrator.py:139-146) streamed over
// all sites: 4 sites per thread, the neighbours' first half-drift recomputed
// locally, so the three barrier-separated reference kernels become one pass
// (48 B/site of HBM traffic: read h, p, (y/2)y, lnRV; write h, p).  Out of
// place (the halo reads would race with other blocks' writes otherwise).
__global__ void __launch_bounds__(ES_NT) estep_kernel(const double *__restrict__ h, const double *__restrict__ p,
                                                      double *__restrict__ ho, double *__restrict__ po,
                                                      const double *__restrict__ a, const double *__restrict__ lrv,
                                                      const DevParams *prm, double dt, int64_t T, int32_t *flag) {
  const RefScal s = ref_scal(*prm);
  const double c = __dmul_rn(0.5, dt);
  const int64_t i0 = ((int64_t)blockIdx.x * ES_NT + threadIdx.x) * ES_R;
  if (i0 >= T) return;
  double hh[ES_R + 2], pv[ES_R + 2], av[ES_R], lv[ES_R];
  const bool full = i0 + ES_R <= T;
  if (full) {
    const double2 h01 = __ldcs(reinterpret_cast<const double2 *>(h + i0));
    const double2 h23 = __ldcs(reinterpret_cast<const double2 *>(h + i0 + 2));
    const double2 p01 = __ldcs(reinterpret_cast<const double2 *>(p + i0));
    const double2 p23 = __ldcs(reinterpret_cast<const double2 *>(p + i0 + 2));
    const double2 a01 = __ldcs(reinterpret_cast<const double2 *>(a + i0));
    const double2 a23 = __ldcs(reinterpret_cast<const double2 *>(a + i0 + 2));
    const double2 l01 = __ldcs(reinterpret_cast<const double2 *>(lrv + i0));
    const double2 l23 = __ldcs(reinterpret_cast<const double2 *>(lrv + i0 + 2));
    hh[1] = h01.x; hh[2] = h01.y; hh[3] = h23.x; hh[4] = h23.y;
    pv[1] = p01.x; pv[2] = p01.y; pv[3] = p23.x; pv[4] = p23.y;
    av[0] = a01.x; av[1] = a01.y; av[2] = a23.x; av[3] = a23.y;
    lv[0] = l01.x; lv[1] = l01.y; lv[2] = l23.x; lv[3] = l23.y;
  } else {
#pragma unroll
    for (int r = 0; r < ES_R; r++) {
      const bool in = i0 + r < T;
      hh[r + 1] = in ? h[i0 + r] : 0.0;
      pv[r + 1] = in ? p[i0 + r] : 0.0;
      av[r] = in ? a[i0 + r] : 0.0;
      lv[r] = in ? lrv[i0 + r] : 0.0;
    }
  }
  hh[0] = i0 > 0 ? h[i0 - 1] : 0.0;
  pv[0] = i0 > 0 ? p[i0 - 1] : 0.0;
  hh[ES_R + 1] = i0 + ES_R < T ? h[i0 + ES_R] : 0.0;
  pv[ES_R + 1] = i0 + ES_R < T ? p[i0 + ES_R] : 0.0;
#pragma unroll
  for (int r = 0; r < ES_R + 2; r++) hh[r] = __dadd_rn(hh[r], __dmul_rn(c, pv[r]));  // kernel 1
  int bad = 0;
  double hn[ES_R], pn[ES_R];
#pragma unroll
  for (int r = 0; r < ES_R; r++) {
    const int64_t i = i0 + r;
    const double v = hh[r + 1];
    bad |= (i < T) && h_bad(v);
    const double g = grad_site_ref(v, hh[r], hh[r + 2], i > 0, i < T - 1, av[r], lv[r], s);
    pn[r] = __dsub_rn(pv[r + 1], __dmul_rn(dt, g));  // kernel 2
    hn[r] = __dadd_rn(v, __dmul_rn(c, pn[r]));       // kernel 3
  }
  if (full) {
    __stcs(reinterpret_cast<double2 *>(ho + i0), make_double2(hn[0], hn[1]));
    __stcs(reinterpret_cast<double2 *>(ho + i0 + 2), make_double2(hn[2], hn[3]));
    __stcs(reinterpret_cast<double2 *>(po + i0), make_double2(pn[0], pn[1]));
    __stcs(reinterpret_cast<double2 *>(po + i0 + 2), make_double2(pn[2], pn[3]));
  } else {
    for (int r = 0; r < ES_R; r++)
      if (i0 + r < T) { ho[i0 + r] = hn[r]; po[i0 + r] = pn[r]; }
  }
  if (bad) atomicOr(flag, 1);
}

int launch_elementary_step(const double *h, const double *p, double *ho, double *po, const double *a,
                           const double *lrv, const DevParams *prm, double dt, int64_t T, int32_t *flag,
                           cudaStream_t st, int *launches) {
  const int64_t threads = (T + ES_R - 1) / ES_R;
  estep_kernel<<<(unsigned)((threads + ES_NT - 1) / ES_NT), ES_NT, 0, st>>>(h, p, ho, po, a, lrv, prm, dt, T, flag);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---- kernel-level plug-in kernels (exact reference arithmetic) -------------
__global__ void pos_kernel(double *h, const double *p, double c, int64_t lo, int64_t hi) {
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi) h[i] = __dadd_rn(h[i], __dmul_rn(c, p[i]));
}
__global__ void mom_kernel(const double *h, double *p, const double *y, const double *lrv, double dt, PackedScal sc,
                           int64_t n, int64_t lo, int64_t hi, int32_t *flag, int fill_grad) {
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  RefScal s;
  s.half = sc.v[0]; s.phi = sc.v[1]; s.mu = sc.v[2]; s.xi = sc.v[3];
  s.inv_su2 = sc.v[4]; s.inv_se2 = sc.v[5]; s.one_m_phi2 = sc.v[6];
  const double v = h[i];
  const double yy = __dmul_rn(__dmul_rn(s.half, y[i]), y[i]);
  const double g = grad_site_ref(v, i > 0 ? h[i - 1] : 0.0, i < n - 1 ? h[i + 1] : 0.0, i > 0, i < n - 1, yy, lrv[i], s);
  if (fill_grad) p[i] = g;
  else p[i] = __dsub_rn(p[i], __dmul_rn(dt, g));
  if (h_bad(v)) atomicOr(flag, 1);
}

int launch_position_update(double *h, const double *p, double c, int64_t lo, int64_t hi, cudaStream_t s,
                           int *launches) {
  if (hi <= lo) return 0;
  pos_kernel<<<(unsigned)((hi - lo + 255) / 256), 256, 0, s>>>(h, p, c, lo, hi);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
int launch_momentum_update(const double *h, double *p, const double *y, const double *lrv, double dt,
                           PackedScal sc, int64_t n, int64_t lo, int64_t hi, int32_t *flag, cudaStream_t s,
                           int *launches) {
  if (hi <= lo) return 0;
  mom_kernel<<<(unsigned)((hi - lo + 255) / 256), 256, 0, s>>>(h, p, y, lrv, dt, sc, n, lo, hi, flag, 0);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
int launch_gradient(const double *h, const double *y, const double *lrv, PackedScal sc, double *out, int64_t n,
                    int64_t lo, int64_t hi, int32_t *flag, cudaStream_t s, int *launches) {
  if (hi <= lo) return 0;
  mom_kernel<<<(unsigned)((hi - lo + 255) / 256), 256, 0, s>>>(h, out, y, lrv, 0.0, sc, n, lo, hi, flag, 1);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---- deterministic reductions (model.py:134-182, sampler.py:170-272) ------
constexpr int RD_NT = 256, RD_R = 4, RD_NV = 6;
int reduce_partials_count(int64_t T) { return (int)((T + RD_NT * RD_R - 1) / (RD_NT * RD_R)); }

// mode 0: energy sums {sum p^2, sum h, sum y^2 e^-h, sum (lrv-xi-h)^2, sum tr^2, 0}
// mode 1: statistics   {sum d, sum d^2, sum d d_prev, sum e, sum e^2, 0}
__global__ void __launch_bounds__(RD_NT) reduce1_kernel(const double *h, const double *p, const double *y,
                                                        const double *lrv, const DevParams *prm, int64_t T,
                                                        double c_mu, double c_xi, int mode, double *partials) {
  __shared__ double s_red[RD_NT / 32][RD_NV];
  DevParams P = {0, 0, 0, 1, 1};
  if (mode == 0) P = *prm;
  double v[RD_NV] = {0, 0, 0, 0, 0, 0};
  const int64_t i0 = ((int64_t)blockIdx.x * RD_NT + threadIdx.x) * RD_R;
  for (int r = 0; r < RD_R; r++) {
    const int64_t i = i0 + r;
    if (i >= T) break;
    const double hv = h[i];
    if (mode == 0) {
      v[0] += p[i] * p[i];
      v[1] += hv;
      v[2] += y[i] * y[i] * exp(-hv);
      const double ru = lrv[i] - P.xi - hv;
      v[3] += ru * ru;
      if (i > 0) {
        const double tr = (hv - P.mu) - P.phi * (h[i - 1] - P.mu);
        v[4] += tr * tr;
      }
    } else {
      const double d = hv - c_mu, e = lrv[i] - hv - c_xi;
      v[0] += d;
      v[1] += d * d;
      if (i > 0) v[2] += d * (h[i - 1] - c_mu);
      v[3] += e;
      v[4] += e * e;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < RD_NV; k++)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
    for (int k = 0; k < RD_NV; k++) s_red[warp][k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < RD_NV; k++) {
      double acc = s_red[0][k];
      for (int w = 1; w < RD_NT / 32; w++) acc += s_red[w][k];
      partials[(int64_t)blockIdx.x * RD_NV + k] = acc;
    }
  }
}

__global__ void __launch_bounds__(RD_NT) reduce2_kernel(const double *partials, int nparts, const double *h,
                                                        const DevParams *prm, int64_t T, double c_mu, int mode,
                                                        double *out) {
  __shared__ double s_v[RD_NT][RD_NV];
  double v[RD_NV] = {0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < nparts; i += RD_NT)
    for (int k = 0; k < RD_NV; k++) v[k] += partials[(int64_t)i * RD_NV + k];
  for (int k = 0; k < RD_NV; k++) s_v[threadIdx.x][k] = v[k];
  __syncthreads();
  for (int w = RD_NT / 2; w >= 1; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < RD_NV; k++) s_v[threadIdx.x][k] += s_v[threadIdx.x + w][k];
    __syncthreads();
  }
  if (threadIdx.x) return;
  const double *t = s_v[0];
  if (mode == 0) {
    const DevParams P = *prm;
    const double Td = (double)T;
    const double se2 = P.se2, su2 = P.su2, phi = P.phi;
    const double d0 = h[0] - P.mu;
    const double returns_block = -0.5 * t[1] - 0.5 * t[2];
    const double rv_block = -0.5 * Td * log(su2) - t[3] / (2.0 * su2);
    const double ar_block = -0.5 * log(se2 / (1.0 - phi * phi)) - (1.0 - phi * phi) * d0 * d0 / (2.0 * se2) -
                            0.5 * (Td - 1.0) * log(se2) - t[4] / (2.0 * se2);
    out[0] = 0.5 * t[0];
    out[1] = returns_block + rv_block + ar_block;
  } else {
    out[0] = h[0] - c_mu;
    out[1] = h[T - 1] - c_mu;
    for (int k = 0; k < 5; k++) out[2 + k] = t[k];
  }
}

int launch_energy(const double *h, const double *p, const double *y, const double *lrv, const DevParams *prm,
                  int64_t T, double *partials, double *out, cudaStream_t s, int *launches) {
  const int nb = reduce_partials_count(T);
  reduce1_kernel<<<nb, RD_NT, 0, s>>>(h, p, y, lrv, prm, T, 0.0, 0.0, 0, partials);
  reduce2_kernel<<<1, RD_NT, 0, s>>>(partials, nb, h, prm, T, 0.0, 0, out);
  *launches += 2;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
int launch_suff_stats(const double *h, const double *lrv, int64_t T, double c_mu, double c_xi, double *partials,
                      double *out, cudaStream_t s, int *launches) {
  const int nb = reduce_partials_count(T);
  reduce1_kernel<<<nb, RD_NT, 0, s>>>(h, nullptr, nullptr, lrv, nullptr, T, c_mu, c_xi, 1, partials);
  reduce2_kernel<<<1, RD_NT, 0, s>>>(partials, nb, h, nullptr, T, c_mu, 1, out);
  *launches += 2;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace rsv
