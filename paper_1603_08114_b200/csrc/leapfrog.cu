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

__device__ __align__(128) const unsigned long long g_exp_tab2[RSV_EXP_TAB_N] = RSV_EXP_TAB2_INIT;

constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
constexpr int EXP_HI_SHIFT = 20 - RSV_EXP_TAB_BITS;

// exp(-d) for the model's range.  n = rint(-2048 d / ln2) via the magic-number
// add, r = -d - n ln2/2048 (Cody-Waite, two FMAs), e^r - 1 by a degree-3
// Horner polynomial (|r| <= ln2/4096, truncation ~3e-17), and S = 2^(n/2048)
// built exactly from a scale-ready table entry (bits(2^(j/2048)) - (j << 41))
// plus n << 41: one shared-memory load and one integer add.  8 FP64
// instructions, <= 1.3 ulp (tools/gen_exp_table.py).
// `t` is returned for the integer range test of the divergence flag.
__device__ __forceinline__ double exp_neg(double d, const unsigned long long *tab, double &t) {
  t = fma(-d, RSV_INV_LN2_N, MAGIC);
  const double nd = t - MAGIC;
  double r = fma(nd, -RSV_LN2_N_HI, -d);
  r = fma(nd, -RSV_LN2_N_LO, r);
  double q = fma(r, 1.0 / 6.0, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const int n = __double2loint(t);
  const unsigned long long tb = tab[n & (RSV_EXP_TAB_N - 1)];
  const double S = __hiloint2double((int)(tb >> 32) + (n << EXP_HI_SHIFT), (int)(unsigned)tb);
  return fma(S, q, S);
}

// Same evaluation, constants taken from the kernel's parameter block so the
// hot loop uses constant-bank operands (no per-iteration immediates).
template <typename K>
__device__ __forceinline__ double exp_neg_k(double d, const unsigned long long *tab, double &t, const K &k) {
  t = fma(-d, k.e_k, MAGIC);
  const double nd = t - MAGIC;
  double r = fma(nd, -k.e_hi, -d);
  r = fma(nd, -k.e_lo, r);
  double q = fma(r, k.e_c3, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const int n = __double2loint(t);
  const unsigned long long tb = tab[n & (RSV_EXP_TAB_N - 1)];
  const double S = __hiloint2double((int)(tb >> 32) + (n << EXP_HI_SHIFT), (int)(unsigned)tb);
  return fma(S, q, S);
}

// |h| <= 50 <=> n in [n_lo, n_lo + span]; NaN or huge d leave the magic
// sum's high word outside {0x4337FFFF, 0x43380000}.  Integer ops only.
__device__ __forceinline__ bool out_of_range(double t, int n_lo, int n_span) {
  const int n = __double2loint(t);
  const unsigned hw = (unsigned)__double2hiint(t) - 0x4337FFFFu;
  return ((unsigned)(n - n_lo) > (unsigned)n_span) | (hw > 1u);
}


// Variable part of H at one site (the theta-only constants are added in
// the Metropolis step): 0.5 p^2 + 0.5 d + a e^{-mu} e^{-d} + (q-d)^2/2su2 + AR.
template <bool KIN = true>
__device__ __forceinline__ double site_energy(double d, double dprev, double p, double ae, double q, bool first,
                                              const TrajConsts &s, const unsigned long long *tab) {
  double t;
  const double E = exp_neg(d, tab, t);
  const double r = q - d;
  const double tr = d - s.phi * dprev;
  const double ar = first ? s.one_m_phi2 * d * d * s.inv2se : tr * tr * s.inv2se;
  if (!KIN) return 0.5 * d + ae * E + r * r * s.inv2su + ar;  // potential part (momenta not yet drawn)
  return 0.5 * p * p + 0.5 * d + ae * E + r * r * s.inv2su + ar;
}

// Energies and statistics of the thread's owned core sites (branch-free on
// the common path; `edge` threads handle the global first site).
// firstm bit r: site r is the first of its series (stationary AR prior, no
// predecessor term).
// KIN = false: the potential part only (the caller adds 0.5 p^2 later).
template <int R, bool STATS = true, bool KIN = true>
__device__ __forceinline__ void tile_energy(const double (&d)[R], const double (&p)[R], const double (&av)[R],
                                            const double (&lv)[R], double dl, uint32_t core, uint32_t firstm,
                                            const TrajConsts &s, const unsigned long long *tab, double (&v)[6]) {
#pragma unroll
  for (int r = 0; r < R; r++) {
    const double dprev = r ? d[r - 1] : dl;
    const double q = lv[r] - s.xm;
    const bool first = (firstm >> r) & 1;
    const double en = site_energy<KIN>(d[r], dprev, p[r], s.emu * av[r], q, first, s, tab);
    const bool c = (core >> r) & 1;
    v[0] += c ? en : 0.0;
    if (STATS) {
      const double e = q - d[r];
      v[1] += c ? d[r] : 0.0;
      v[2] += c ? d[r] * d[r] : 0.0;
      v[3] += (c && !first) ? d[r] * dprev : 0.0;
      v[4] += c ? e : 0.0;
      v[5] += c ? e * e : 0.0;
    }
  }
}

// Exchange the first / last register site with the neighbouring threads.
template <int NW>
__device__ __forceinline__ void exchange(double first, double last, double &left, double &right, double *s_first,
                                         double *s_last, int lane, int warp) {
  left = __shfl_up_sync(0xffffffffu, last, 1);
  right = __shfl_down_sync(0xffffffffu, first, 1);
  if (lane == 31) s_last[warp] = last;
  if (lane == 0) s_first[warp] = first;
  __syncthreads();
  if (lane == 0) left = warp > 0 ? s_last[warp - 1] : 0.0;
  if (lane == 31) right = warp < NW - 1 ? s_first[warp + 1] : 0.0;
}

// Fixed-order block sum (deterministic): warp butterflies, then warp totals
// in warp order by thread 0.
template <int NV, int NW>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *s_red, int lane, int warp) {
#pragma unroll
  for (int k = 0; k < NV; k++) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; k++) s_red[warp * NV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; k++) {
      double acc = s_red[k];
      for (int w = 1; w < NW; w++) acc += s_red[w * NV + k];
      v[k] = acc;
    }
  }
}

// One kick p -= dt * dU/dh for the thread's R sites (d-space):
//   p <- p - Cd - G d + beta phi (d_{i-1} + d_{i+1}) + Ad e^{-d}
// The divergence test (|h| > 50) is accumulated as the largest
// (unsigned)(n - n_lo) over the thread's core sites and checked once at the
// end; NaN or astronomically large states (which no longer map to a sane n)
// propagate to a non-finite dH, which the Metropolis step rejects the same
// way (sampler.py:157-162).
template <bool EDGE, int R>
__device__ __forceinline__ void kick(double (&d)[R], double (&p)[R], const double (&Ad)[R],
                                     const double (&Cd)[R], double dl, double dr, const TrajConsts &s,
                                     const unsigned long long *tab, uint32_t live, uint32_t endm,
                                     const unsigned (&cm)[R], unsigned &nmax) {
#pragma unroll
  for (int r = 0; r < R; r++) {
    const double dm = r ? d[r - 1] : dl;
    const double dp = r < R - 1 ? d[r + 1] : dr;
    double t;
    const double E = exp_neg_k(d[r], tab, t, s);
    // lean warps: each thread's sites are all core or none (the caller keeps
    // the thread's maximum only in the first case), so no per-site mask
    if (EDGE) nmax = max(nmax, ((unsigned)__double2loint(t) - (unsigned)s.n_lo) & cm[r]);
    else nmax = max(nmax, (unsigned)__double2loint(t) - (unsigned)s.n_lo);
    const double G = EDGE && ((endm >> r) & 1) ? s.g_end : s.g_int;
    double pp = p[r] - Cd[r];
    pp = fma(-G, d[r], pp);
    pp = fma(s.bphi, dm + dp, pp);
    pp = fma(Ad[r], E, pp);
    p[r] = (EDGE && !((live >> r) & 1)) ? 0.0 : pp;
  }
}

template <int R>
__device__ __forceinline__ void drift(double (&d)[R], const double (&p)[R], double c) {
#pragma unroll
  for (int r = 0; r < R; r++) d[r] = fma(c, p[r], d[r]);
}

template <int R, int NT>
__device__ __forceinline__ void ghost_refresh(double (&d)[R], double (&p)[R], double *s_gx, int lane, int warp,
                                              int parity);

// The L leapfrog steps of a tile (integrator.py:149-179), unrolled by the
// ghost-refresh period R: loop control and the refresh test once per R
// steps.  EDGE is warp-uniform (masked kick for partially live / end / mixed
// core threads).  cf / cl: ensemble chain boundaries cut the coupling.
template <bool EDGE, int R, int NT, bool FUSE, bool ENS>
__device__ __forceinline__ void run_steps(double (&d)[R], double (&p)[R], const double (&Ad)[R],
                                          const double (&Cd)[R], const TrajConsts &s,
                                          const unsigned long long *tab, uint32_t live, uint32_t endm,
                                          const unsigned (&cm)[R], bool cf, bool cl, int L, double *gx, int lane,
                                          int warp, unsigned &nmax) {
  constexpr int NW = NT / 32;
  int gpar = 0;
  auto one = [&](int step) {
    if (!FUSE) drift(d, p, s.c_half);
    // lanes 0 / 31 get their own value back: those are ghost lanes (or the
    // CTA window edges, inside the halo) whose stale values never reach a
    // core site; next to a global end the neighbour lane is non-live (d = 0)
    double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
    double dr = __shfl_down_sync(0xffffffffu, d[0], 1);
    if (ENS) {  // no coupling across chain boundaries
      dl = cf ? 0.0 : dl;
      dr = cl ? 0.0 : dr;
    }
    kick<EDGE, R>(d, p, Ad, Cd, dl, dr, s, tab, live, endm, cm, nmax);
    if (FUSE) drift(d, p, step < L - 1 ? s.c_full : s.c_half);
    else drift(d, p, s.c_half);
  };
  if (FUSE) drift(d, p, s.c_half);
  int step = 0;
  for (; step + R <= L; step += R) {
#pragma unroll
    for (int u = 0; u < R; u++) one(step + u);
    if (NW > 1 && step + R < L) {
      ghost_refresh<R, NT>(d, p, gx, lane, warp, gpar);
      gpar ^= 1;
    }
  }
  for (; step < L; step++) one(step);
  if (NW > 1) ghost_refresh<R, NT>(d, p, gx, lane, warp, gpar);
}

// Metropolis step (sampler.py:155-167) on the tile partials, run by the last
// tile to finish; deterministic (fixed-order sums).
// TilePart slot of the i-th reduced value (without statistics: 0, 1, 2, 13)
template <bool STATS>
__host__ __device__ constexpr int tr_slot(int i) {
  return STATS ? i : (i < 3 ? i : 13);
}
template <int NT, bool STATS = true>
__device__ void metropolis_n(const TrajArgs &A, double *s_v, int n_parts);
template <int NT>
__device__ __forceinline__ void metropolis(const TrajArgs &A, double *s_v) {
  metropolis_n<NT, true>(A, s_v, A.g.n_tiles);
}

// Warp windows overlap by one lane on each side ("ghost lanes"): warp w
// holds sites [w*30R, w*30R + 32R) of the CTA window, its lanes 0 and 31
// duplicate the last / first core lane of its neighbours.  Within a warp the
// stencil needs only shuffles; a ghost lane's values go stale from the
// window edge inwards one site per step, so after R steps they are refreshed
// from the neighbours' core lanes through shared memory (one CTA barrier per
// R steps).  Core lanes (1..30) are always exact; a site belongs to the one
// warp whose core lane holds it.
template <int R, int NT>
__device__ __forceinline__ void ghost_refresh(double (&d)[R], double (&p)[R], double *s_gx, int lane, int warp,
                                              int parity) {
  constexpr int NW = NT / 32;
  // s_gx layout: [parity][warp][side 0: lane 30 -> right neighbour's lane 0,
  //                                side 1: lane 1 -> left neighbour's lane 31][2R]
  double *slot = s_gx + (size_t)parity * NW * 4 * R;
  if (lane == 30 || lane == 1) {
    double *dst = slot + (warp * 2 + (lane == 1)) * 2 * R;
#pragma unroll
    for (int r = 0; r < R; r++) { dst[r] = d[r]; dst[R + r] = p[r]; }
  }
  __syncthreads();
  if (lane == 0 && warp > 0) {
    const double *src = slot + ((warp - 1) * 2 + 0) * 2 * R;
#pragma unroll
    for (int r = 0; r < R; r++) { d[r] = src[r]; p[r] = src[R + r]; }
  }
  if (lane == 31 && warp < NW - 1) {
    const double *src = slot + ((warp + 1) * 2 + 1) * 2 * R;
#pragma unroll
    for (int r = 0; r < R; r++) { d[r] = src[r]; p[r] = src[R + r]; }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RSV_STAMP(k)                                                                  \
  do {                                                                                \
    if (A.dbg && threadIdx.x == 0) A.dbg[(size_t)blockIdx.x * 8 + (k)] = gtimer(); \
  } while (0)

template <int R, int NT, int MINB, bool FUSE>
__global__ void __launch_bounds__(NT, MINB) traj_kernel(TrajArgs A) {
  constexpr int NW = NT / 32;
  constexpr int WSTEP = 30 * R;  // window advance per warp
  RSV_STAMP(0);
  __shared__ unsigned long long s_tab[RSV_EXP_TAB_N];
  __shared__ double s_first[NW], s_last[NW];
  __shared__ double s_red[NW * TR_NV];
  __shared__ double s_v[NW * TR_NV + TR_NV];
  __shared__ double s_gx[2 * NW * 4 * R];
  __shared__ double s_old[6 * NT];
  __shared__ int s_last_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < RSV_EXP_TAB_N; i += NT) s_tab[i] = g_exp_tab2[i];

  const TrajConsts &s = A.k;
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
  const int H = A.g.halo;                    // multiple of R (>= n_steps + 1)
  const int64_t t0 = (int64_t)blockIdx.x * A.g.core;  // core is a multiple of R
  const int64_t t1 = min(t0 + A.g.core, T);
  // live range [t0 - H, t1 + H): lanes start on multiples of R, so only the
  // lanes at the global ends of the series hold partially live sites
  const int64_t lo_live = max((int64_t)0, t0 - H), hi_live = min(T, t1 + H);
  const int64_t g0 = t0 - H + (int64_t)warp * WSTEP + (int64_t)lane * R;
  const bool own_lane = (lane >= 1 && lane <= 30) || (lane == 0 && warp == 0) || (lane == 31 && warp == NW - 1);

  // ---- load: vectorised when the lane's R sites are all live ----
  double d[R], p[R], av[R], lv[R];
  const bool full = g0 >= lo_live && g0 + R <= hi_live;
  if (full) {
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const double2 h2 = __ldg(reinterpret_cast<const double2 *>(hsrc + g0 + r));
      const double2 p2 = __ldg(reinterpret_cast<const double2 *>(A.p_in + g0 + r));
      const double2 a2 = __ldg(reinterpret_cast<const double2 *>(A.a + g0 + r));
      const double2 l2 = __ldg(reinterpret_cast<const double2 *>(A.lrv + g0 + r));
      d[r] = h2.x; d[r + 1] = h2.y;
      p[r] = p2.x; p[r + 1] = p2.y;
      av[r] = a2.x; av[r + 1] = a2.y;
      lv[r] = l2.x; lv[r + 1] = l2.y;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t gi = g0 + r;
      const bool in = gi >= lo_live && gi < hi_live;
      d[r] = in ? hsrc[gi] : s.mu;
      p[r] = in ? A.p_in[gi] : 0.0;
      av[r] = in ? A.a[gi] : 0.0;
      lv[r] = in ? A.lrv[gi] : 0.0;
    }
  }
  uint32_t live = 0, core = 0, endm = 0;
  double Ad[R], Cd[R];
  unsigned cm[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int64_t gi = g0 + r;
    const bool in = gi >= lo_live && gi < hi_live;
    const bool c = in && own_lane && gi >= t0 && gi < t1;
    live |= (uint32_t)in << r;
    core |= (uint32_t)c << r;
    endm |= (uint32_t)(gi == 0 || gi == T - 1) << r;
    cm[r] = c ? ~0u : 0u;
    d[r] = d[r] - s.mu;
    Ad[r] = s.dt * (s.emu * av[r]);
    Cd[r] = in ? fma(-s.alpha, lv[r] - s.xm, s.half_dt) : 0.0;
  }
  const bool any_live = live != 0;
  const bool edge = (any_live && live != (1u << R) - 1) || endm;
  __syncthreads();  // s_tab

  // ---- H_old and statistics of the current path (owned core sites) ----
  double hold;
  {
    double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
    double v[6] = {0, 0, 0, 0, 0, 0};
    tile_energy<R>(d, p, av, lv, dl, core, (edge && g0 <= 0 && g0 + R > 0) ? 1u << (int)(-g0) : 0u, s, s_tab, v);
    hold = v[0];
    asm volatile("" ::: "memory");
#pragma unroll
    for (int k = 0; k < 6; k++) s_old[k * NT + tid] = v[k];  // reduced with the new ones at the end
    if (edge && !A.h_src) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if ((core >> r) & 1) {
          if (g0 + r == 0) A.ctrl->ends_old[0] = d[r];
          if (g0 + r == T - 1) A.ctrl->ends_old[1] = d[r];
        }
      }
    }
  }

  // ---- the trajectory: shuffles only, ghost lanes refreshed every R steps ----
  RSV_STAMP(2);
  const bool masked = edge || (core != 0 && core != (1u << R) - 1);
  unsigned nmax = 0;
  const int L = A.n_steps;
  int parity = 0;
  if (FUSE) drift(d, p, s.c_half);
  for (int step = 0; step < L; step++) {
    if (!FUSE) drift(d, p, s.c_half);
    double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
    double dr = __shfl_down_sync(0xffffffffu, d[0], 1);
    if (lane == 0) dl = 0.0;   // window edges: stale ghosts, never read by core results
    if (lane == 31) dr = 0.0;
    if (masked) kick<true, R>(d, p, Ad, Cd, dl, dr, s, s_tab, live, endm, cm, nmax);
    else if (any_live) kick<false, R>(d, p, Ad, Cd, dl, dr, s, s_tab, live, endm, cm, nmax);
    if (FUSE) drift(d, p, step < L - 1 ? s.c_full : s.c_half);
    else drift(d, p, s.c_half);
    if (NW > 1 && (step + 1) % R == 0 && step + 1 < L) {
      ghost_refresh<R, NT>(d, p, s_gx, lane, warp, parity);
      parity ^= 1;
    }
  }
  if (NW > 1) ghost_refresh<R, NT>(d, p, s_gx, lane, warp, parity);  // exact d_{i-1} for the energies
  if (!masked && !core) nmax = 0;  // the lean kick does not mask non-core sites
  const bool bad = nmax > (unsigned)s.n_span;
  RSV_STAMP(3);

  // ---- H_new, statistics of the proposal, write-back ----
  {
    // reload the static per-site data (L2-resident) rather than holding it
    // in registers through the trajectory
    if (full) {
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        const double2 a2 = __ldg(reinterpret_cast<const double2 *>(A.a + g0 + r));
        const double2 l2 = __ldg(reinterpret_cast<const double2 *>(A.lrv + g0 + r));
        av[r] = a2.x; av[r + 1] = a2.y;
        lv[r] = l2.x; lv[r + 1] = l2.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; r++) {
        const int64_t gi = g0 + r;
        const bool in = gi >= lo_live && gi < hi_live;
        av[r] = in ? A.a[gi] : 0.0;
        lv[r] = in ? A.lrv[gi] : 0.0;
      }
    }
    double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
    double v[6] = {0, 0, 0, 0, 0, 0};
    tile_energy<R>(d, p, av, lv, dl, core, (edge && g0 <= 0 && g0 + R > 0) ? 1u << (int)(-g0) : 0u, s, s_tab, v);
    const int64_t gi0 = g0;
    if (full && core == (1u << R) - 1) {
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        *reinterpret_cast<double2 *>(hdst + gi0 + r) = make_double2(d[r] + s.mu, d[r + 1] + s.mu);
        if (A.p_out) *reinterpret_cast<double2 *>(A.p_out + gi0 + r) = make_double2(p[r], p[r + 1]);
      }
    } else if (core) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if ((core >> r) & 1) {
          hdst[gi0 + r] = d[r] + s.mu;
          if (A.p_out) A.p_out[gi0 + r] = p[r];
        }
      }
    }
    if (edge && !A.h_src) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if ((core >> r) & 1) {
          if (g0 + r == 0) A.ctrl->ends_new[0] = d[r];
          if (g0 + r == T - 1) A.ctrl->ends_new[1] = d[r];
        }
      }
    }
    double w[TR_NV];
    w[0] = v[0] - hold;
    w[1] = s_old[0 * NT + tid];
    w[2] = v[0];
#pragma unroll
    for (int k = 0; k < 5; k++) {
      w[3 + k] = s_old[(k + 1) * NT + tid];
      w[8 + k] = v[1 + k];
    }
    w[13] = bad ? 1.0 : 0.0;
    __syncthreads();  // s_red reuse
    block_sum<TR_NV, NW>(w, s_red, lane, warp);
    if (tid == 0) {
      TilePart *tp = A.parts + blockIdx.x;
      tp->dh = w[0];
      tp->hold = w[1];
      tp->hnew = w[2];
      for (int k = 0; k < 5; k++) {
        tp->so[k] = w[3 + k];
        tp->sn[k] = w[8 + k];
      }
      tp->flag = w[13];
      __threadfence();
      const unsigned done = atomicAdd(&A.ctrl->tiles_done, 1u);
      s_last_tile = (done == (unsigned)gridDim.x - 1);
    }
  }
  RSV_STAMP(4);
  __syncthreads();
  if (s_last_tile) {
    __threadfence();
    metropolis<NT>(A, s_v);
    RSV_STAMP(5);
  }
  (void)s_first;
  (void)s_last;
}

// ---------------------------------------------------------------------------
// Persistent, TMA-staged trajectory kernel.  The grid is MINB CTAs per SM;
// CTA c runs tiles c, c + G, c + 2G, ...  While a tile's trajectory runs in
// registers, the next tile's h, p, (y/2)y and lnRV windows stream from HBM
// into shared memory with 1-D bulk-tensor copies (cp.async.bulk, completion
// on an mbarrier), so the HBM latency of a tile is hidden behind the
// previous tile's FP64 work.  Per-thread energy / statistics partials are
// accumulated in shared memory across tiles and reduced once per CTA.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Issue the window [t0 - H, t0 - H + W) of the four arrays into stage[4][W]
// (clamped to [0, Tpad); arrays are padded to a multiple of 8 doubles).
// part: 1 = h, (y/2)y, lnRV, 2 = the momenta, 3 = all, each on `bar` with
// its own byte count (the first tile stages parts 1 and 2 on two barriers).
template <int W>
__device__ __forceinline__ void stage_tile(const TrajArgs &A, const double *hsrc, int tile, double *stage,
                                           uint64_t *bar, int part = 3) {
  const int64_t g = (int64_t)tile * A.g.core - A.g.halo;
  const int64_t lo = g < 0 ? 0 : g, hi = min(g + W, A.Tpad);
  const uint32_t bytes = (uint32_t)((hi - lo) * 8);
  const int off = (int)(lo - g);
  mbar_expect_tx(bar, (part == 3 ? 4 : part == 1 ? 3 : 1) * bytes);
  if (part & 1) {
    tma_load_1d(stage + 0 * W + off, hsrc + lo, bytes, bar);
    tma_load_1d(stage + 2 * W + off, A.a + lo, bytes, bar);
    tma_load_1d(stage + 3 * W + off, A.lrv + lo, bytes, bar);
  }
  if (part & 2) tma_load_1d(stage + 1 * W + off, A.p_in + lo, bytes, bar);
}

// Ensemble: the h window is split at chain boundaries, each piece read from
// its chain's current buffer (boundaries sit on multiples of Tc, a multiple of
// 8 sites, so every piece stays 16-byte aligned).
template <int W>
__device__ __forceinline__ void stage_tile_ens(const TrajArgs &A, int tile, double *stage, uint64_t *bar) {
  const int64_t g = (int64_t)tile * A.g.core - A.g.halo;
  const int64_t lo = g < 0 ? 0 : g, hi = min(g + W, A.Tpad);
  const uint32_t bytes = (uint32_t)((hi - lo) * 8);
  const int off = (int)(lo - g);
  mbar_expect_tx(bar, 4 * bytes);
  for (int64_t x = lo; x < hi;) {
    const int64_t c = x / A.Tc;
    const int64_t e = min(hi, (c + 1) * A.Tc);
    const double *src = (A.ens_cur[c] ? A.hbuf1 : A.hbuf0) + x;
    tma_load_1d(stage + 0 * W + (x - g), src, (uint32_t)((e - x) * 8), bar);
    x = e;
  }
  tma_load_1d(stage + 1 * W + off, A.p_in + lo, bytes, bar);
  tma_load_1d(stage + 2 * W + off, A.a + lo, bytes, bar);
  tma_load_1d(stage + 3 * W + off, A.lrv + lo, bytes, bar);
}

template <int R, int NT>
struct PersistSmem {
  static constexpr int NW = NT / 32;
  static constexpr int W = NW > 1 ? NW * 30 * R + 2 * R : 32 * R;
  double stage[2][4 * W];       // double-buffered tile windows
  double acc[TR_NV * NT];       // per-thread partials across tiles
  double gx[2 * NW * 4 * R];    // ghost-lane refresh slots
  double red[NW * TR_NV];
  double v[NW * TR_NV + TR_NV];
  alignas(16) unsigned long long tab[RSV_EXP_TAB_N];
  double epart[2][NW][8];  // ensemble: per-warp chain partials of a tile (by staging buffer)
  uint64_t bar[4];  // two staging buffers, the exp table, the first tile's momenta
  int last;
};

template <int R, int NT, int MINB, bool FUSE, bool STATS, bool ENS = false, bool DEVK = false>
__global__ void __launch_bounds__(NT, MINB) traj_persistent_kernel(TrajArgs A) {
  using SM = PersistSmem<R, NT>;
  constexpr int NW = SM::NW, W = SM::W;
  constexpr int WSTEP = 30 * R;
  extern __shared__ __align__(128) unsigned char psmem[];
  SM &S = *reinterpret_cast<SM *>(psmem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // DEVK (run_chain on the device): the theta-dependent constants come from
  // device memory, written by the theta kernel of the previous sweep; the
  // others stay constant-bank operands of the parameter block
  TrajConsts sk = A.k;
  if (DEVK) {
    const TrajConsts &q = *A.kdev;
    sk.mu = q.mu; sk.phi = q.phi; sk.alpha = q.alpha; sk.bphi = q.bphi; sk.g_int = q.g_int;
    sk.g_end = q.g_end; sk.emu = q.emu; sk.xm = q.xm; sk.inv2su = q.inv2su; sk.inv2se = q.inv2se;
    sk.one_m_phi2 = q.one_m_phi2; sk.hconst = q.hconst; sk.n_lo = q.n_lo; sk.n_span = q.n_span;
  }
  const TrajConsts &s = DEVK ? sk : A.k;
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
  if (tid == 0 && blockIdx.x == 0) A.ctrl->t_stamp[2] = gtimer();
  const unsigned long long t_entry = A.dbg ? gtimer() : 0ull;
  for (int k = 0; k < TR_NV; k++) S.acc[k * NT + tid] = 0.0;
  const int n_tiles = A.g.n_tiles;
  int tile = blockIdx.x;
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_init(&S.bar[2], 1);
    mbar_init(&S.bar[3], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the exp table (16 KB) arrives by one bulk copy alongside the first tile
    mbar_expect_tx(&S.bar[2], (uint32_t)sizeof(S.tab));
    tma_load_1d(S.tab, g_exp_tab2, (uint32_t)sizeof(S.tab), &S.bar[2]);
    // the first tile's h, (y/2)y and lnRV do not depend on the momenta kernel
    if (!ENS && tile < n_tiles) stage_tile<W>(A, hsrc, tile, S.stage[0], &S.bar[0], 1);
  }
  // programmatic dependent launch: everything above overlapped the momenta
  // kernel's tail; its normals (and stream bookkeeping) are read only after
  // griddepcontrol.wait -- here for ensembles, inside the first tile (after
  // its momentum-free prologue) otherwise
  if (ENS) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0 && tile < n_tiles) stage_tile_ens<W>(A, tile, S.stage[0], &S.bar[0]);
  }
  __syncthreads();
  mbar_wait(&S.bar[2], 0);
  const int64_t T = A.T;       // local series length (a shard's extended range, or the chain)
  const int64_t goff = A.goff; // global index of local site 0
  const int64_t Tg = A.Tg;     // global series length
  const int H = A.g.halo;
  const bool own_lane = (lane >= 1 && lane <= 30) || (lane == 0 && warp == 0) || (lane == 31 && warp == NW - 1);
  const int lw = warp * WSTEP + lane * R;  // my first site inside the window
  uint32_t parity[2] = {0, 0};
  int buf = 0;
  long long cyc_wait = 0, cyc_pre = 0, cyc_loop = 0, cyc_post = 0, c0, c1;
  bool first = !ENS;  // first tile of a single chain: momenta not yet readable
  for (; tile < n_tiles; tile += gridDim.x, buf ^= 1) {
    c0 = clock64();
    // the other buffer was released at the end of the previous tile: stream
    // the next tile into it while this one runs (first tile: after the wait)
    if (tid == 0 && !first && tile + (int)gridDim.x < n_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (ENS) stage_tile_ens<W>(A, tile + gridDim.x, S.stage[buf ^ 1], &S.bar[buf ^ 1]);
      else stage_tile<W>(A, hsrc, tile + gridDim.x, S.stage[buf ^ 1], &S.bar[buf ^ 1]);
    }
    const double *stg = S.stage[buf];
    const int64_t t0 = (int64_t)tile * A.g.core;
    const int64_t t1 = min(t0 + A.g.core, T);
    const int64_t lo_live = max((int64_t)0, t0 - H), hi_live = min(T, t1 + H);
    const int64_t g0 = t0 - H + lw;

    // ---- tile data from the staging buffer ----
    mbar_wait(&S.bar[buf], parity[buf]);
    parity[buf] ^= 1;
    c1 = clock64(); cyc_wait += c1 - c0; c0 = c1;
    double d[R], p[R], Ad[R], Cd[R], av[R], lv[R];
    uint32_t live = 0, core = 0, wcore = 0, endm = 0;
    unsigned cm[R];
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const double2 h2 = *reinterpret_cast<const double2 *>(stg + 0 * W + lw + r);
      const double2 a2 = *reinterpret_cast<const double2 *>(stg + 2 * W + lw + r);
      const double2 l2 = *reinterpret_cast<const double2 *>(stg + 3 * W + lw + r);
      d[r] = h2.x; d[r + 1] = h2.y;
      av[r] = a2.x; av[r + 1] = a2.y;
      lv[r] = l2.x; lv[r + 1] = l2.y;
      if (!first) {
        const double2 p2 = *reinterpret_cast<const double2 *>(stg + 1 * W + lw + r);
        p[r] = p2.x; p[r + 1] = p2.y;
      } else {
        p[r] = 0.0; p[r + 1] = 0.0;
      }
    }
    // ensemble: a thread's R sites never straddle a chain boundary (Tc and
    // the window offsets are multiples of R); cf / cl: my first / last site
    // is the first / last of its chain, so the neighbour across is cut off
    bool cf = false, cl = false;
    int64_t chain = 0;
    if (ENS) {
      const int64_t m = ((g0 % A.Tc) + A.Tc) % A.Tc;
      cf = m == 0;
      cl = m + R == A.Tc;
      chain = g0 >= 0 ? g0 / A.Tc : -1;
    }
    uint32_t firstm = 0;
    // only a lane whose sites include global site 0 or Tg-1 has end sites
    const bool near_end = (g0 + goff <= 0 && g0 + goff + R > 0) || (g0 + goff <= Tg - 1 && g0 + goff + R > Tg - 1);
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t gi = g0 + r;
      const bool in = gi >= lo_live && gi < hi_live;
      // wcore: tile-core sites of the local range (written back; a shard keeps
      // its margins evolving too); core: those this context owns (the sums)
      const bool wc = in && own_lane && gi >= t0 && gi < t1;
      const bool c = wc && gi >= A.own_lo && gi < A.own_hi;
      live |= (uint32_t)in << r;
      core |= (uint32_t)c << r;
      wcore |= (uint32_t)wc << r;
      if (ENS) {
        endm |= (uint32_t)((cf && r == 0) || (cl && r == R - 1)) << r;
        firstm |= (uint32_t)(cf && r == 0) << r;
      } else if (near_end) {
        endm |= (uint32_t)(gi + goff == 0 || gi + goff == Tg - 1) << r;
        firstm |= (uint32_t)(gi + goff == 0) << r;
      }
      cm[r] = c ? ~0u : 0u;
      d[r] = in ? d[r] - s.mu : 0.0;
      p[r] = in ? p[r] : 0.0;
      Ad[r] = in ? s.dt * (s.emu * av[r]) : 0.0;
      Cd[r] = in ? fma(-s.alpha, lv[r] - s.xm, s.half_dt) : 0.0;
    }
    const bool any_live = live != 0;
    const bool edge = (any_live && live != (1u << R) - 1) || endm;
    // warp-uniform kick path: the masked (edge) kick handles partially or
    // non-live lanes, the global end sites and threads whose sites are only
    // partly core (shard ownership); all other warps run the lean one
    const bool mixed_core = core != 0 && core != (1u << R) - 1;
    const bool warp_edge = __any_sync(0xffffffffu, edge || !any_live || mixed_core);
    // H_old of the owned core sites while a / lnRV are at hand
    double vold[6] = {0, 0, 0, 0, 0, 0};
    {
      const double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
      if (first) tile_energy<R, STATS, false>(d, p, av, lv, dl, core, firstm, s, S.tab, vold);
      else tile_energy<R, STATS>(d, p, av, lv, dl, core, firstm, s, S.tab, vold);
    }
    if (!ENS && edge && !A.h_src) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if ((core >> r) & 1) {
          if (g0 + r + goff == 0) A.ctrl->ends_old[0] = d[r];
          if (g0 + r + goff == Tg - 1) A.ctrl->ends_old[1] = d[r];
        }
      }
    }
    if (!ENS && first) {
      // the momenta kernel's normals: wait for it (everything above
      // overlapped its tail), stage this tile's momenta and the next tile
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (tid == 0) {
        stage_tile<W>(A, hsrc, tile, S.stage[buf], &S.bar[3], 2);
        if (tile + (int)gridDim.x < n_tiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          stage_tile<W>(A, hsrc, tile + gridDim.x, S.stage[buf ^ 1], &S.bar[buf ^ 1]);
        }
      }
      mbar_wait(&S.bar[3], 0);
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        const double2 p2 = *reinterpret_cast<const double2 *>(stg + 1 * W + lw + r);
        p[r] = ((live >> r) & 1) ? p2.x : 0.0;
        p[r + 1] = ((live >> (r + 1)) & 1) ? p2.y : 0.0;
      }
#pragma unroll
      for (int r = 0; r < R; r++)
        if ((core >> r) & 1) vold[0] += 0.5 * p[r] * p[r];  // kinetic part of H_old
      first = false;
    }
    const double hold = vold[0];
#pragma unroll
    for (int k = 0; k < (STATS ? 6 : 1); k++) S.acc[(k == 0 ? 1 : 2 + k) * NT + tid] += vold[k];  // slots 1, 3..7

    // ---- the trajectory ----
    c1 = clock64(); cyc_pre += c1 - c0; c0 = c1;
    unsigned nmax = 0;
    const int L = A.n_steps;
    if (warp_edge) {
      run_steps<true, R, NT, FUSE, ENS>(d, p, Ad, Cd, s, S.tab, live, endm, cm, cf, cl, L, S.gx, lane, warp, nmax);
    } else {
      run_steps<false, R, NT, FUSE, ENS>(d, p, Ad, Cd, s, S.tab, live, endm, cm, cf, cl, L, S.gx, lane, warp, nmax);
      nmax = core ? nmax : 0u;
    }
    __syncthreads();  // refresh slots reused by the next tile
    c1 = clock64(); cyc_loop += c1 - c0; c0 = c1;

    // ---- H_new, statistics, write-back ----
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const double2 a2 = *reinterpret_cast<const double2 *>(stg + 2 * W + lw + r);
      const double2 l2 = *reinterpret_cast<const double2 *>(stg + 3 * W + lw + r);
      av[r] = a2.x; av[r + 1] = a2.y;
      lv[r] = l2.x; lv[r + 1] = l2.y;
    }
    double vnew[6] = {0, 0, 0, 0, 0, 0};
    {
      const double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
      tile_energy<R, STATS>(d, p, av, lv, dl, core, firstm, s, S.tab, vnew);
    }
    double *hd = hdst;
    if (ENS && core) hd = A.ens_cur[chain] ? A.hbuf0 : A.hbuf1;
    if (wcore == (1u << R) - 1) {
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        *reinterpret_cast<double2 *>(hd + g0 + r) = make_double2(d[r] + s.mu, d[r + 1] + s.mu);
        if (A.p_out) *reinterpret_cast<double2 *>(A.p_out + g0 + r) = make_double2(p[r], p[r + 1]);
      }
    } else if (wcore) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if ((wcore >> r) & 1) {
          hd[g0 + r] = d[r] + s.mu;
          if (A.p_out) A.p_out[g0 + r] = p[r];
        }
      }
    }
    if (!ENS && edge && !A.h_src) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if ((core >> r) & 1) {
          if (g0 + r + goff == 0) A.ctrl->ends_new[0] = d[r];
          if (g0 + r + goff == Tg - 1) A.ctrl->ends_new[1] = d[r];
        }
      }
    }
    if (ENS) {
      // per-tile partials of the (<= 2) chains the core touches, in a fixed
      // order: the Metropolis step of each chain sums its tiles in tile order
      const bool right = g0 >= (t0 / A.Tc + 1) * A.Tc;
      const double fl = nmax > (unsigned)s.n_span ? 1.0 : 0.0;
      const double dhv = vnew[0] - hold;
      double w8[8] = {right ? 0.0 : dhv, right ? 0.0 : hold, right ? 0.0 : vnew[0], right ? 0.0 : fl,
                      right ? dhv : 0.0, right ? hold : 0.0, right ? vnew[0] : 0.0, right ? fl : 0.0};
      // warp butterflies only (no CTA barrier, no serial thread-0 sum): the
      // Metropolis step adds the NW warp partials of each tile in warp order
#pragma unroll
      for (int k = 0; k < 8; k++) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) w8[k] += __shfl_xor_sync(0xffffffffu, w8[k], o);
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 8; k++) S.epart[buf][warp][k] = w8[k];
      }
    } else {
      S.acc[0 * NT + tid] += vnew[0] - hold;
      S.acc[2 * NT + tid] += vnew[0];
#pragma unroll
      for (int k = 0; k < (STATS ? 5 : 0); k++) S.acc[(8 + k) * NT + tid] += vnew[1 + k];
      if (nmax > (unsigned)s.n_span) S.acc[13 * NT + tid] = 1.0;
    }
    __syncthreads();  // all reads of this tile's buffer done before it is refilled
    if (ENS && warp == 0 && lane < 8) {  // the tile's two chain records, warps summed in order
      double v = S.epart[buf][0][lane];
#pragma unroll
      for (int w = 1; w < NW; w++) v += S.epart[buf][w][lane];
      double *q = reinterpret_cast<double *>(A.ens_parts + 2 * (size_t)tile);
      q[lane] = v;  // EnsPart {dh, hold, hnew, flag} x 2
    }
    c1 = clock64(); cyc_post += c1 - c0;
  }
  if (A.dbg && tid == 0) {
    A.dbg[(size_t)blockIdx.x * 8 + 0] = cyc_wait;
    A.dbg[(size_t)blockIdx.x * 8 + 1] = cyc_pre;
    A.dbg[(size_t)blockIdx.x * 8 + 2] = cyc_loop;
    A.dbg[(size_t)blockIdx.x * 8 + 3] = cyc_post;
    A.dbg[(size_t)blockIdx.x * 8 + 4] = (tile - (int)blockIdx.x) / (int)gridDim.x;  // tiles processed
    A.dbg[(size_t)blockIdx.x * 8 + 7] = t_entry;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    A.dbg[(size_t)blockIdx.x * 8 + 5] = smid;
    A.dbg[(size_t)blockIdx.x * 8 + 6] = gtimer();
  }

  // a programmatic dependent (the theta kernel of rsv_run_chain) may launch
  // once every CTA is past its tiles; it waits for this grid's completion
  // before reading the results
  asm volatile("griddepcontrol.launch_dependents;");
  if (ENS) return;  // every chain's decision: ens_decide_kernel
  // ---- one reduction per CTA (without statistics only dh, H_old, H_new
  // and the flag: TilePart slots 0, 1, 2, 13) ----
  constexpr int NU = STATS ? TR_NV : 4;
  double w[NU];
#pragma unroll
  for (int i = 0; i < NU; i++) w[i] = S.acc[tr_slot<STATS>(i) * NT + tid];
#pragma unroll
  for (int i = 0; i < NU; i++) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) w[i] += __shfl_xor_sync(0xffffffffu, w[i], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NU; i++) S.red[warp * TR_NV + tr_slot<STATS>(i)] = w[i];
  }
  __syncthreads();
  if (tid < NU) {  // value k: warp totals in warp order, one thread per value
    const int k = tr_slot<STATS>(tid);
    double acc = S.red[k];
    for (int q = 1; q < NW; q++) acc += S.red[q * TR_NV + k];
    reinterpret_cast<double *>(A.parts + blockIdx.x)[k] = acc;  // TilePart = TR_NV doubles in w order
  }
  __syncthreads();
  if (tid == 0) {
    // acquire-release count: this CTA's partials (ordered by the barrier)
    // are released; the last CTA acquires everyone's
    unsigned done;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(done) : "l"(&A.ctrl->tiles_done) : "memory");
    S.last = (done == (unsigned)gridDim.x - 1);
    if (A.dbg && S.last) A.dbg[(size_t)blockIdx.x * 8 + 5] = gtimer();  // last CTA: count done
  }
  __syncthreads();
  if (S.last) metropolis_n<NT, STATS>(A, S.v, gridDim.x);
}

struct TrajVariant {
  int R, NT, MINB;
};
static const TrajVariant kVariants[] = {{8, 256, 2}, {4, 256, 3}, {4, 128, 6}, {8, 128, 4}, {16, 128, 2},
                                        {2, 256, 4}, {8, 64, 8}, {4, 256, 2}, {8, 32, 16},
                                        // persistent + TMA-staged (9..14); 12..14 are the
                                        // small-window shapes for short series
                                        {8, 256, 2}, {4, 256, 3}, {4, 256, 2}, {4, 128, 3}, {4, 64, 5},
                                        {4, 32, 8}, {8, 256, 1}, {6, 256, 1}, {4, 512, 1}};
static bool variant_persistent(int v) { return v >= 9; }
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

int traj_num_variants() { return kNumVariants; }

static TrajGeom traj_geometry_v(int64_t T, int n_steps, int sm_count, int variant) {
  TrajGeom g;
  if (variant < 0 || variant >= kNumVariants) variant = 0;
  const TrajVariant v = kVariants[variant];
  const int64_t NWv = v.NT / 32;
  const int64_t W = NWv > 1 ? NWv * 30 * v.R + 2 * v.R : (int64_t)v.R * 32;  // CTA window (ghost lanes overlap)
  g.variant = variant;
  g.halo = (n_steps + 1 + v.R - 1) / v.R * v.R;
  const int64_t core_max = (W - 2 * (int64_t)g.halo) / v.R * v.R;
  g.ok = core_max >= W / 4;
  if (!g.ok) { g.core = 0; g.n_tiles = 0; return g; }
  int64_t n = (T + core_max - 1) / core_max;
  const int64_t slots = (int64_t)v.MINB * sm_count;
  if (n > slots / 2) n = (n + slots - 1) / slots * slots;
  g.core = ((T + n - 1) / n + v.R - 1) / v.R * v.R;
  g.n_tiles = (int)((T + g.core - 1) / g.core);
  g.grid = variant_persistent(variant) ? (int)((int64_t)g.n_tiles < slots ? (int64_t)g.n_tiles : slots) : g.n_tiles;
  return g;
}

// variant < 0: automatic shape.  Long series use the 256-thread persistent
// kernel (11); when that leaves SMs idle, the CTA window shrinks (128 / 64 /
// 32 threads) so a short series still spreads over the whole GPU -- at small
// T the trajectory is latency-bound per step, and more, smaller tiles
// shorten it even though the halo share grows.
TrajGeom traj_geometry(int64_t T, int n_steps, int sm_count, int variant) {
  if (variant >= 0) return traj_geometry_v(T, n_steps, sm_count, variant);
  static const int kAuto[] = {11, 12, 13, 14};
  TrajGeom best{};
  bool have = false;
  for (int v : kAuto) {
    const TrajGeom g = traj_geometry_v(T, n_steps, sm_count, v);
    if (!g.ok) continue;
    best = g;
    have = true;
    if (g.n_tiles >= sm_count) break;
  }
  return have ? best : traj_geometry_v(T, n_steps, sm_count, 11);
}

template <int R, int NT, int MINB>
static void launch_v(const TrajArgs &a, cudaStream_t s) {
  if (a.fuse) traj_kernel<R, NT, MINB, true><<<a.g.n_tiles, NT, 0, s>>>(a);
  else traj_kernel<R, NT, MINB, false><<<a.g.n_tiles, NT, 0, s>>>(a);
}

template <int R, int NT, int MINB, bool FUSE, bool STATS, bool ENS = false, bool DEVK = false>
static void launch_p2(const TrajArgs &a, cudaStream_t s) {
  const size_t smem = sizeof(PersistSmem<R, NT>);
  cudaFuncSetAttribute(traj_persistent_kernel<R, NT, MINB, FUSE, STATS, ENS, DEVK>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // same (maximal) shared-memory carveout as the momenta kernel: no L1/shared
  // reconfiguration of the SMs between the two kernels of a proposal
  cudaFuncSetAttribute(traj_persistent_kernel<R, NT, MINB, FUSE, STATS, ENS, DEVK>,
                       cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (a.pdl) {  // overlap this launch with the tail of the momenta kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.g.grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, traj_persistent_kernel<R, NT, MINB, FUSE, STATS, ENS, DEVK>, a);
  } else {
    traj_persistent_kernel<R, NT, MINB, FUSE, STATS, ENS, DEVK><<<a.g.grid, NT, smem, s>>>(a);
  }
}

// run_chain on the device: the statistics variant with device-resident
// theta constants (persistent shapes of the automatic geometry only)
template <int R, int NT, int MINB>
static void launch_pd(const TrajArgs &a, cudaStream_t s) {
  if (a.fuse) launch_p2<R, NT, MINB, true, true, false, true>(a, s);
  else launch_p2<R, NT, MINB, false, true, false, true>(a, s);
}
static bool launch_devk(const TrajArgs &a, cudaStream_t s) {
  switch (a.g.variant) {
    case 11: launch_pd<4, 256, 2>(a, s); return true;
    case 12: launch_pd<4, 128, 3>(a, s); return true;
    case 13: launch_pd<4, 64, 5>(a, s); return true;
    case 14: launch_pd<4, 32, 8>(a, s); return true;
    default: return false;
  }
}
const void *traj_kernel_fn_devk(int variant, int fuse) {
#define RSV_FN(R, NT, MB)                                                                  \
  (fuse ? (const void *)traj_persistent_kernel<R, NT, MB, true, true, false, true>        \
        : (const void *)traj_persistent_kernel<R, NT, MB, false, true, false, true>)
  switch (variant) {
    case 11: return RSV_FN(4, 256, 2);
    case 12: return RSV_FN(4, 128, 3);
    case 13: return RSV_FN(4, 64, 5);
    case 14: return RSV_FN(4, 32, 8);
    default: return nullptr;
  }
#undef RSV_FN
}
template <int R, int NT, int MINB>
static void launch_p(const TrajArgs &a, cudaStream_t s) {
  if (a.fuse) {
    if (a.stats) launch_p2<R, NT, MINB, true, true>(a, s);
    else launch_p2<R, NT, MINB, true, false>(a, s);
  } else {
    if (a.stats) launch_p2<R, NT, MINB, false, true>(a, s);
    else launch_p2<R, NT, MINB, false, false>(a, s);
  }
}

const void *traj_kernel_fn(int variant, int fuse, int stats) {
#define RSV_FN(R, NT, MB) (fuse ? (const void *)traj_kernel<R, NT, MB, true> : (const void *)traj_kernel<R, NT, MB, false>)
  switch (variant) {
    case 0: return RSV_FN(8, 256, 2);
    case 1: return RSV_FN(4, 256, 3);
    case 2: return RSV_FN(4, 128, 6);
    case 3: return RSV_FN(8, 128, 4);
    case 4: return RSV_FN(16, 128, 2);
    case 5: return RSV_FN(2, 256, 4);
    case 6: return RSV_FN(8, 64, 8);
    case 7: return RSV_FN(4, 256, 2);
    case 8: return RSV_FN(8, 32, 16);
#undef RSV_FN
#define RSV_FN(R, NT, MB)                                                                                   \
  (fuse ? (stats ? (const void *)traj_persistent_kernel<R, NT, MB, true, true>                             \
                 : (const void *)traj_persistent_kernel<R, NT, MB, true, false>)                           \
        : (stats ? (const void *)traj_persistent_kernel<R, NT, MB, false, true>                            \
                 : (const void *)traj_persistent_kernel<R, NT, MB, false, false>))
    case 9: return RSV_FN(8, 256, 2);
    case 10: return RSV_FN(4, 256, 3);
    case 12: return RSV_FN(4, 128, 3);
    case 13: return RSV_FN(4, 64, 5);
    case 14: return RSV_FN(4, 32, 8);
    case 15: return RSV_FN(8, 256, 1);
    case 16: return RSV_FN(6, 256, 1);
    case 17: return RSV_FN(4, 512, 1);
    default: return RSV_FN(4, 256, 2);
  }
#undef RSV_FN
}

// ensemble geometry: the 256-thread persistent shape with the tile core
// capped at the chain length (a core then touches at most two chains)
TrajGeom traj_geometry_ens(int64_t T, int64_t Tc, int n_steps, int sm_count) {
  TrajGeom g = traj_geometry_v(T, n_steps, sm_count, 11);
  if (!g.ok || g.core <= Tc) return g;
  g.core = Tc;
  g.n_tiles = (int)((T + g.core - 1) / g.core);
  const int slots = kVariants[11].MINB * sm_count;
  g.grid = g.n_tiles < slots ? g.n_tiles : slots;
  return g;
}

const void *traj_kernel_fn_ens(int fuse) {
  return fuse ? (const void *)traj_persistent_kernel<4, 256, 2, true, false, true>
              : (const void *)traj_persistent_kernel<4, 256, 2, false, false, true>;
}

__global__ void ens_decide_kernel(TrajArgs A);

int launch_trajectory(const TrajArgs &a, cudaStream_t s, int *launches) {
  if (a.kdev) {
    if (!launch_devk(a, s)) return -1;
    (*launches)++;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  if (a.Tc > 0) {
    if (a.fuse) launch_p2<4, 256, 2, true, false, true>(a, s);
    else launch_p2<4, 256, 2, false, false, true>(a, s);
    ens_decide_kernel<<<(a.n_chains + 127) / 128, 128, 0, s>>>(a);
    (*launches) += 2;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  switch (a.g.variant) {
    case 0: launch_v<8, 256, 2>(a, s); break;
    case 1: launch_v<4, 256, 3>(a, s); break;
    case 2: launch_v<4, 128, 6>(a, s); break;
    case 3: launch_v<8, 128, 4>(a, s); break;
    case 4: launch_v<16, 128, 2>(a, s); break;
    case 5: launch_v<2, 256, 4>(a, s); break;
    case 6: launch_v<8, 64, 8>(a, s); break;
    case 7: launch_v<4, 256, 2>(a, s); break;
    case 8: launch_v<8, 32, 16>(a, s); break;
    case 9: launch_p<8, 256, 2>(a, s); break;
    case 10: launch_p<4, 256, 3>(a, s); break;
    case 12: launch_p<4, 128, 3>(a, s); break;
    case 13: launch_p<4, 64, 5>(a, s); break;
    case 14: launch_p<4, 32, 8>(a, s); break;
    case 15: launch_p<8, 256, 1>(a, s); break;
    case 16: launch_p<6, 256, 1>(a, s); break;
    case 17: launch_p<4, 512, 1>(a, s); break;
    default: launch_p<4, 256, 2>(a, s); break;
  }
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------
// Metropolis (sampler.py:155-167) on the reduced tile partials.
template <int NT, bool STATS>
__device__ void metropolis_n(const TrajArgs &A, double *s_v, int n_parts) {
  constexpr int NW = NT / 32;
  constexpr int NU = STATS ? TR_NV : 4;  // reduced values (TilePart slots tr_slot<STATS>(i))
  double v[NU];
#pragma unroll
  for (int i = 0; i < NU; i++) v[i] = 0.0;
  // two parts per thread per round, loaded together (one memory latency;
  // the summation order is the plain loop's: part j, then j + NT, ...)
  for (int j = threadIdx.x; j < n_parts; j += 2 * NT) {
    const double *t0 = reinterpret_cast<const double *>(A.parts + j);
    const double *t1 = reinterpret_cast<const double *>(A.parts + j + NT);
    const bool second = j + NT < n_parts;
    double a0[NU], a1[NU];
#pragma unroll
    for (int i = 0; i < NU; i++) {
      a0[i] = t0[tr_slot<STATS>(i)];
      a1[i] = second ? t1[tr_slot<STATS>(i)] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < NU; i++) {
      v[i] += a0[i];
      if (second) v[i] += a1[i];
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NU; i++) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if (lane == 0)
    for (int i = 0; i < NU; i++) s_v[warp * TR_NV + tr_slot<STATS>(i)] = v[i];
  __syncthreads();
  // the warp totals of value k are added in warp order by thread k (in
  // parallel over k), then thread 0 reads the NV results (0 for the
  // statistics slots when they are not evaluated)
  if (threadIdx.x < TR_NV) {
    const int k = threadIdx.x;
    const bool used = STATS || k < 3 || k == 13;
    double acc = used ? s_v[k] : 0.0;
    for (int w = 1; w < NW; w++) acc += used ? s_v[w * TR_NV + k] : 0.0;
    s_v[NW * TR_NV + k] = acc;
  }
  __syncthreads();
  if (threadIdx.x) return;
  double tot[TR_NV];
  for (int k = 0; k < TR_NV; k++) tot[k] = s_v[NW * TR_NV + k];
  DevControl *C = A.ctrl;
  C->tiles_done = 0;  // re-arm for the next launch
  C->t_stamp[3] = gtimer();
  if (C->halt) return;  // rsv_run_chain stopped at an earlier sweep: stream, path and statistics untouched
  if (A.shard) {  // time-sharded chain: the host combines the shards' totals
    for (int k = 0; k < TR_NV; k++) C->shard_parts[k] = tot[k];
    return;
  }
  const double cst = A.kdev ? A.kdev->hconst : A.k.hconst;
  DevResult r;
  r.h_old = tot[1] + cst;
  r.h_new = tot[2] + cst;
  r.accept = 0;
  r.u = __longlong_as_double(0x7ff8000000000000LL);
  r.words_used = 0;
  const bool flagged = tot[13] > 0.0;
  if (A.integrate_only) {
    // a non-finite final state only arises from a kick the reference flags
    // (NaN / inf are absorbing under the leapfrog map, _kernels.py:50-51)
    r.diverged = flagged || !isfinite(tot[2]);
    r.delta_h = tot[0];
    C->res = r;
    return;
  }
  const uint64_t used = C->zig_used;
  bool drew = false;
  const double dh = tot[0];
  if (flagged || !isfinite(dh) || fabs(dh) > 1000.0) {
    r.diverged = 1;
    r.delta_h = __longlong_as_double(0x7ff0000000000000LL);
  } else {
    r.diverged = 0;
    r.delta_h = dh;
    r.u = u01(C->u_word);  // raw word at stream position pos0 + used (momenta kernel)
    drew = true;
    r.accept = (dh <= 0.0) || (r.u < exp(-dh));
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
  if (C->stream.kind == PRNG_PCG32) {
    uint64_t q = C->seq_next;
    if (drew) { q = q * PCG_MULT + C->stream.s[1]; q = q * PCG_MULT + C->stream.s[1]; }
    C->seq_state = q;
  } else if (C->stream.kind == PRNG_MINSTD) {
    uint64_t q = C->seq_next;
    if (drew) q = mod31(mod31(mod31(q * MINSTD_A) * MINSTD_A) * MINSTD_A);
    C->seq_state = q;
  }
  if (r.accept) C->cur ^= 1;
  const double *sm = r.accept ? tot + 8 : tot + 3;
  C->stats[0] = r.accept ? C->ends_new[0] : C->ends_old[0];
  C->stats[1] = r.accept ? C->ends_new[1] : C->ends_old[1];
  for (int k = 0; k < 5; k++) C->stats[2 + k] = sm[k];
  C->res = r;
}

// Metropolis step of every chain of an ensemble (sampler.py:155-167 per
// chain), one thread per chain: sum the chain's tile records in tile order,
// decide with the chain's own uniform, keep the matching stream state, flip
// its buffer.
__global__ void ens_decide_kernel(TrajArgs A) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) A.ctrl->t_stamp[3] = gtimer();
  if (c >= A.n_chains) return;
  const int64_t Tc = A.Tc, core = A.g.core;
  const int64_t s0 = (int64_t)c * Tc, s1 = s0 + Tc - 1;
  const int ta = (int)(s0 / core), tb = (int)(s1 / core);
  double dh = 0.0, fl = 0.0;
  for (int t = ta; t <= tb; t++) {
    const int slot = ((int64_t)t * core) / Tc == c ? 0 : 1;
    const EnsPart &q = A.ens_parts[2 * (size_t)t + slot];
    dh += q.dh;
    fl += q.flag;
  }
  EnsChain &e = A.ens[c];
  bool accept = false, drew = false;
  if (e.overflow) atomicOr(&A.ctrl->err, 4);  // a tail draw beyond the parse window (never in practice)
  if (fl > 0.0 || e.overflow || !isfinite(dh) || fabs(dh) > 1000.0) {
    e.last_dh = __longlong_as_double(0x7ff0000000000000LL);
    e.n_diverged++;
  } else {
    e.last_dh = dh;
    const double u = u01(e.u_word);
    drew = true;
    accept = (dh <= 0.0) || (u < exp(-dh));
  }
  const uint64_t *st = drew ? e.st_used1 : e.st_used;
  for (int k = 0; k < 4; k++) e.st[k] = st[k];
  e.last_accept = accept;
  if (accept) {
    e.n_accept++;
    A.ens_cur[c] ^= 1;
  }
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
  // consecutive steps as programmatic dependents (launch_elementary_step with
  // pdl): the next step's CTAs launch while this one runs and wait below for
  // its completion before reading h, p (no-ops for a plain launch)
  asm volatile("griddepcontrol.launch_dependents;");
  const RefScal s = ref_scal(*prm);
  const double c = __dmul_rn(0.5, dt);
  const int64_t i0 = ((int64_t)blockIdx.x * ES_NT + threadIdx.x) * ES_R;
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
                           cudaStream_t st, int *launches, int pdl) {
  const int64_t threads = (T + ES_R - 1) / ES_R;
  const unsigned nb = (unsigned)((threads + ES_NT - 1) / ES_NT);
  if (pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(ES_NT);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, estep_kernel, h, p, ho, po, a, lrv, prm, dt, T, flag) != cudaSuccess) return -1;
  } else {
    estep_kernel<<<nb, ES_NT, 0, st>>>(h, p, ho, po, a, lrv, prm, dt, T, flag);
  }
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
  if (mode == 2) {  // statistics shifted by the parameters held on the device
    c_mu = prm->mu;
    c_xi = prm->xi;
  }
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
  if (mode == 2) c_mu = prm->mu;
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
int launch_suff_stats_dev(const double *h, const double *lrv, int64_t T, const DevParams *prm, double *partials,
                          double *out, cudaStream_t s, int *launches) {
  const int nb = reduce_partials_count(T);
  reduce1_kernel<<<nb, RD_NT, 0, s>>>(h, nullptr, nullptr, lrv, prm, T, 0.0, 0.0, 2, partials);
  reduce2_kernel<<<1, RD_NT, 0, s>>>(partials, nb, h, prm, T, 0.0, 2, out);
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
