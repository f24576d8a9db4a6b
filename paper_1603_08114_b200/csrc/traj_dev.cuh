// traj_dev.cuh -- the per-site leapfrog arithmetic of the trajectory kernels
// (leapfrog.cu): e^{-d} on d and on the scaled state, the kick and the
// drifts, the per-site potential energy and the thread-group sums, and the
// 128-bit fixed-point helpers.  Any kernel that forms a site's update or a
// group's energies with these functions gets the tiled kernel's bits (the
// energies use explicit round-to-nearest intrinsics: no context-dependent
// FMA contraction).
#pragma once
#include <math.h>
#include <stdint.h>

#include "exp_table.h"
#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

static __device__ __align__(128) const unsigned long long g_exp_tab2[RSV_EXP_TAB_N] = RSV_EXP_TAB2_INIT;

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

// e^{-d} of the step loop, on the scaled state x = K d (K = 2048 / ln 2,
// DESIGN.md 4.2): n = rint(-x) by the magic-number add, f = -x - n exactly
// (|f| <= 1/2, no Cody-Waite split), e^{f ln2/2048} - 1 by a degree-3 Horner
// polynomial in f, and S = 2^(n/2048) from the scale-ready table as above.
// 7 FP64 instructions (3 DADD, 3 DFMA / DMUL, 1 DFMA), constants from the
// kernel's parameter block (constant-bank operands).
template <typename K>
__device__ __forceinline__ double exp_neg_x(double x, const unsigned long long *tab, double &t, const K &k) {
  t = MAGIC - x;
  const double nd = t - MAGIC;
  const double f = -x - nd;
  double q = fma(f, k.ex3, k.ex2);
  q = fma(q, f, k.ex1);
  q = q * f;
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


// Variable potential part of H at one site (the theta-only constants are
// added in the Metropolis step): 0.5 d + a e^{-mu} e^{-d} + (q-d)^2/2su2 + AR.
// Every operation is an explicit round-to-nearest intrinsic: the compiler's
// FMA contraction would otherwise depend on the surrounding code, and every
// kernel variant (shapes, statistics, shards) must form the same per-group
// energies bit for bit (their fixed-point sums are compared exactly).
__device__ __forceinline__ double site_potential(double d, double dprev, double ae, double q, bool first,
                                                 const TrajConsts &s, const unsigned long long *tab) {
  double t;
  const double E = exp_neg(d, tab, t);
  const double r = __dsub_rn(q, d);
  const double tr = __fma_rn(-s.phi, dprev, d);
  const double ar = first ? __dmul_rn(__dmul_rn(__dmul_rn(s.one_m_phi2, d), d), s.inv2se)
                          : __dmul_rn(__dmul_rn(tr, tr), s.inv2se);
  double en = __fma_rn(ae, E, __dmul_rn(0.5, d));
  en = __fma_rn(__dmul_rn(r, r), s.inv2su, en);
  return __dadd_rn(en, ar);
}

// Potential energy and statistics of the thread's owned core sites, summed
// in site order (branch-free on the common path).  firstm bit r: site r is
// the first of its series (stationary AR prior, no predecessor term).  The
// kinetic part is added by the caller (kinetic()), in the same order for
// every tile, so a group's H is the same value whatever tile it falls in.
template <int R, bool STATS = true>
__device__ __forceinline__ void tile_energy(const double (&d)[R], const double (&av)[R], const double (&lv)[R],
                                            double dl, uint32_t core, uint32_t firstm, const TrajConsts &s,
                                            const unsigned long long *tab, double (&v)[6]) {
#pragma unroll
  for (int r = 0; r < R; r++) {
    const double dprev = r ? d[r - 1] : dl;
    const double q = __dsub_rn(lv[r], s.xm);
    const bool first = (firstm >> r) & 1;
    const double en = site_potential(d[r], dprev, __dmul_rn(s.emu, av[r]), q, first, s, tab);
    const bool c = (core >> r) & 1;
    v[0] = __dadd_rn(v[0], c ? en : 0.0);
    if (STATS) {
      const double e = __dsub_rn(q, d[r]);
      v[1] = __dadd_rn(v[1], c ? d[r] : 0.0);
      v[2] = __dadd_rn(v[2], c ? __dmul_rn(d[r], d[r]) : 0.0);
      v[3] = __dadd_rn(v[3], (c && !first) ? __dmul_rn(d[r], dprev) : 0.0);
      v[4] = __dadd_rn(v[4], c ? e : 0.0);
      v[5] = __dadd_rn(v[5], c ? __dmul_rn(e, e) : 0.0);
    }
  }
}
template <int R>
__device__ __forceinline__ double kinetic(const double (&p)[R], uint32_t core) {
  double k = 0.0;
#pragma unroll
  for (int r = 0; r < R; r++) k = __dadd_rn(k, ((core >> r) & 1) ? __dmul_rn(__dmul_rn(0.5, p[r]), p[r]) : 0.0);
  return k;
}

// Round-toward-zero of v * 2^64 as a 128-bit integer (exact for the 53-bit
// significand down to 2^-64; the caller keeps |v| < 2^62).  Integer sums of
// these are associative: the reductions of dH, H_old and H_new give the same
// bits for any grouping of the partials.
__device__ __forceinline__ __int128 fix128(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const int ex = (int)((b >> 52) & 0x7ff);
  const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | (ex ? 0x10000000000000ull : 0ull);
  const int sh = ex - 1075 + 64;  // v * 2^64 = m * 2^sh
  __int128 r;
  if (sh >= 0) r = (__int128)m << (sh < 74 ? sh : 74);
  else r = (__int128)(sh > -64 ? m >> (-sh) : 0ull);
  return (b >> 63) ? -r : r;
}
__device__ __forceinline__ double unfix128(__int128 q) {  // nearest double of q * 2^-64
  const bool neg = q < 0;
  const unsigned __int128 a = neg ? (unsigned __int128)(-q) : (unsigned __int128)q;
  const unsigned long long hi = (unsigned long long)(a >> 64), lo = (unsigned long long)a;
  // hi + lo 2^-64, both exact in two doubles up to rounding of the sum
  const double r = __ull2double_rn(hi) + __ull2double_rn(lo) * 0x1p-64;
  return neg ? -r : r;
}
__device__ __forceinline__ __int128 shfl_xor_128(__int128 v, int o) {
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
  return (__int128)(((unsigned __int128)h2 << 64) | l2);
}
__device__ __forceinline__ __int128 ld128(const long long (&w)[2]) {
  return (__int128)(((unsigned __int128)(unsigned long long)w[1] << 64) | (unsigned long long)w[0]);
}
__device__ __forceinline__ void st128(long long (&w)[2], __int128 v) {
  w[0] = (long long)(unsigned long long)v;
  w[1] = (long long)(v >> 64);
}
// 128-bit sums through 64-bit atomics: q = L0 + L1 2^42 + L2 2^84 with
// L0, L1 in [0, 2^42) and L2 signed; sums of up to 2^22 such limbs fit a
// 64-bit word, and the total is rebuilt exactly (mod 2^128)
__device__ __forceinline__ void fx_add(unsigned long long *fx, __int128 q) {
  const unsigned __int128 u = (unsigned __int128)q;
  const unsigned long long l0 = (unsigned long long)u & ((1ull << 42) - 1);
  const unsigned long long l1 = (unsigned long long)(u >> 42) & ((1ull << 42) - 1);
  const unsigned long long l2 = (unsigned long long)(long long)(q >> 84);
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(fx + 0), "l"(l0) : "memory");
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(fx + 1), "l"(l1) : "memory");
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(fx + 2), "l"(l2) : "memory");
}
__device__ __forceinline__ __int128 fx_total(const unsigned long long *fx) {
  return (__int128)fx[0] + ((__int128)fx[1] << 42) + ((__int128)(long long)fx[2] << 84);
}

// energies beyond 2^62 per group (or non-finite) cannot be represented: they
// poison the sum to a non-finite dH, which the Metropolis step rejects
constexpr double FIX_MAX = 0x1p62;

// One kick p -= dt * dU/dh for the thread's R sites, on x = K (h - mu):
//   p <- p - Cd - (G/K) x + (beta phi/K) (x_{i-1} + x_{i+1}) + Ad e^{-x/K}
// (d-space form: p - Cd - G d + beta phi (d_{i-1} + d_{i+1}) + Ad e^{-d}).
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
    const double E = exp_neg_x(d[r], tab, t, s);
    // lean warps: each thread's sites are all core or none (the caller keeps
    // the thread's maximum only in the first case), so no per-site mask
    if (EDGE) nmax = max(nmax, ((unsigned)__double2loint(t) - (unsigned)s.n_lo) & cm[r]);
    else nmax = max(nmax, (unsigned)__double2loint(t) - (unsigned)s.n_lo);
    const double G = EDGE && ((endm >> r) & 1) ? s.xg_end : s.xg_int;
    double pp = p[r] - Cd[r];
    pp = fma(-G, d[r], pp);
    pp = fma(s.xbphi, dm + dp, pp);
    pp = fma(Ad[r], E, pp);
    p[r] = (EDGE && !((live >> r) & 1)) ? 0.0 : pp;
  }
}

template <int R>
__device__ __forceinline__ void drift(double (&d)[R], const double (&p)[R], double c) {
#pragma unroll
  for (int r = 0; r < R; r++) d[r] = fma(c, p[r], d[r]);
}


}  // namespace rsv
