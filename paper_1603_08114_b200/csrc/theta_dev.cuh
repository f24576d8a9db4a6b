// theta_dev.cuh -- numpy's ziggurat tables and the theta draws of one Gibbs
// sweep (sampler.py:170-272, run_chain :339-344) as device code of the theta
// kernel (momenta.cu), callable by any one-thread consumer:
// numpy's normal / uniform / Marsaglia-Tsang gamma restated on the raw-word
// stream (ThetaGen), the five full conditionals from the 7 moments of the
// kept path, the storm guard and the sample store.
#pragma once
#include <math.h>
#include <stdint.h>

#include "prng.cuh"
#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

static __device__ const uint64_t g_ki[256] = RSV_KI_DOUBLE_INIT;
static __device__ const double g_wi[256] = RSV_WI_DOUBLE_INIT;
static __device__ const double g_fi[256] = RSV_FI_DOUBLE_INIT;

// glibc log1p as one out-of-line copy: the exponential-tail path of the
// ziggurat is rare, so its code is cold in the instruction cache (after an L2
// flush it comes from DRAM); one shared copy halves those fetches.
static __device__ __noinline__ double log1p_ool(double x) { return glibc_log1p(x); }
static __device__ __noinline__ double log_ool(double x) { return log(x); }
static __device__ __noinline__ double exp_ool(double x) { return exp(x); }

// Speculative draws of a sweep's theta chain (pcg32 / minstd): lane j holds
// the normal, the gamma(shape) draw and the raw word that start at word j
// after the position the proposal is predicted to leave the stream at (its
// uniform drawn).  Filled while the trajectory kernel finishes; used only if
// the generator state there is the predicted one, so the draws are the same
// numbers on the same words -- the chain only looks them up.
struct ThetaSpec {
  uint64_t state;  // predicted generator state at window word 0
  double shape;
  double nval, gval;
  int nlen, glen;
  uint64_t word;
};

struct ThetaGen {
  int kind;
  SeqGen g;
  uint64_t s[4];
  uint64_t used;
  const uint64_t *ki;  // ziggurat tables (shared-memory copies)
  const double *wi, *fi;
  bool spec;             // draws served from *sp while `used` stays inside its window
  const ThetaSpec *sp;
  uint64_t seq0, inc;    // pcg32 / minstd: state at word 0 (for leaving the window)
  __device__ __noinline__ void unspec() {  // the sequential generator at word `used`
    spec = false;
    g.a = kind == PRNG_PCG32 ? pcg_advance(seq0, 2 * used, inc) : mod31(minstd_pow(3 * used) * seq0);
    g.b = inc;
  }
  __device__ __noinline__ uint64_t next() {
    if (spec) unspec();
    used++;
    return kind == PRNG_SFC64 ? sfc64_next(s) : g.next();
  }
  __device__ double next_double() {
    if (spec && used < 32) {
      const uint64_t w = __shfl_sync(0xffffffffu, sp->word, (int)used);
      used++;
      return u01(w);
    }
    return u01(next());
  }
  __device__ __noinline__ double normal() {  // numpy random_standard_normal
    if (spec && used < 32) {
      const int len = __shfl_sync(0xffffffffu, sp->nlen, (int)used);
      const double v = __shfl_sync(0xffffffffu, sp->nval, (int)used);
      used += (uint64_t)len;
      return v;
    }
    for (;;) {
      uint64_t r = next();
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const int sign = (int)(r & 0x1);
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = __dmul_rn((double)rabs, wi[idx]);
      if (sign) x = -x;
      if (rabs < ki[idx]) return x;
      if (idx == 0) {
        for (;;) {
          const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R, log1p_ool(-next_double()));
          const double yy = -log1p_ool(-next_double());
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
            return ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xx) : __dadd_rn(RSV_ZIG_R, xx);
        }
      }
      const double u = next_double();
      if (__dadd_rn(__dmul_rn(__dsub_rn(fi[idx - 1], fi[idx]), u), fi[idx]) <
          exp_ool(__dmul_rn(__dmul_rn(-0.5, x), x)))
        return x;
    }
  }
  __device__ __noinline__ double gamma(double shape) {  // numpy random_standard_gamma, shape > 1
    if (spec && used < 32 && shape == sp->shape) {
      const int len = __shfl_sync(0xffffffffu, sp->glen, (int)used);
      const double v = __shfl_sync(0xffffffffu, sp->gval, (int)used);
      used += (uint64_t)len;
      return v;
    }
    const double b = __dsub_rn(shape, 1.0 / 3.0);
    const double c = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(9.0, b)));
    for (;;) {
      double X, V;
      do {
        X = normal();
        V = __dadd_rn(1.0, __dmul_rn(c, X));
      } while (V <= 0.0);
      V = __dmul_rn(__dmul_rn(V, V), V);
      const double U = next_double();
      const double X2 = __dmul_rn(X, X);
      if (U < __dsub_rn(1.0, __dmul_rn(__dmul_rn(0.0331, X2), X2))) return __dmul_rn(b, V);
      if (log_ool(U) < __dadd_rn(__dmul_rn(0.5, X2), __dmul_rn(b, __dadd_rn(__dsub_rn(1.0, V), log_ool(V)))))
        return __dmul_rn(b, V);
    }
  }
};

// Every lane: the draws that would start at word `lane` after `state`
// (computed with the same functions the chain uses, so the same bits).
static __device__ __noinline__ void theta_spec_fill(ThetaSpec &sp, int kind, uint64_t state, uint64_t inc,
                                                    double shape, const uint64_t *ki, const double *wi,
                                                    const double *fi) {
  const uint64_t lane = threadIdx.x & 31;
  sp.state = state;
  sp.shape = shape;
  const uint64_t st_l =
      kind == PRNG_PCG32 ? pcg_advance(state, 2 * lane, inc) : mod31(minstd_pow(3 * lane) * state);
  ThetaGen g;
  g.kind = kind;
  g.ki = ki;
  g.wi = wi;
  g.fi = fi;
  g.spec = false;
  g.sp = nullptr;
  g.seq0 = st_l;
  g.inc = inc;
  g.g.kind = kind;
  g.g.k = 0;
  g.g.a = st_l;
  g.g.b = inc;
  SeqGen w = g.g;
  sp.word = w.next();
  g.used = 0;
  sp.nval = g.normal();
  sp.nlen = (int)g.used;
  g.g.a = st_l;
  g.used = 0;
  sp.gval = g.gamma(shape);
  sp.glen = (int)g.used;
}

// _recentre (sampler.py mirror): moments of d' = h - mu from d = h - c
struct Recentred {
  double d0n, sxx, sall, sxz;
};
static __device__ Recentred recentre(const double *st, double Td, double c, double mu) {
  const double delta = __dsub_rn(mu, c);
  const double d0 = st[0], dl = st[1], s1 = st[2], s2 = st[3], sx = st[4];
  const double Tm1 = Td - 1.0;
  Recentred r;
  r.d0n = __dsub_rn(d0, delta);
  r.sxx = __dadd_rn(__dsub_rn(__dsub_rn(s2, __dmul_rn(dl, dl)), __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(s1, dl))),
                    __dmul_rn(__dmul_rn(Tm1, delta), delta));
  r.sall = __dadd_rn(__dsub_rn(s2, __dmul_rn(__dmul_rn(2.0, delta), s1)), __dmul_rn(__dmul_rn(Td, delta), delta));
  r.sxz = __dadd_rn(__dsub_rn(sx, __dmul_rn(delta, __dadd_rn(__dsub_rn(s1, d0), __dsub_rn(s1, dl)))),
                    __dmul_rn(__dmul_rn(Tm1, delta), delta));
  return r;
}

// The theta body runs on all 32 lanes of one warp with identical values (the
// same sequential draws in every lane); where it needs several independent
// logarithms, each lane evaluates one and the results are gathered by
// shuffles -- one glibc log1p latency instead of six on the chain of the phi
// update.  (Spreading the quotients of the mu / xi updates the same way was
// measured slower: the divisions already overlap within one thread.)
__device__ __forceinline__ double lane_pick(double v, int k) { return __shfl_sync(0xffffffffu, v, k); }

static __device__ double phi_log_ratio(double prop, double phi, double h1_sq, double se2, const DevPrior &pr) {
  const int lane = threadIdx.x & 31;
  const double pp = __dmul_rn(prop, prop), ff = __dmul_rn(phi, phi);
  const double arg = lane == 0 ? -pp : lane == 1 ? -ff : lane == 2 ? prop : lane == 3 ? phi : lane == 4 ? -prop : -phi;
  const double lg = log1p_ool(arg);
  const double a = __dmul_rn(0.5, __dsub_rn(lane_pick(lg, 0), lane_pick(lg, 1)));
  const double b = __ddiv_rn(__dmul_rn(h1_sq, __dsub_rn(__dsub_rn(1.0, pp), __dsub_rn(1.0, ff))), __dmul_rn(2.0, se2));
  const double c = __dmul_rn(__dsub_rn(pr.phi_a, 1.0), __dsub_rn(lane_pick(lg, 2), lane_pick(lg, 3)));
  const double d = __dmul_rn(__dsub_rn(pr.phi_b, 1.0), __dsub_rn(lane_pick(lg, 4), lane_pick(lg, 5)));
  return __dadd_rn(__dadd_rn(__dsub_rn(a, b), c), d);
}


// One sweep's theta draws, run by one thread after the proposal (C->res,
// C->stats hold its result and the kept path's statistics): storm guard,
// mu, phi, sigma_eta^2, xi, sigma_u^2 in the reference's order on the same
// raw words, new DevParams / TrajConsts, and the sample store.  ki / wi / fi:
// the ziggurat tables (shared-memory copies).
static __device__ __noinline__ void theta_sweep_body(DevControl *C, DevParams *P, TrajConsts *K, DevRun *R,
                                                     const DevPrior &pr, double dt, int64_t T, const uint64_t *ki,
                                                     const double *wi, const double *fi, const ThetaSpec *sp) {
  // every input in one round of independent loads (one thread: each load
  // issued on its own would cost a full memory latency on the critical path)
  const int halt = C->halt;
  const DevResult res = C->res;
  const StreamState ss = C->stream;
  const uint64_t seq0 = C->seq_state;
  double st[7];
#pragma unroll
  for (int k = 0; k < 7; k++) st[k] = C->stats[k];
  const DevParams P0 = *P;
  const int32_t ring_n = R->ring_n, ring_pos = R->ring_pos, ring_div0 = R->ring_div;
  const int64_t storm0 = R->storm_sweep, sweep0 = R->sweep;
  const int64_t n_burnin = R->n_burnin, thin = R->thin, n_store = R->n_store, stored0 = R->stored;
  double *const r_params = R->params, *const r_dh = R->delta_h;
  int32_t *const r_acc = R->accept;
  int64_t *const r_it = R->iters;
  const uint8_t ring_old = R->ring[ring_pos];
  if (halt) return;  // the run stopped at an earlier sweep
  // storm guard (sampler.py:329-337), checked on the proposal just made; the
  // reference raises before any theta draw, so the run stops right here
  {
    const int div = res.diverged ? 1 : 0;
    int rn = ring_n, rd = ring_div0;
    if (rn == RUN_STORM_WINDOW) rd -= ring_old;
    else rn++;
    rd += div;
    R->ring[ring_pos] = (uint8_t)div;
    R->ring_n = rn;
    R->ring_div = rd;
    R->ring_pos = (ring_pos + 1) % RUN_STORM_WINDOW;
    if (rn == RUN_STORM_WINDOW && rd > RUN_STORM_LIMIT && storm0 < 0) {
      R->storm_sweep = sweep0;
      C->halt = 1;
      return;
    }
  }
  ThetaGen G;
  G.kind = ss.kind;
  G.used = 0;
  G.ki = ki;
  G.wi = wi;
  G.fi = fi;
  G.spec = false;
  G.sp = sp;
  G.seq0 = seq0;
  G.inc = ss.s[1];
  if (G.kind == PRNG_SFC64) {
    for (int k = 0; k < 4; k++) G.s[k] = ss.s[k];
  } else if (G.kind == PRNG_PHILOX) {
    G.g.init(ss, ss.pos);
  } else {  // pcg32 / minstd: the sequential state at the position is kept by the Metropolis step
    G.g.kind = G.kind;
    G.g.k = ss.pos;
    G.g.a = seq0;
    G.g.b = ss.s[1];
    G.spec = sp != nullptr && sp->state == seq0;  // the position the speculation assumed
  }
  const double Td = (double)T, Tm1 = Td - 1.0;
  double phi = P0.phi, mu = P0.mu, xi = P0.xi, se2 = P0.se2, su2 = P0.su2;
  const double c_mu = mu, c_xi = xi;
  bool degenerate = false;
  // update_mu (sampler.py:170-188)
  {
    const double omp = __dsub_rn(1.0, phi);
    const double prec = __dadd_rn(
        __ddiv_rn(__dadd_rn(__dsub_rn(1.0, __dmul_rn(phi, phi)), __dmul_rn(Tm1, __dmul_rn(omp, omp))), se2),
        __ddiv_rn(1.0, pr.mu_var));
    const double d0 = st[0], dl = st[1], s1 = st[2];
    const double h0 = __dadd_rn(d0, c_mu);
    const double trans = __dadd_rn(__dsub_rn(__dsub_rn(s1, d0), __dmul_rn(phi, __dsub_rn(s1, dl))),
                                   __dmul_rn(__dmul_rn(Tm1, omp), c_mu));
    const double num = __dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(__dsub_rn(1.0, __dmul_rn(phi, phi)), h0), se2),
                                           __ddiv_rn(__dmul_rn(omp, trans), se2)),
                                 __ddiv_rn(pr.mu_mean, pr.mu_var));
    if (!(isfinite(prec) && prec > 0.0)) {
      degenerate = true;
    } else {
      const double sd = __dsqrt_rn(__ddiv_rn(1.0, prec));
      mu = __dadd_rn(__ddiv_rn(num, prec), __dmul_rn(sd, G.normal()));
    }
  }
  // update_phi (sampler.py:249-272)
  if (!degenerate) {
    const Recentred r = recentre(st, Td, c_mu, mu);
    const double sxx = r.sxx > 1e-300 ? r.sxx : 1e-300;
    const double phi_hat = __ddiv_rn(r.sxz, sxx);
    const double sd = __dsqrt_rn(__ddiv_rn(se2, sxx));
    const double prop = __dadd_rn(phi_hat, __dmul_rn(sd, G.normal()));
    if (-1.0 < prop && prop < 1.0) {
      const double lr = phi_log_ratio(prop, phi, __dmul_rn(r.d0n, r.d0n), se2, pr);
      const double u = G.next_double();
      if (lr >= 0.0 || u < exp_ool(lr)) phi = prop;
    }
  }
  // update_sigma_eta_sq (sampler.py:218-230)
  if (!degenerate) {
    const Recentred r = recentre(st, Td, c_mu, mu);
    const double tail_sq = __dsub_rn(r.sall, __dmul_rn(r.d0n, r.d0n));
    const double q = __dadd_rn(
        __dmul_rn(__dmul_rn(__dsub_rn(1.0, __dmul_rn(phi, phi)), r.d0n), r.d0n),
        __dadd_rn(__dsub_rn(tail_sq, __dmul_rn(__dmul_rn(2.0, phi), r.sxz)), __dmul_rn(__dmul_rn(phi, phi), r.sxx)));
    const double shape = __dadd_rn(pr.var_shape, __dmul_rn(0.5, Td));
    const double scale = __dadd_rn(pr.var_scale, __dmul_rn(0.5, q));
    se2 = __ddiv_rn(scale, G.gamma(shape));
  }
  // update_xi (sampler.py:191-202)
  if (!degenerate) {
    const double sum_r = __dadd_rn(st[5], __dmul_rn(Td, c_xi));
    const double prec = __dadd_rn(__ddiv_rn(Td, su2), __ddiv_rn(1.0, pr.xi_var));
    const double num = __dadd_rn(__ddiv_rn(sum_r, su2), __ddiv_rn(pr.xi_mean, pr.xi_var));
    if (!(isfinite(prec) && prec > 0.0)) {
      degenerate = true;
    } else {
      const double sd = __dsqrt_rn(__ddiv_rn(1.0, prec));
      xi = __dadd_rn(__ddiv_rn(num, prec), __dmul_rn(sd, G.normal()));
    }
  }
  // update_sigma_u_sq (sampler.py:209-215)
  if (!degenerate) {
    const double delta = __dsub_rn(xi, c_xi);
    const double ss = __dadd_rn(__dsub_rn(st[6], __dmul_rn(__dmul_rn(2.0, delta), st[5])),
                                __dmul_rn(__dmul_rn(Td, delta), delta));
    const double shape = __dadd_rn(pr.var_shape, __dmul_rn(0.5, Td));
    const double scale = __dadd_rn(pr.var_scale, __dmul_rn(0.5, ss));
    su2 = __ddiv_rn(scale, G.gamma(shape));
  }
  // the stream continues after the draws (those made before a degenerate
  // precision included: the reference raises after them, sampler.py:186,200)
  if (G.spec) G.unspec();  // the generator state after the last draw
  C->stream.pos = ss.pos + G.used;
  if (G.kind == PRNG_SFC64)
    for (int k = 0; k < 4; k++) C->stream.s[k] = G.s[k];
  else if (G.kind == PRNG_PCG32 || G.kind == PRNG_MINSTD)
    C->seq_state = G.g.a;
  if (degenerate) {  // ValueError in the reference: parameters unchanged, nothing stored
    R->degenerate = 1;
    C->halt = 1;
    return;
  }
  // new parameters and the constants derived from them (rsv_set_params)
  DevParams q = P0;
  q.phi = phi; q.mu = mu; q.xi = xi; q.se2 = se2; q.su2 = su2;
  q.inv_su2 = 1.0 / su2;
  q.inv_se2 = 1.0 / se2;
  q.one_m_phi2 = 1.0 - phi * phi;
  {
    const int lane = threadIdx.x & 31;
    const double lg = log_ool(lane == 0 ? su2 : lane == 1 ? se2 / (1.0 - phi * phi) : se2);
    const double l_su2 = lane_pick(lg, 0), l_st = lane_pick(lg, 1), l_se2 = lane_pick(lg, 2);
    q.emu = exp_ool(-mu);
    q.hconst = 0.5 * Td * mu + 0.5 * Td * l_su2 + 0.5 * l_st + 0.5 * Tm1 * l_se2;
  }
  q.n_lo = (int32_t)floor((mu - 50.0) * RSV_INV_LN2_N);
  q.n_span = (int32_t)ceil((mu + 50.0) * RSV_INV_LN2_N) - q.n_lo;
  *P = q;
  *K = traj_consts(q, dt);
  // store (sampler.py:346-354)
  const int64_t sw = sweep0;
  if (sw >= n_burnin && (sw - n_burnin) % thin == 0 && stored0 < n_store) {
    const int64_t i = stored0;
    R->stored = stored0 + 1;
    double *o = r_params + 5 * i;
    o[0] = phi; o[1] = mu; o[2] = xi; o[3] = se2; o[4] = su2;
    r_acc[i] = res.accept;
    r_dh[i] = res.diverged ? __longlong_as_double(0x7ff0000000000000LL) : res.delta_h;
    r_it[i] = sw;
  }
  R->sweep = sw + 1;
}

}  // namespace rsv
