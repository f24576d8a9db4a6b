/*
 * rsv_oracle.c -- CPU restatement of the reference's HMC volatility path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1603_08114_b200/ links, loads or
 * calls this file; it is used by tests/ (as the parity checker),
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 *
 * Every function cites the reference line it restates (paths relative to
 * /root/reference).  Arithmetic is plain IEEE double compiled with
 * -ffp-contract=off so the leapfrog kernels evaluate in the same order and
 * with the same roundings as the numba kernels in pkg/src/rsvhmc/_kernels.py.
 *
 * Pinning: tests/golden/make_golden.py runs the reference itself (in the
 * build container, with the same bit generators plugged into numpy's
 * Generator) and commits its outputs; tests/test_oracle.py checks this file
 * against them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#include "zig_tables_oracle.h"

/* ------------------------------------------------------------------ */
/* Bit generators.  Stream state convention (shared with include/rsvhmc_b200.h):
 *   kind 0 philox : s[0..1] = key, pos = words drawn   (numpy Philox4x64-10)
 *   kind 1 minstd : s[0] = x0,      pos = words drawn  (std::minstd_rand, 3 draws / word)
 *   kind 2 pcg32  : s[0] = state0, s[1] = inc, pos    (pcg_basic, 2 draws / word)
 *   kind 3 sfc64  : s[0..3] = a,b,c,w current state    (numpy SFC64)
 */
typedef struct {
  int32_t kind;
  int32_t pad;
  uint64_t s[4];
  uint64_t pos;
  /* sequential-access cache (not part of the stream's identity): the LCG
   * state in front of word cache_pos, so consecutive draws cost O(1) */
  uint64_t cache_pos, cache_state;
  int32_t cache_ok, pad2;
} orc_stream;

static inline uint64_t mulhilo64(uint64_t a, uint64_t b, uint64_t *hi) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  return (uint64_t)p;
}

/* numpy/random/src/philox/philox.h: philox4x64_round / bumpkey, 10 rounds. */
static void philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    uint64_t hi0, hi1;
    uint64_t lo0 = mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0);
    uint64_t lo1 = mulhilo64(0xCA5A826395121157ULL, c2, &hi1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

#define MINSTD_M 2147483647ULL
#define MINSTD_A 48271ULL
static uint64_t powmod31(uint64_t a, uint64_t e) {
  uint64_t r = 1; a %= MINSTD_M;
  while (e) { if (e & 1) r = (r * a) % MINSTD_M; a = (a * a) % MINSTD_M; e >>= 1; }
  return r;
}
/* minstd output j (0-based): x_{j+1} = a^{j+1} x0 mod m (std::minstd_rand). */
static inline uint64_t minstd_out(uint64_t x0, uint64_t j) { return (powmod31(MINSTD_A, j + 1) * x0) % MINSTD_M; }

#define PCG_MULT 6364136223846793005ULL
/* pcg_basic pcg32_advance_r: O(log n) LCG jump. */
static uint64_t pcg_advance(uint64_t state, uint64_t delta, uint64_t mult, uint64_t plus) {
  uint64_t acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) { acc_mult *= mult; acc_plus = acc_plus * mult + plus; }
    plus = (mult + 1) * plus; mult *= mult; delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}
static inline uint32_t pcg_output(uint64_t old) {
  uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = (uint32_t)(old >> 59u);
  return (xs >> rot) | (xs << ((-rot) & 31));
}

static inline uint64_t sfc64_step(uint64_t *s) {
  uint64_t tmp = s[0] + s[1] + s[3]++;
  s[0] = s[1] ^ (s[1] >> 11);
  s[1] = s[2] + (s[2] << 3);
  s[2] = ((s[2] << 24) | (s[2] >> 40)) + tmp;
  return tmp;
}

/* Raw 64-bit word at the stream's current position; advances by one word. */
uint64_t orc_next_u64(orc_stream *st) {
  uint64_t n = st->pos++;
  switch (st->kind) {
    case 0: {
      uint64_t ctr[4] = {n / 4 + 1, 0, 0, 0}, out[4];
      philox4x64_10(ctr, st->s, out);
      return out[n % 4];
    }
    case 1: {
      /* x_{3n} then three steps */
      uint64_t x = (st->cache_ok && st->cache_pos == n) ? st->cache_state
                                                        : (powmod31(MINSTD_A, 3 * n) * st->s[0]) % MINSTD_M;
      uint64_t xa = (x * MINSTD_A) % MINSTD_M, xb = (xa * MINSTD_A) % MINSTD_M, xc = (xb * MINSTD_A) % MINSTD_M;
      st->cache_ok = 1; st->cache_pos = n + 1; st->cache_state = xc;
      return (xa << 33) | (xb << 2) | (xc >> 29);
    }
    case 2: {
      uint64_t s0 = (st->cache_ok && st->cache_pos == n) ? st->cache_state
                                                         : pcg_advance(st->s[0], 2 * n, PCG_MULT, st->s[1]);
      uint64_t s1 = s0 * PCG_MULT + st->s[1];
      st->cache_ok = 1; st->cache_pos = n + 1; st->cache_state = s1 * PCG_MULT + st->s[1];
      return ((uint64_t)pcg_output(s0) << 32) | pcg_output(s1);
    }
    default:
      return sfc64_step(st->s);
  }
}
/* numpy: (next_uint64 >> 11) * 2^-53 for every generator used here. */
double orc_next_double(orc_stream *st) { return (double)(orc_next_u64(st) >> 11) * (1.0 / 9007199254740992.0); }
uint32_t orc_next_u32(orc_stream *st) { return (uint32_t)(orc_next_u64(st) >> 32); }

/* seeding helpers (raw seed material is produced by numpy.SeedSequence in Python) */
void orc_stream_init(orc_stream *st, int kind, const uint64_t *seed) {
  memset(st, 0, sizeof(*st));
  st->kind = kind;
  switch (kind) {
    case 0: st->s[0] = seed[0]; st->s[1] = seed[1]; break;
    case 1: { uint64_t x = seed[0] % MINSTD_M; st->s[0] = x ? x : 1; break; }
    case 2: { /* pcg32_srandom_r(initstate=seed[0], initseq=seed[1]) */
      uint64_t inc = (seed[1] << 1u) | 1u, s = 0;
      s = s * PCG_MULT + inc; s += seed[0]; s = s * PCG_MULT + inc;
      st->s[0] = s; st->s[1] = inc; break; }
    default: /* numpy sfc64_set_seed: a,b,c from SeedSequence, w = 1, 12 discards */
      st->s[0] = seed[0]; st->s[1] = seed[1]; st->s[2] = seed[2]; st->s[3] = 1;
      for (int i = 0; i < 12; i++) sfc64_step(st->s);
      break;
  }
}
void orc_fill_u64(orc_stream *st, uint64_t *out, int64_t n) { for (int64_t i = 0; i < n; i++) out[i] = orc_next_u64(st); }

/* numpy-compatible bitgen_t so numpy's own Generator can drive the reference */
typedef struct { void *state; uint64_t (*next_uint64)(void *); uint32_t (*next_uint32)(void *);
                 double (*next_double)(void *); uint64_t (*next_raw)(void *); } orc_bitgen;
static uint64_t bg_u64(void *s) { return orc_next_u64((orc_stream *)s); }
static uint32_t bg_u32(void *s) { return orc_next_u32((orc_stream *)s); }
static double bg_dbl(void *s) { return orc_next_double((orc_stream *)s); }
void orc_bitgen_bind(orc_bitgen *bg, orc_stream *st) {
  bg->state = st; bg->next_uint64 = bg_u64; bg->next_uint32 = bg_u32; bg->next_double = bg_dbl; bg->next_raw = bg_u64;
}

/* ------------------------------------------------------------------ */
/* glibc 2.39 log1p as selected on FMA-capable x86-64 (the fdlibm algorithm
 * with Estrin evaluation, contracted exactly as the FMA ifunc variant is);
 * verified bit-identical to the system log1p by tests/test_oracle.py.
 * numpy's ziggurat tail draws call log1p(-u). */
static inline int32_t hiw(double x) { uint64_t u; memcpy(&u, &x, 8); return (int32_t)(u >> 32); }
static inline double sethiw(double x, int32_t h) { uint64_t u; memcpy(&u, &x, 8); u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)h << 32); memcpy(&x, &u, 8); return x; }
double orc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double hfsq, f = 0, c = 0, s, z, R, u;
  int32_t k, hx, hu = 0, ax;
  hx = hiw(x); ax = hx & 0x7fffffff; k = 1;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) { if (x == -1.0) return -INFINITY; return NAN; }
    if (ax < 0x3e200000) { if (ax < 0x3c900000) return x; return fma(-(x * x), 0.5, x); }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) { k = 0; f = x; hu = 1; }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) { u = 1.0 + x; hu = hiw(u); k = (hu >> 20) - 1023; c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0); c /= u; }
    else { u = x; hu = hiw(u); k = (hu >> 20) - 1023; c = 0; }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) u = sethiw(u, hu | 0x3ff00000);
    else { k += 1; u = sethiw(u, hu | 0x3fe00000); hu = (0x00100000 - hu) >> 2; }
    f = u - 1.0;
  }
  hfsq = (f * 0.5) * f;
  double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) { if (k == 0) return 0.0; c = fma(dk, ln2_lo, c); return fma(dk, ln2_hi, c); }
    R = fma(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  s = f / (2.0 + f);
  z = s * s;
  double R4 = fma(z, Lp7, Lp6), R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4);
  double z2 = z * z, z4 = z2 * z2, z6 = z2 * z4;
  R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, z2 * R2)));
  double t = (hfsq + R) * s;
  if (k == 0) return f - (hfsq - t);
  return fma(dk, ln2_hi, -((hfsq - (t + fma(dk, ln2_lo, c))) - f));
}

/* ------------------------------------------------------------------ */
/* numpy random_standard_normal (distributions.c, numpy 2.3.5), restated.
 * Call site: pkg/src/rsvhmc/sampler.py:141 (refresh_momenta). */
double orc_standard_normal(orc_stream *st) {
  for (;;) {
    uint64_t r = orc_next_u64(st);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 0x1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * orc_wi_double[idx];
    if (sign & 0x1) x = -x;
    if (rabs < orc_ki_double[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = ORC_ZIG_NEG_INV_R * orc_log1p(-orc_next_double(st));
        double yy = -orc_log1p(-orc_next_double(st));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 0x1) ? -(ORC_ZIG_R + xx) : ORC_ZIG_R + xx;
      }
    } else {
      if (((orc_fi_double[idx - 1] - orc_fi_double[idx]) * orc_next_double(st) + orc_fi_double[idx]) <
          exp(-0.5 * x * x))
        return x;
    }
  }
}
void orc_fill_normal(orc_stream *st, double *out, int64_t n) { for (int64_t i = 0; i < n; i++) out[i] = orc_standard_normal(st); }

/* ------------------------------------------------------------------ */
/* numpy pairwise summation (umath loops, PW_BLOCKSIZE 128) */
static double pairwise(const double *a, int64_t n) {
  if (n < 8) { double r = 0.; for (int64_t i = 0; i < n; i++) r += a[i]; return r; }
  if (n <= 128) {
    double r[8]; int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8) for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  int64_t n2 = n / 2; n2 -= n2 % 8;
  return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

typedef struct { double phi, mu, xi, sigma_eta_sq, sigma_u_sq; } orc_params;

/* pkg/src/rsvhmc/model.py:134-163 log_posterior (three blocks, pairwise sums). */
double orc_log_posterior(const double *h, const orc_params *P, const double *y, const double *lrv, int64_t T) {
  double *w = (double *)malloc(sizeof(double) * (size_t)(T > 1 ? T : 1));
  double phi = P->phi, mu = P->mu, xi = P->xi, se2 = P->sigma_eta_sq, su2 = P->sigma_u_sq;
  double sh = pairwise(h, T);
  for (int64_t i = 0; i < T; i++) w[i] = y[i] * y[i] * exp(-h[i]);
  double returns_block = -0.5 * sh - 0.5 * pairwise(w, T);
  for (int64_t i = 0; i < T; i++) { double ru = lrv[i] - xi - h[i]; w[i] = ru * ru; }
  double rv_block = -0.5 * (double)T * log(su2) - pairwise(w, T) / (2.0 * su2);
  for (int64_t i = 0; i + 1 < T; i++) { double tr = (h[i + 1] - mu) - phi * (h[i] - mu); w[i] = tr * tr; }
  double d0 = h[0] - mu;
  double ar_block = -0.5 * log(se2 / (1.0 - phi * phi)) - (1.0 - phi * phi) * d0 * d0 / (2.0 * se2) -
                    0.5 * (double)(T - 1) * log(se2) - pairwise(w, T - 1) / (2.0 * se2);
  free(w);
  return returns_block + rv_block + ar_block;
}

/* pkg/src/rsvhmc/model.py:178-182 hamiltonian */
double orc_hamiltonian(const double *h, const double *p, const orc_params *P, const double *y, const double *lrv, int64_t T) {
  double *w = (double *)malloc(sizeof(double) * (size_t)T);
  for (int64_t i = 0; i < T; i++) w[i] = p[i] * p[i];
  double kin = 0.5 * pairwise(w, T);
  free(w);
  return kin - orc_log_posterior(h, P, y, lrv, T);
}

/* pkg/src/rsvhmc/_kernels.py:23-34 _grad_site; scalars as model.py:185-199 scalar_pack */
typedef struct { double half, phi, mu, xi, inv_su2, inv_se2, one_m_phi2; } orc_scal;
static orc_scal pack(const orc_params *P) {
  orc_scal s = {0.5, P->phi, P->mu, P->xi, 1.0 / P->sigma_u_sq, 1.0 / P->sigma_eta_sq, 1.0 - P->phi * P->phi};
  return s;
}
static inline double grad_site(const double *h, const double *y, const double *lrv, int64_t i, int64_t T, const orc_scal *s) {
  double v = h[i];
  double g = s->half - s->half * y[i] * y[i] * exp(-v) + (s->xi + v - lrv[i]) * s->inv_su2;
  if (i == 0) g += s->one_m_phi2 * (v - s->mu) * s->inv_se2;
  else g += (v - s->mu - s->phi * (h[i - 1] - s->mu)) * s->inv_se2;
  if (i < T - 1) g -= s->phi * (h[i + 1] - s->mu - s->phi * (v - s->mu)) * s->inv_se2;
  return g;
}

/* _kernels.py:57-67 gradient_fill; model.py:166-175 grad_neg_log_posterior */
int orc_gradient(const double *h, const orc_params *P, const double *y, const double *lrv, double *out, int64_t T) {
  orc_scal s = pack(P);
  int flag = 0;
  for (int64_t i = 0; i < T; i++) {
    double v = h[i];
    if (!(-50.0 <= v && v <= 50.0)) flag = 1;
    out[i] = grad_site(h, y, lrv, i, T, &s);
  }
  return flag;
}


/* ------------------------------------------------------------------ */
/* Minimal persistent pthread pool for the multi-threaded CPU baseline:
 * a static partition of [0, n) over the workers (the reference's
 * ParallelBackend, integrator.py:68-96, chunks the range the same way:
 * results do not depend on the worker count because writes are disjoint). */
typedef void (*orc_task_fn)(void *ctx, int64_t lo, int64_t hi, int *flag);
static struct {
  int n;                 /* threads incl. caller */
  pthread_t th[256];
  pthread_barrier_t start, done;
  orc_task_fn fn; void *ctx; int64_t len; int flags[256]; int quit;
} g_pool;
static void *pool_main(void *arg) {
  int id = (int)(intptr_t)arg;
  for (;;) {
    pthread_barrier_wait(&g_pool.start);
    if (g_pool.quit) return NULL;
    int64_t n = g_pool.len, per = (n + g_pool.n - 1) / g_pool.n, lo = id * per, hi = lo + per < n ? lo + per : n;
    g_pool.flags[id] = 0;
    if (lo < hi) g_pool.fn(g_pool.ctx, lo, hi, &g_pool.flags[id]);
    pthread_barrier_wait(&g_pool.done);
  }
}
static void pool_shutdown(void) {
  if (g_pool.n > 1) {
    g_pool.quit = 1;
    pthread_barrier_wait(&g_pool.start);
    for (int i = 1; i < g_pool.n; i++) pthread_join(g_pool.th[i], NULL);
    pthread_barrier_destroy(&g_pool.start); pthread_barrier_destroy(&g_pool.done);
  }
  g_pool.n = 0; g_pool.quit = 0;
}
static void pool_ensure(int n) {
  if (n < 1) n = 1;
  if (n > 256) n = 256;
  if (g_pool.n == n) return;
  pool_shutdown();
  g_pool.n = n;
  if (n > 1) {
    pthread_barrier_init(&g_pool.start, NULL, (unsigned)n);
    pthread_barrier_init(&g_pool.done, NULL, (unsigned)n);
    for (int i = 1; i < n; i++) pthread_create(&g_pool.th[i], NULL, pool_main, (void *)(intptr_t)i);
  }
}
static int pool_run(int nthreads, orc_task_fn fn, void *ctx, int64_t len) {
  if (nthreads <= 1 || len < 4096) { int f = 0; fn(ctx, 0, len, &f); return f; }
  pool_ensure(nthreads);
  g_pool.fn = fn; g_pool.ctx = ctx; g_pool.len = len;
  pthread_barrier_wait(&g_pool.start);
  int64_t per = (len + g_pool.n - 1) / g_pool.n, hi = per < len ? per : len;
  g_pool.flags[0] = 0;
  fn(ctx, 0, hi, &g_pool.flags[0]);
  pthread_barrier_wait(&g_pool.done);
  int f = 0;
  for (int i = 0; i < g_pool.n; i++) f |= g_pool.flags[i];
  return f;
}
void orc_pool_shutdown(void) { pool_shutdown(); }

typedef struct { double *h; double *p; const double *y, *lrv; double c, dt; const void *s; int64_t T; } lf_ctx;

/* _kernels.py:37-41 position_update (integrator.py:111-116 kernel1/3) */
static void pos_task(void *v, int64_t lo, int64_t hi, int *flag) {
  lf_ctx *c = (lf_ctx *)v;
  (void)flag;
  for (int64_t i = lo; i < hi; i++) c->h[i] += c->c * c->p[i];
}
static void position_update(double *h, double *p, double c, int64_t T, int nthreads) {
  lf_ctx ctx = {h, p, NULL, NULL, c, 0.0, NULL, T};
  pool_run(nthreads, pos_task, &ctx, T);
}
/* _kernels.py:44-54 momentum_update (integrator.py:119-131 kernel2) */
static void mom_task(void *v, int64_t lo, int64_t hi, int *flag) {
  lf_ctx *c = (lf_ctx *)v;
  const orc_scal *s = (const orc_scal *)c->s;
  int f = 0;
  for (int64_t i = lo; i < hi; i++) {
    double x = c->h[i];
    if (!(-50.0 <= x && x <= 50.0)) f = 1;
    c->p[i] -= c->dt * grad_site(c->h, c->y, c->lrv, i, c->T, s);
  }
  *flag = f;
}
static int momentum_update(double *h, double *p, const double *y, const double *lrv, double dt, const orc_scal *s,
                           int64_t T, int nthreads) {
  lf_ctx ctx = {h, p, y, lrv, 0.0, dt, s, T};
  return pool_run(nthreads, mom_task, &ctx, T);
}

/* integrator.py:139-146 elementary_step: K1 -> K2 -> K3 in place */
int orc_elementary_step(double *h, double *p, const orc_params *P, const double *y, const double *lrv, int64_t T,
                        double dt, int nthreads) {
  orc_scal s = pack(P);
  double c = 0.5 * dt;
  position_update(h, p, c, T, nthreads);
  int d = momentum_update(h, p, y, lrv, dt, &s, T, nthreads);
  position_update(h, p, c, T, nthreads);
  return d;
}

/* integrator.py:149-179 integrate_trajectory on (h, p) in place (caller copies).
 * Returns 1 if diverged (state then meaningless), 0 otherwise. */
int orc_integrate(double *h, double *p, const orc_params *P, const double *y, const double *lrv, int64_t T, double dt,
                  int n_steps, int fuse, int nthreads) {
  orc_scal s = pack(P);
  if (!fuse) {
    for (int k = 0; k < n_steps; k++)
      if (orc_elementary_step(h, p, P, y, lrv, T, dt, nthreads)) return 1;
    return 0;
  }
  position_update(h, p, 0.5 * dt, T, nthreads);
  for (int k = 0; k < n_steps; k++) {
    if (momentum_update(h, p, y, lrv, dt, &s, T, nthreads)) return 1;
    if (k < n_steps - 1) position_update(h, p, dt, T, nthreads);
  }
  position_update(h, p, 0.5 * dt, T, nthreads);
  return 0;
}

/* sampler.py:144-167 hmc_update_volatility.  h is updated in place on
 * acceptance; returns accept flag; *delta_h gets dH or +inf (divergence). */
int orc_hmc_update(double *h, const orc_params *P, const double *y, const double *lrv, int64_t T, double dt,
                   int n_steps, orc_stream *st, double *delta_h, double *work, int nthreads, int fuse) {
  double *p = work, *hp = work + T;
  orc_fill_normal(st, p, T);                                   /* sampler.py:153 */
  double h_old = orc_hamiltonian(h, p, P, y, lrv, T);           /* :155 */
  memcpy(hp, h, sizeof(double) * (size_t)T);                    /* integrator.py:160 */
  if (orc_integrate(hp, p, P, y, lrv, T, dt, n_steps, fuse, nthreads)) /* integrator.py:149 fuse_half_steps */ { *delta_h = INFINITY; return 0; }
  double h_new = orc_hamiltonian(hp, p, P, y, lrv, T);          /* :159 */
  double dh = h_new - h_old;
  if (!isfinite(dh) || fabs(dh) > 1000.0) { *delta_h = INFINITY; return 0; }
  double u = orc_next_double(st);                               /* :163 */
  *delta_h = dh;
  int accept = dh <= 0.0 || u < exp(-dh);
  if (accept) memcpy(h, hp, sizeof(double) * (size_t)T);
  return accept;
}

/* Sufficient statistics of h for the theta full conditionals
 * (sampler.py:170-230, 249-272), shifted by c_mu (for h) and c_xi (for
 * lnRV - h) to avoid cancellation:
 *   m[0] = d_0, m[1] = d_{T-1}, m[2] = sum d, m[3] = sum d^2,
 *   m[4] = sum_{t>=1} d_t d_{t-1}, m[5] = sum e, m[6] = sum e^2
 * with d = h - c_mu and e = lnRV - h - c_xi. */
void orc_suff_stats(const double *h, const double *lrv, int64_t T, double c_mu, double c_xi, double m[7]) {
  double *w = (double *)malloc(sizeof(double) * (size_t)T);
  m[0] = h[0] - c_mu; m[1] = h[T - 1] - c_mu;
  for (int64_t i = 0; i < T; i++) w[i] = h[i] - c_mu;
  m[2] = pairwise(w, T);
  for (int64_t i = 0; i < T; i++) { double d = h[i] - c_mu; w[i] = d * d; }
  m[3] = pairwise(w, T);
  for (int64_t i = 0; i + 1 < T; i++) w[i] = (h[i + 1] - c_mu) * (h[i] - c_mu);
  m[4] = pairwise(w, T - 1);
  for (int64_t i = 0; i < T; i++) w[i] = lrv[i] - h[i] - c_xi;
  m[5] = pairwise(w, T);
  for (int64_t i = 0; i < T; i++) { double e = lrv[i] - h[i] - c_xi; w[i] = e * e; }
  m[6] = pairwise(w, T);
  free(w);
}

int orc_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
