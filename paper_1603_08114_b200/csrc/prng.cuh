// prng.cuh -- raw-word bit generators and numpy's ziggurat on sm_100a.
//
// Replaces the reference's RNG path: sampler.py:131-133 make_rng (numpy
// Philox) and sampler.py:141 rng.standard_normal (numpy ziggurat,
// numpy/random/src/distributions/distributions.c random_standard_normal,
// numpy 2.3.5).  Every generator exposes word(k) = the k-th raw 64-bit word
// of the stream (random access for the counter/jump-ahead kinds), so the
// momenta can be drawn by thousands of threads and still match the
// sequential numpy stream bit for bit.  See DESIGN.md "Momenta".
#pragma once
#include <stdint.h>

#include "zig_tables.h"

#ifndef RSV_HD
#define RSV_HD __host__ __device__ __forceinline__
#endif

namespace rsv {

enum { PRNG_PHILOX = 0, PRNG_MINSTD = 1, PRNG_PCG32 = 2, PRNG_SFC64 = 3 };

struct StreamState {  // mirrors rsv_prng_state
  int32_t kind;
  int32_t reserved;
  uint64_t s[4];
  uint64_t pos;
};

RSV_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((__uint128_t)a * b) >> 64);
#endif
}

// Random123 / numpy philox4x64_10: ctr = {blk + 1, 0, 0, 0} for block blk
// (numpy increments the counter before generating each block of 4 words).
RSV_HD void philox_block(uint64_t blk, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = blk + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = mulhi64(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = mulhi64(0xCA5A826395121157ULL, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// std::minstd_rand: x_{j+1} = 48271 x_j mod (2^31 - 1).
constexpr uint64_t MINSTD_M = 2147483647ULL;
constexpr uint64_t MINSTD_A = 48271ULL;
RSV_HD uint64_t mod31(uint64_t x) {  // x < 2^62
  x = (x & MINSTD_M) + (x >> 31);
  x = (x & MINSTD_M) + (x >> 31);
  return x >= MINSTD_M ? x - MINSTD_M : x;
}
RSV_HD uint64_t minstd_pow(uint64_t e) {
  uint64_t r = 1, a = MINSTD_A;
  while (e) {
    if (e & 1) r = mod31(r * a);
    a = mod31(a * a);
    e >>= 1;
  }
  return r;
}

// pcg_basic: pcg32_random_r / pcg32_advance_r.
constexpr uint64_t PCG_MULT = 6364136223846793005ULL;
RSV_HD uint64_t pcg_advance(uint64_t state, uint64_t delta, uint64_t plus) {
  uint64_t mult = PCG_MULT, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) { acc_mult *= mult; acc_plus = acc_plus * mult + plus; }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}
RSV_HD uint32_t pcg_output(uint64_t old) {
  const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  const uint32_t rot = (uint32_t)(old >> 59u);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

// numpy sfc64_next
RSV_HD uint64_t sfc64_next(uint64_t s[4]) {
  const uint64_t tmp = s[0] + s[1] + s[3]++;
  s[0] = s[1] ^ (s[1] >> 11);
  s[1] = s[2] + (s[2] << 3);
  s[2] = ((s[2] << 24) | (s[2] >> 40)) + tmp;
  return tmp;
}

// Random access to raw word k (absolute stream index) of a counter /
// jump-ahead stream.  SFC64 is sequential and never goes through here.
RSV_HD uint64_t word_at(const StreamState &st, uint64_t k) {
  if (st.kind == PRNG_PHILOX) {
    uint64_t b[4];
    philox_block(k >> 2, st.s[0], st.s[1], b);
    return b[k & 3];
  } else if (st.kind == PRNG_MINSTD) {
    const uint64_t xa = mod31(minstd_pow(3 * k + 1) * st.s[0]);
    const uint64_t xb = mod31(xa * MINSTD_A);
    const uint64_t xc = mod31(xb * MINSTD_A);
    return (xa << 33) | (xb << 2) | (xc >> 29);
  } else {  // PCG32
    const uint64_t s0 = pcg_advance(st.s[0], 2 * k, st.s[1]);
    const uint64_t s1 = s0 * PCG_MULT + st.s[1];
    return ((uint64_t)pcg_output(s0) << 32) | pcg_output(s1);
  }
}

// Sequential generator positioned at absolute word k (cheap next()).
struct SeqGen {
  int kind;
  uint64_t a, b;      // philox key | minstd x | pcg state, inc
  uint64_t k;         // next word index
  uint64_t buf[4];
  RSV_HD void init(const StreamState &st, uint64_t k0) {
    kind = st.kind;
    k = k0;
    if (kind == PRNG_PHILOX) {
      a = st.s[0]; b = st.s[1];
      if (k0 & 3) philox_block(k0 >> 2, a, b, buf);
    } else if (kind == PRNG_MINSTD) {
      a = mod31(minstd_pow(3 * k0) * st.s[0]);  // x_{3k0}; next output is x_{3k0+1}
    } else {
      a = pcg_advance(st.s[0], 2 * k0, st.s[1]);
      b = st.s[1];
    }
  }
  RSV_HD uint64_t next() {
    uint64_t w;
    if (kind == PRNG_PHILOX) {
      if ((k & 3) == 0) philox_block(k >> 2, a, b, buf);
      w = buf[k & 3];
    } else if (kind == PRNG_MINSTD) {
      const uint64_t xa = mod31(a * MINSTD_A), xb = mod31(xa * MINSTD_A), xc = mod31(xb * MINSTD_A);
      a = xc;
      w = (xa << 33) | (xb << 2) | (xc >> 29);
    } else {
      const uint64_t s0 = a, s1 = s0 * PCG_MULT + b;
      a = s1 * PCG_MULT + b;
      w = ((uint64_t)pcg_output(s0) << 32) | pcg_output(s1);
    }
    k++;
    return w;
  }
};

RSV_HD double u01(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

// glibc 2.39 log1p (fdlibm algorithm, Estrin polynomial) exactly as its
// FMA-capable x86-64 variant evaluates it -- every multiply/add/fma is
// spelled out so nvcc cannot contract differently.  numpy's ziggurat tail
// calls log1p(-u); matching glibc keeps those normals bit-exact.
#ifdef __CUDA_ARCH__
#define RSV_FMA(a, b, c) __fma_rn(a, b, c)
#define RSV_MUL(a, b) __dmul_rn(a, b)
#define RSV_ADD(a, b) __dadd_rn(a, b)
#define RSV_SUB(a, b) __dsub_rn(a, b)
#define RSV_DIV(a, b) __ddiv_rn(a, b)
#else
#define RSV_FMA(a, b, c) fma(a, b, c)
#define RSV_MUL(a, b) ((a) * (b))
#define RSV_ADD(a, b) ((a) + (b))
#define RSV_SUB(a, b) ((a) - (b))
#define RSV_DIV(a, b) ((a) / (b))
#endif

RSV_HD int32_t hi_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2hiint(x);
#else
  uint64_t u; __builtin_memcpy(&u, &x, 8); return (int32_t)(u >> 32);
#endif
}
RSV_HD double with_hi_word(double x, int32_t h) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(h, __double2loint(x));
#else
  uint64_t u; __builtin_memcpy(&u, &x, 8);
  u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)h << 32);
  __builtin_memcpy(&x, &u, 8); return x;
#endif
}

RSV_HD double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double hfsq, f = 0, c = 0, s, z, R, u;
  int32_t k = 1, hu = 0;
  const int32_t hx = hi_word(x), ax = hx & 0x7fffffff;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -__builtin_huge_val() : __builtin_nan("");
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return RSV_FMA(-RSV_MUL(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) { k = 0; f = x; hu = 1; }
  }
  if (hx >= 0x7ff00000) return RSV_ADD(x, x);
  if (k != 0) {
    if (hx < 0x43400000) {
      u = RSV_ADD(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? RSV_SUB(1.0, RSV_SUB(u, x)) : RSV_SUB(x, RSV_SUB(u, 1.0));
      c = RSV_DIV(c, u);
    } else {
      u = x; hu = hi_word(u); k = (hu >> 20) - 1023; c = 0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = with_hi_word(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = RSV_SUB(u, 1.0);
  }
  hfsq = RSV_MUL(RSV_MUL(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = RSV_FMA(dk, ln2_lo, c);
      return RSV_FMA(dk, ln2_hi, c);
    }
    R = RSV_MUL(RSV_FMA(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return RSV_SUB(f, R);
    return RSV_FMA(dk, ln2_hi, -RSV_SUB(RSV_SUB(R, RSV_FMA(dk, ln2_lo, c)), f));
  }
  s = RSV_DIV(f, RSV_ADD(2.0, f));
  z = RSV_MUL(s, s);
  const double R4 = RSV_FMA(z, Lp7, Lp6), R2 = RSV_FMA(z, Lp3, Lp2), R3 = RSV_FMA(z, Lp5, Lp4);
  const double z2 = RSV_MUL(z, z), z4 = RSV_MUL(z2, z2), z6 = RSV_MUL(z2, z4);
  R = RSV_FMA(z6, R4, RSV_FMA(z4, R3, RSV_FMA(z, Lp1, RSV_MUL(z2, R2))));
  const double t = RSV_MUL(RSV_ADD(hfsq, R), s);
  if (k == 0) return RSV_SUB(f, RSV_SUB(hfsq, t));
  return RSV_FMA(dk, ln2_hi, -RSV_SUB(RSV_SUB(hfsq, RSV_ADD(t, RSV_FMA(dk, ln2_lo, c))), f));
}

}  // namespace rsv
