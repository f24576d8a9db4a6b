// momenta.cu -- bit-exact numpy momenta on the GPU, one kernel per draw.
//
// Replaces sampler.py:136-141 refresh_momenta = rng.standard_normal(T):
// numpy's 256-layer ziggurat (random_standard_normal, numpy 2.3.5).  A
// ziggurat draw consumes a variable number of raw words (1 on the 98.9 %
// fast path, 2 for a wedge test, 1 + 2m for m exponential-tail loops), so
// normal i's place in the raw stream depends on every earlier draw.
//
// zig_kernel parses the stream in parallel with *speculation + local
// verification*:
//   1. a CTA owns 2048 raw words (8 per thread) and stages them, plus a
//      16-word guard before and 32 look-ahead words after, in shared memory;
//   2. every word k is classified as if an attempt started there:
//      (len_k, acc_k, x_k);
//   3. each thread assumes the parse is "in sync" 16 words before its
//      segment (state 0 there) and walks forward to its segment: the
//      attempt chains of a ziggurat stream merge within a few words, so the
//      entry state it finds is the true one -- and it is *checked*: it must
//      equal the exit state of the previous thread's walk (and, for thread 0,
//      of the previous CTA).  By induction from word 0 every entry is exact;
//      any mismatch (p ~ 1e-30) or an attempt needing > 7 tail loops
//      (p ~ 1e-12 per word) diverts the draw to an exact serial walk;
//   4. per-thread normal counts are scanned in the CTA and across CTAs by a
//      decoupled look-back (single pass), and the normals are written to
//      their final slots.  The thread that emits normal T-1 records how many
//      words the draw used and the next raw word (the Metropolis uniform).
#include <math.h>

#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

__device__ const uint64_t g_ki[256] = RSV_KI_DOUBLE_INIT;
__device__ const double g_wi[256] = RSV_WI_DOUBLE_INIT;
__device__ const double g_fi[256] = RSV_FI_DOUBLE_INIT;

constexpr int ZG = 16;                 // guard words before a CTA's block
constexpr int ZLA = 32;                // look-ahead words after it
constexpr int ZSW = ZG + ZB + ZLA;     // staged words per CTA
constexpr int ZCH = ZSW / ZW;          // 8-word chunks per CTA (262)
constexpr int ZDIRECT = 4096;          // up to this many CTAs: direct predecessor sums

struct ZigJump {  // per-chunk jump-ahead constants (inc-free), built once
  uint64_t pcg_a[ZCH], pcg_g[ZCH];     // state_c = a * base + inc * g  (16 c outputs ahead)
  uint64_t minstd_a[ZCH];              // x_c = a * x_base mod m        (24 c outputs ahead)
};
__device__ ZigJump g_jump;

__global__ void zig_jump_init_kernel() {
  if (threadIdx.x || blockIdx.x) return;
  // pcg: 16 outputs per chunk; accumulate (A^k, G_k) with G_k = sum_{i<k} A^i
  uint64_t a = 1, g = 0;
  uint64_t A16 = 1, G16 = 0;
  for (int i = 0; i < 16; i++) { G16 = G16 * PCG_MULT + 1; A16 *= PCG_MULT; }
  uint64_t m = 1, m24 = minstd_pow(24);
  for (int c = 0; c < ZCH; c++) {
    g_jump.pcg_a[c] = a;
    g_jump.pcg_g[c] = g;
    g_jump.minstd_a[c] = m;
    g = g * A16 + G16;  // (A^k,G_k) o (A^16,G_16)
    a *= A16;
    m = mod31(m * m24);
  }
}

struct ZigShared {
  uint64_t w[ZSW];        // raw words: local index i <-> draw word b*ZB - ZG + i
  double x[ZB];           // candidate normal of an attempt starting at block word k
  uint8_t len[ZG + ZB];   // attempt length | acc << 7 for guard + block words
  uint64_t ki[256];
  double wi[256];
  int32_t warp_tot[ZT / 32];
  int32_t warp_exit[ZT / 32];
  uint64_t base_a, base_b;  // sequential-generator state at local word 0
  uint64_t blk_off;         // exclusive normal offset of this CTA
  int32_t blk;              // dynamic CTA index (ticket)
  int32_t bad;
  int32_t warp0_entry;      // thread 0's speculative entry state
  uint32_t epoch;           // this draw's tag in the look-back status words
};

// Classify the attempt starting at local word i (numpy random_standard_normal).
__device__ __forceinline__ void zig_classify_at(const ZigShared &S, int i, int mmax, int &len, int &acc, double &x) {
  uint64_t r = S.w[i];
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const int sign = (int)(r & 0x1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  // rabs < 2^52: (2^52 | rabs) - 2^52 is exactly (double)rabs
  const double fr = __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | rabs)), 4503599627370496.0);
  x = __dmul_rn(fr, S.wi[idx]);
  if (sign) x = -x;
  if (rabs < S.ki[idx]) { len = 1; acc = 1; return; }
  if (idx == 0) {
    for (int m = 1; m <= mmax; m++) {
      const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R, glibc_log1p(-u01(S.w[i + 2 * m - 1])));
      const double yy = -glibc_log1p(-u01(S.w[i + 2 * m]));
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        x = ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xx) : __dadd_rn(RSV_ZIG_R, xx);
        len = 1 + 2 * m;
        acc = 1;
        return;
      }
    }
    len = 0;  // needs more tail loops than staged words: exact serial fallback
    acc = 0;
    return;
  }
  const double u = u01(S.w[i + 1]);
  const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(g_fi[idx - 1], g_fi[idx]), u), g_fi[idx]);
  acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x)) ? 1 : 0;
  len = 2;
}

// decoupled look-back status word: [63:62] flag (1 aggregate, 2 prefix),
// [61:58] exit state of the CTA's parse, [57:34] draw epoch (words from an
// earlier draw read as "not ready", so the array needs no reset), [33:0] count
constexpr uint64_t ZCNT = (1ULL << 34) - 1;
__device__ __forceinline__ uint64_t zpack(int flag, int exitst, uint32_t epoch, uint64_t cnt) {
  return ((uint64_t)flag << 62) | ((uint64_t)exitst << 58) | ((uint64_t)epoch << 34) | cnt;
}
__device__ __forceinline__ bool zready(uint64_t v, uint32_t epoch) {
  return (v >> 62) != 0 && (uint32_t)((v >> 34) & 0xffffffu) == epoch;
}

template <int KIND>
__device__ __forceinline__ void stage_words(ZigShared &S, const DevControl *ctrl, const uint64_t *words, int b,
                                            int64_t nwords_buf, const uint64_t *bjump) {
  const int tid = threadIdx.x;
  const int64_t rel0 = (int64_t)b * ZB - ZG;  // draw-relative index of local word 0
  if (KIND == PRNG_SFC64) {
    for (int i = tid; i < ZSW; i += ZT) {
      const int64_t k = rel0 + i;
      S.w[i] = (k >= 0 && k < nwords_buf) ? words[k] : 0;
    }
    return;
  }
  const StreamState &st = ctrl->stream;
  if (tid == 0) {
    // state in front of local word 0 (draw word rel0 may be negative for CTA 0:
    // the guard is never walked there, start at word 0 and shift): the
    // generator state at the stream position, jumped by this CTA's offset
    // with a precomputed per-CTA constant (bjump, built once per context)
    if (KIND == PRNG_PCG32) S.base_a = bjump[2 * b] * ctrl->seq_state + st.s[1] * bjump[2 * b + 1];
    else if (KIND == PRNG_MINSTD) S.base_a = mod31(bjump[b] * ctrl->seq_state);
  }
  __syncthreads();
  const int shift = rel0 < 0 ? ZG : 0;  // CTA 0: local word ZG is draw word 0
  for (int c = tid; c < ZCH; c += ZT) {
    const int i0 = c * ZW;
    if (i0 + ZW <= shift) {  // pure guard chunk of CTA 0: no words there
      for (int i = 0; i < ZW; i++) S.w[i0 + i] = 0;
    } else if (KIND == PRNG_PHILOX) {
      SeqGen g;
      g.init(st, st.pos + (uint64_t)(rel0 + i0));
#pragma unroll
      for (int i = 0; i < ZW; i++) S.w[i0 + i] = g.next();
    } else if (KIND == PRNG_PCG32) {
      const int cc = c - shift / ZW;
      uint64_t s0 = g_jump.pcg_a[cc] * S.base_a + st.s[1] * g_jump.pcg_g[cc];
#pragma unroll
      for (int i = 0; i < ZW; i++) {
        const uint64_t s1 = s0 * PCG_MULT + st.s[1];
        S.w[i0 + i] = ((uint64_t)pcg_output(s0) << 32) | pcg_output(s1);
        s0 = s1 * PCG_MULT + st.s[1];
      }
    } else {  // MINSTD
      const int cc = c - shift / ZW;
      uint64_t x = mod31(g_jump.minstd_a[cc] * S.base_a);
#pragma unroll
      for (int i = 0; i < ZW; i++) {
        const uint64_t xa = mod31(x * MINSTD_A), xb = mod31(xa * MINSTD_A), xc = mod31(xb * MINSTD_A);
        x = xc;
        S.w[i0 + i] = (xa << 33) | (xb << 2) | (xc >> 29);
      }
    }
  }
}

__device__ void zig_serial(DevControl *ctrl, const uint64_t *words, int64_t nbuf, double *normals, int64_t T);

__device__ __forceinline__ unsigned long long zgt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int KIND>
__global__ void __launch_bounds__(ZT) zig_kernel(DevControl *ctrl, const uint64_t *words, int64_t nwords_buf,
                                                 double *normals, int64_t T, uint64_t *status, const uint64_t *bjump,
                                                 unsigned long long *dbg) {
#define ZSTAMP(k) \
  do { if (dbg && threadIdx.x == 0) dbg[(size_t)blockIdx.x * 8 + (k)] = zgt(); } while (0)
  ZSTAMP(0);
  extern __shared__ __align__(16) unsigned char zsmem[];
  ZigShared &S = *reinterpret_cast<ZigShared *>(zsmem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    S.blk = (int)atomicAdd(&ctrl->zig_ticket, 1u);
    S.epoch = ctrl->zig_epoch & 0xffffffu;
    S.bad = 0;
  }
  for (int i = tid; i < 256; i += ZT) {
    S.ki[i] = g_ki[i];
    S.wi[i] = g_wi[i];
  }
  __syncthreads();
  const int b = S.blk;
  ZSTAMP(1);
  stage_words<KIND>(S, ctrl, words, b, nwords_buf, bjump);
  __syncthreads();
  ZSTAMP(2);

  // ---- classify every guard + block word as an attempt start
  const int first = (b == 0) ? ZG : 0;  // CTA 0 has no guard
  int ovf = 0;
  for (int i = tid; i < ZG + ZB; i += ZT) {
    if (i < first) { S.len[i] = 1; continue; }
    int len, acc;
    double x;
    zig_classify_at(S, i, ZMMAX, len, acc, x);
    S.len[i] = (uint8_t)(len | (acc << 7));
    if (i >= ZG) S.x[i - ZG] = x;
    ovf |= (len == 0);
  }
  if (ovf) atomicOr(&ctrl->zig_overflow, 1);
  __syncthreads();
  ZSTAMP(3);

  // ---- speculative walk: in sync 16 words before my segment
  const int seg = ZG + tid * ZW;
  int pos = (b == 0 && tid == 0) ? ZG : seg - ZG;
  while (pos < seg) {
    const int L = S.len[pos] & 15;
    pos += L ? L : 1;
  }
  const int entry = pos - seg;
  if (tid == 0) S.warp0_entry = entry;
  int cnt = 0;
  while (pos < seg + ZW) {
    const uint8_t m = S.len[pos];
    cnt += m >> 7;
    const int L = m & 15;
    pos += L ? L : 1;
  }
  const int exitst = pos - (seg + ZW);
  // verify: my entry == previous thread's exit
  int prev_exit = __shfl_up_sync(0xffffffffu, exitst, 1);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) {
    S.warp_tot[warp] = incl;
    S.warp_exit[warp] = exitst;
  }
  __syncthreads();
  if (lane == 0 && warp > 0) prev_exit = S.warp_exit[warp - 1];
  if (tid > 0 && prev_exit != entry) S.bad = 1;
  int woff = 0, btot = 0;
  for (int w = 0; w < ZT / 32; w++) {
    if (w < warp) woff += S.warp_tot[w];
    btot += S.warp_tot[w];
  }
  const int toff = woff + incl - cnt;  // exclusive offset of my normals in the CTA

  ZSTAMP(4);
  // ---- decoupled look-back over CTAs for the global normal offset
  // (warp 0 inspects 32 predecessors per round)
  if (warp == 0) {
    const int bexit = S.warp_exit[ZT / 32 - 1];
    volatile uint64_t *vst = status;
    if (b == 0) {
      if (lane == 0) {
        vst[0] = zpack(2, bexit, S.epoch, (uint64_t)btot);
        S.blk_off = 0;
        if (entry != 0) S.bad = 1;
      }
    } else {
      if (lane == 0) vst[b] = zpack(1, bexit, S.epoch, (uint64_t)btot);
      uint64_t acc = 0;
      if (gridDim.x <= ZDIRECT) {
        // small grids: every CTA sums all its predecessors' aggregates in one
        // round of independent loads (no chain of published prefixes)
        for (;;) {
          uint64_t part = 0;
          bool ok = true;
          for (int j = lane; j < b; j += 32) {
            const uint64_t v = vst[j];
            ok &= zready(v, S.epoch);
            part += v & ZCNT;
          }
          if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            acc = part;
            break;
          }
          __nanosleep(100);
        }
        if (lane == 0) {
          const uint64_t prev = vst[b - 1];
          if ((int)((prev >> 58) & 15) != S.warp0_entry) S.bad = 1;
        }
      } else {
      // look back 256 predecessors per round (8 independent loads per lane)
      int hi = b - 1;
      bool checked = false;
      for (;;) {
        // 8 independent loads per lane, re-issued until every predecessor in
        // the window has published (no serial chain of dependent loads)
        uint64_t sv[8];
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int w = 0; w < 8; w++) {
            const int j = hi - lane - 32 * w;
            sv[w] = j >= 0 ? vst[j] : (uint64_t)S.epoch << 34 | 2ULL << 62;  // before CTA 0: empty prefix
          }
#pragma unroll
          for (int w = 0; w < 8; w++) ok &= zready(sv[w], S.epoch);
          if (__all_sync(0xffffffffu, ok)) break;
          __nanosleep(200);  // back off: hundreds of CTAs poll the same lines
        }
        if (!checked) {  // the previous CTA's exit must equal my thread 0's entry
          const uint64_t prev = __shfl_sync(0xffffffffu, sv[0], 0);
          if (lane == 0 && (int)((prev >> 58) & 15) != S.warp0_entry) S.bad = 1;
          checked = true;
        }
        bool done = false;
        uint64_t mine = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) {
          if (!done) {
            const unsigned pref = __ballot_sync(0xffffffffu, (sv[w] >> 62) == 2);
            const int stop = pref ? __ffs(pref) - 1 : 32;  // nearest predecessor holding a prefix
            if (lane <= stop) mine += sv[w] & ZCNT;
            done = pref != 0;
          }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        acc += mine;
        if (done) break;
        hi -= 256;
      }
      }
      if (lane == 0) {
        S.blk_off = acc;
        // prefixes are only consumed by the chained look-back of large grids
        // (the direct sums need every CTA's own count to stay in place)
        if (gridDim.x > ZDIRECT) {
          __threadfence();
          vst[b] = zpack(2, bexit, S.epoch, acc + (uint64_t)btot);
        }
      }
    }
    if (lane == 0 && S.bad) atomicOr(&ctrl->zig_overflow, 2);
  }
  __syncthreads();

  ZSTAMP(5);
  // ---- write my normals to their final slots
  uint64_t off = S.blk_off + (uint64_t)toff;
  pos = seg + entry;
  if (off < (uint64_t)T) {
    while (pos < seg + ZW) {
      const uint8_t m = S.len[pos];
      const int L = m & 15;
      if (m >> 7) {
        if (off < (uint64_t)T) normals[off] = S.x[pos - ZG];
        if (off == (uint64_t)T - 1) {
          const int nxt = pos + L;  // local index of the next unread word
          ctrl->zig_used = (uint64_t)((int64_t)b * ZB - ZG + nxt);
          ctrl->u_word = S.w[nxt];
          const int shift = b == 0 ? ZG : 0;  // local word of the CTA's base state
          if (KIND == PRNG_PCG32) ctrl->seq_next = pcg_advance(S.base_a, 2 * (uint64_t)(nxt - shift), ctrl->stream.s[1]);
          else if (KIND == PRNG_MINSTD) ctrl->seq_next = mod31(minstd_pow(3 * (uint64_t)(nxt - shift)) * S.base_a);
        }
        off++;
      }
      pos += L ? L : 1;
    }
  }
  // the last CTA publishes how many normals the parse produced
  if (tid == ZT - 1 && b == (int)gridDim.x - 1) ctrl->zig_avail = S.blk_off + (uint64_t)btot;
  ZSTAMP(6);
  // the CTA that finishes last re-arms the bookkeeping and, if the parallel
  // parse could not be trusted (p ~ 1e-12 per word), redoes it serially
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned done = atomicAdd(&ctrl->zig_done, 1u);
    if (done == gridDim.x - 1) {
      __threadfence();
      if (ctrl->zig_overflow != 0 || ctrl->zig_avail < (uint64_t)T) zig_serial(ctrl, words, nwords_buf, normals, T);
      ctrl->zig_overflow = 0;
      ctrl->zig_ticket = 0;
      ctrl->zig_done = 0;
      ctrl->zig_epoch = ctrl->zig_epoch + 1;
    }
  }
}

// Exact serial walk of the whole draw (fallback; normally exits at once).
__device__ uint64_t serial_word(const StreamState &st, const uint64_t *words, int64_t nbuf, uint64_t j) {
  if (st.kind == PRNG_SFC64) return j < (uint64_t)nbuf ? words[j] : 0;  // past the buffer: flagged below
  return word_at(st, st.pos + j);
}

__device__ void zig_serial(DevControl *ctrl, const uint64_t *words, int64_t nbuf, double *normals, int64_t T) {
  const StreamState st = ctrl->stream;
  uint64_t j = 0;
  for (int64_t i = 0; i < T;) {
    uint64_t r = serial_word(st, words, nbuf, j);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, g_wi[idx]);
    if (sign) x = -x;
    j++;
    if (rabs < g_ki[idx]) { normals[i++] = x; continue; }
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R, glibc_log1p(-u01(serial_word(st, words, nbuf, j))));
        const double yy = -glibc_log1p(-u01(serial_word(st, words, nbuf, j + 1)));
        j += 2;
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          normals[i++] = ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xx) : __dadd_rn(RSV_ZIG_R, xx);
          break;
        }
      }
    } else {
      const double u = u01(serial_word(st, words, nbuf, j));
      j++;
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(g_fi[idx - 1], g_fi[idx]), u), g_fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) normals[i++] = x;
    }
  }
  ctrl->zig_used = j;
  ctrl->u_word = serial_word(st, words, nbuf, j);
  if (st.kind == PRNG_PCG32) ctrl->seq_next = pcg_advance(st.s[0], 2 * (st.pos + j), st.s[1]);
  else if (st.kind == PRNG_MINSTD) ctrl->seq_next = mod31(minstd_pow(3 * (st.pos + j)) * st.s[0]);
  ctrl->zig_avail = (uint64_t)T;
  ctrl->err |= 2;
  if (st.kind == PRNG_SFC64 && j + 1 > (uint64_t)nbuf) ctrl->err |= 1;  // ran past the generated words
}

// Z0: sequential SFC64 words (no jump-ahead exists) + state snapshots.
__global__ void z0_sfc64_kernel(DevControl *ctrl, uint64_t *words, uint64_t *snaps, int64_t n) {
  if (threadIdx.x || blockIdx.x) return;
  uint64_t s[4] = {ctrl->stream.s[0], ctrl->stream.s[1], ctrl->stream.s[2], ctrl->stream.s[3]};
  for (int64_t i = 0; i < n; i++) {
    if ((i % SFC_SNAP) == 0) {
      uint64_t *q = snaps + 4 * (i / SFC_SNAP);
      q[0] = s[0]; q[1] = s[1]; q[2] = s[2]; q[3] = s[3];
    }
    words[i] = sfc64_next(s);
  }
}

// Advance the stream past the last draw (refresh_momenta alone).
__global__ void zadvance_kernel(DevControl *ctrl, const uint64_t *snaps) {
  if (threadIdx.x || blockIdx.x) return;
  const uint64_t used = ctrl->zig_used;
  if (ctrl->stream.kind == PRNG_SFC64) {
    const uint64_t *q = snaps + 4 * (used / SFC_SNAP);
    uint64_t s[4] = {q[0], q[1], q[2], q[3]};
    for (uint64_t i = 0; i < used % SFC_SNAP; i++) sfc64_next(s);
    for (int i = 0; i < 4; i++) ctrl->stream.s[i] = s[i];
  }
  ctrl->stream.pos += used;
  ctrl->seq_state = ctrl->seq_next;
}

// ---------------------------------------------------------------------------
int64_t momenta_words(int64_t T) {
  const int64_t n = T + T / 16 + 512;
  return (n + ZB - 1) / ZB * ZB;
}

size_t momenta_scratch_bytes(int64_t T) {
  const int64_t nb = momenta_words(T) / ZB;
  return (size_t)(nb + 2) * sizeof(uint64_t) + 64;
}

// per-CTA jump constants: CTA b's local word 0 is draw word max(0, b*ZB - ZG)
__global__ void zig_block_jump_kernel(uint64_t *bj, int nb) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint64_t k = b == 0 ? 0 : (uint64_t)b * ZB - ZG;  // words
  // pcg32: (A^n, G_n) for n = 2k outputs, G_n = sum_{i<n} A^i (inc-free)
  uint64_t mult = PCG_MULT, plus = 1, acc_mult = 1, acc_plus = 0, delta = 2 * k;
  while (delta > 0) {
    if (delta & 1) { acc_mult *= mult; acc_plus = acc_plus * mult + plus; }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  bj[2 * b] = acc_mult;
  bj[2 * b + 1] = acc_plus;
  bj[2 * nb + b] = minstd_pow(3 * k);
}

int momenta_init(cudaStream_t s, uint64_t *bjump, int64_t T) {
  zig_jump_init_kernel<<<1, 1, 0, s>>>();
  const int nb = (int)(momenta_words(T) / ZB);
  zig_block_jump_kernel<<<(nb + 127) / 128, 128, 0, s>>>(bjump, nb);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

size_t momenta_jump_bytes(int64_t T) { return (size_t)3 * (momenta_words(T) / ZB) * sizeof(uint64_t); }

int launch_momenta(const MomentaBufs &b, int kind, int64_t T, cudaStream_t s, int *launches) {
  const int64_t N = momenta_words(T);
  const int nb = (int)(N / ZB);
  uint64_t *status = (uint64_t *)b.scratch;
  const uint64_t *words = nullptr;
  const int64_t nbuf = N + 64;
  if (kind == PRNG_SFC64) {
    z0_sfc64_kernel<<<1, 1, 0, s>>>(b.ctrl, b.sfc_words, b.sfc_snaps, nbuf);
    words = b.sfc_words;
    (*launches)++;
  }
  const uint64_t *bj = kind == PRNG_MINSTD ? b.bjump + 2 * nb : b.bjump;
  const size_t smem = sizeof(ZigShared);
  switch (kind) {
    case PRNG_PHILOX:
      cudaFuncSetAttribute(zig_kernel<PRNG_PHILOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      zig_kernel<PRNG_PHILOX><<<nb, ZT, smem, s>>>(b.ctrl, words, nbuf, b.normals, T, status, bj, b.dbg);
      break;
    case PRNG_MINSTD:
      cudaFuncSetAttribute(zig_kernel<PRNG_MINSTD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      zig_kernel<PRNG_MINSTD><<<nb, ZT, smem, s>>>(b.ctrl, words, nbuf, b.normals, T, status, bj, b.dbg);
      break;
    case PRNG_PCG32:
      cudaFuncSetAttribute(zig_kernel<PRNG_PCG32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      zig_kernel<PRNG_PCG32><<<nb, ZT, smem, s>>>(b.ctrl, words, nbuf, b.normals, T, status, bj, b.dbg);
      break;
    default:
      cudaFuncSetAttribute(zig_kernel<PRNG_SFC64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      zig_kernel<PRNG_SFC64><<<nb, ZT, smem, s>>>(b.ctrl, words, nbuf, b.normals, T, status, bj, b.dbg);
      break;
  }
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_momenta_advance(const MomentaBufs &b, cudaStream_t s, int *launches) {
  zadvance_kernel<<<1, 1, 0, s>>>(b.ctrl, b.sfc_snaps);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace rsv
