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
#include "rsv_check.h"
#include "theta_dev.cuh"

namespace rsv {


constexpr int ZG = 2 * ZW;             // guard words before a CTA's block (threads 0, 1)
constexpr int ZCH = ZT;                // 8-word chunks staged per CTA: guard, block, look-ahead
constexpr int ZDIRECT = 4096;          // up to this many CTAs: direct predecessor sums
static_assert(ZB == (ZT - 4) * ZW, "block = threads 2..ZT-3");

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

constexpr int ZQ = 512;  // queue of non-fast-path words per CTA (expected ~23)
// shared-memory skews: thread t touches words / normals ~8 apart, so pad two
// (words) / one (normals) doubles per 16 to spread a warp over all banks
#define ZWS(j) ((j) + 2 * ((j) >> 4))
#define ZXS(j) ((j) + ((j) >> 4))

struct ZigShared {
  uint64_t w[ZWS(ZCH * ZW)];  // raw words: local index i <-> draw word b*ZB - ZG + i, at ZWS(i)
  uint64_t ki[256];
  double wi[256];
  double fi[256];
  double xout[ZXS(ZB)];   // the CTA's normals in block order (copy-out staging), at ZXS(j)
  double qx[ZQ];          // queued attempts: normal, (len | acc << 4), word index
  uint8_t qres[ZQ];
  uint16_t qent[ZQ];
  int32_t nq;
  uint32_t edge_lens[ZT / 32][2];  // lanes 30, 31 of each warp: packed attempt lengths
  uint32_t edge_nu[ZT / 32][2];    // and their non-unit-length start masks
  int32_t warp_tot[ZT / 32];
  int32_t warp_exit[ZT / 32];
  uint64_t blk_off;         // exclusive normal offset of this CTA
  int32_t blk;              // dynamic CTA index (ticket)
  int32_t bad;
  int32_t blk_entry;        // entry state of the block's first chunk (thread 2)
  int32_t blk_exit;         // exit state of its last chunk (thread ZT - 3)
  uint32_t epoch;           // this draw's tag in the look-back status words
};

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

__device__ void zig_serial(DevControl *ctrl, const uint64_t *words, int64_t nbuf, double *normals, int64_t T);
__device__ void zig_serial_window(DevControl *ctrl, const ZigWin &win, int64_t nwords);


__device__ __forceinline__ unsigned long long zgt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// zig_kernel: thread t owns the 8 raw words of chunk t of the CTA's window
// (chunks 0, 1: guard = the last 16 words of the previous block; 2..ZT-3:
// the block; ZT-2, ZT-1: look-ahead for attempts that run past the block).
// Words, attempt lengths and candidate normals live in registers; shared
// memory only holds a copy of the words for the rare multi-word attempts.
template <int KIND>
__global__ void __launch_bounds__(ZT, 4) zig_kernel(DevControl *ctrl, const uint64_t *words, int64_t nwords_buf,
                                                 double *normals, int64_t T, uint64_t *status, const uint64_t *bjump,
                                                 int coresident, unsigned long long *dbg, ZigWin win) {
  // window mode (time-sharded momenta, win.out != null): CTA b parses block
  // wb0 + b of the full stream; the first CTA's entry is speculative (no
  // predecessor in this window), the normals go to win.out in stream order
  // and the anchors' counts to win.info (see WinInfo)
  const bool wmode = win.out != nullptr;
#define ZSTAMP(k) \
  do { if (dbg && threadIdx.x == 0) dbg[(size_t)blockIdx.x * 8 + (k)] = zgt(); } while (0)
  ZSTAMP(0);
  extern __shared__ __align__(16) unsigned char zsmem[];
  ZigShared &S = *reinterpret_cast<ZigShared *>(zsmem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // constant data first: tables, per-chunk and (co-resident grid) per-CTA
  // jump constants -- none of it written by the preceding kernel
  for (int i = tid; i < 256; i += ZT) {
    S.ki[i] = g_ki[i];
    S.wi[i] = g_wi[i];
    S.fi[i] = g_fi[i];
  }
  uint64_t jA = 0, jG = 0;
  if (KIND == PRNG_PCG32) { jA = g_jump.pcg_a[tid]; jG = g_jump.pcg_g[tid]; }
  if (KIND == PRNG_MINSTD) jA = g_jump.minstd_a[tid];
  // (one memory round trip fewer on the draw's critical path)
  uint64_t pbA = 0, pbG = 0;
  if (coresident && (KIND == PRNG_PCG32 || KIND == PRNG_MINSTD)) {
    const int bb = (int)blockIdx.x + (int)win.wb0;
    if (KIND == PRNG_PCG32) { pbA = bjump[2 * bb]; pbG = bjump[2 * bb + 1]; }
    else pbA = bjump[bb];
  }
  // scheduling-order ticket: the CTA's block of the draw.  The look-back
  // below only ever waits on smaller tickets, i.e. on CTAs already running,
  // so the draw makes progress whatever the residency (co-resident grids take
  // it too: their spin falls back to the look-back when the grid turns out
  // not to be resident at once, e.g. beside other kernels).  The counter was
  // re-armed by the previous draw's last CTA, which completed before the
  // kernels this one depends on started.
  unsigned ticket = 0;
  if (tid == 0) ticket = atomicAdd(&ctrl->zig_ticket, 1u);
  // launched as a programmatic dependent of the theta kernel (rsv_run_chain):
  // the stream position it advanced is read from here on (no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the trajectory kernel may launch as soon as every CTA of this grid is
  // past this point (it waits for this grid's completion before reading the
  // normals; its own start reads what the theta kernel wrote, complete here)
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctrl->halt) {  // rsv_run_chain stopped: no draw; the ticket is given back
    if (tid == 0) atomicSub(&ctrl->zig_ticket, 1u);
    return;
  }
  if (tid == 0) {
    // a co-resident grid needs no scheduling-order ticket (every CTA runs at
    // once); otherwise the ticket keeps the look-back deadlock-free
    S.blk = (int)ticket;
    S.epoch = ctrl->zig_epoch & 0xffffffu;
    S.bad = 0;
    S.nq = 0;
    if (S.blk == 0) {
      ctrl->t_stamp[4] = ctrl->t_stamp[3];
      ctrl->t_stamp[0] = zgt();
    }
  }
  const StreamState &st = ctrl->stream;
  const uint64_t inc = st.s[1];
  const uint64_t seq = ctrl->seq_state;
  __syncthreads();
  const int b = S.blk;            // ticket: this CTA's block within the draw (or window)
  const int B = b + (int)win.wb0;  // ... within the full stream
  if (coresident && b != (int)blockIdx.x && (KIND == PRNG_PCG32 || KIND == PRNG_MINSTD)) {
    if (KIND == PRNG_PCG32) { pbA = bjump[2 * B]; pbG = bjump[2 * B + 1]; }  // prefetched for blockIdx.x
    else pbA = bjump[B];
  }
  ZSTAMP(1);

  // ---- my 8 raw words, generated into registers
  const int64_t k_t = (int64_t)B * ZB - ZG + (int64_t)tid * ZW;  // draw word of my chunk's first word
  RSV_CHECK(b >= 0 && b < (int)gridDim.x && B >= 0);
  const bool valid = k_t >= 0;                                    // CTA 0 has no guard words
  uint64_t w[ZW];
  uint64_t base = 0;  // pcg: LCG state before output 2*k_t; minstd: x_{3 k_t}
  if (!valid) {
#pragma unroll
    for (int i = 0; i < ZW; i++) w[i] = 0;
  } else if (KIND == PRNG_SFC64) {
#pragma unroll
    for (int i = 0; i < ZW; i += 2) {
      const int64_t k = k_t + i;
      const ulonglong2 v = k + 2 <= nwords_buf ? *reinterpret_cast<const ulonglong2 *>(words + k) : make_ulonglong2(0, 0);
      w[i] = v.x;
      w[i + 1] = v.y;
    }
  } else if (KIND == PRNG_PHILOX) {
    SeqGen g;
    g.init(st, st.pos + (uint64_t)k_t);
#pragma unroll
    for (int i = 0; i < ZW; i++) w[i] = g.next();
  } else {
    // per-CTA jump (bjump, built once per context) composed with the
    // per-chunk jump: CTA b's base word is max(0, b*ZB - ZG)
    const int cc = B == 0 ? tid - ZG / ZW : tid;
    if (KIND == PRNG_PCG32) {
      const uint64_t bA = coresident ? pbA : bjump[2 * B], bG = coresident ? pbG : bjump[2 * B + 1];
      const uint64_t cA = B == 0 ? g_jump.pcg_a[cc] : jA, cG = B == 0 ? g_jump.pcg_g[cc] : jG;
      uint64_t s0 = cA * (bA * seq + bG * inc) + cG * inc;
      base = s0;
#pragma unroll
      for (int i = 0; i < ZW; i++) {
        const uint64_t s1 = s0 * PCG_MULT + inc;
        w[i] = ((uint64_t)pcg_output(s0) << 32) | pcg_output(s1);
        s0 = s1 * PCG_MULT + inc;
      }
    } else {  // MINSTD
      const uint64_t cA = B == 0 ? g_jump.minstd_a[cc] : jA;
      uint64_t x = mod31(cA * mod31((coresident ? pbA : bjump[B]) * seq));
      base = x;
#pragma unroll
      for (int i = 0; i < ZW; i++) {
        const uint64_t xa = mod31(x * MINSTD_A), xb = mod31(xa * MINSTD_A), xc = mod31(xb * MINSTD_A);
        x = xc;
        w[i] = (xa << 33) | (xb << 2) | (xc >> 29);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < ZW; i += 2)
    *reinterpret_cast<ulonglong2 *>(&S.w[ZWS(tid * ZW + i)]) = make_ulonglong2(w[i], w[i + 1]);
  __syncthreads();
  ZSTAMP(2);

  // ---- classify each word as an attempt start (numpy random_standard_normal).
  // Fast path (98.9 % of words) in registers: one table compare.  The rest
  // (wedge: one more word; tail: pairs of words) are queued and evaluated by
  // the whole CTA at once, so the exp / log1p work is not serialised by
  // divergence inside every warp.
  const bool classify = valid && tid < ZT - 2;  // look-ahead chunks are words only
  uint32_t slow = 0;
  if (classify) {
#pragma unroll
    for (int i = 0; i < ZW; i++) {
      const int idx = (int)(w[i] & 0xff);
      const uint64_t rabs = (w[i] >> 9) & 0x000fffffffffffffULL;
      if (!(rabs < S.ki[idx])) slow |= 1u << i;
    }
  }
  const int nslow = __popc(slow);
  int qbase = 0;
  if (nslow) qbase = atomicAdd(&S.nq, nslow);
  {
    uint32_t m = slow;
    int k = 0;
    while (m) {
      const int i = __ffs(m) - 1;
      m &= m - 1;
      if (qbase + k < ZQ) S.qent[qbase + k] = (uint16_t)(tid * ZW + i);
      k++;
    }
  }
  __syncthreads();
  const int nq = S.nq;
  const int nqe = nq < ZQ ? nq : ZQ;
  if (warp < 2) {
    // wedge entries (one more word and an exp each), one per thread of warps 0-1
    for (int q = tid; q < nqe; q += 64) {
      const int j0 = S.qent[q];
      uint64_t r = S.w[ZWS(j0)];
      const int idx = (int)(r & 0xff);
      if (idx == 0) continue;  // exponential tail: evaluated by warps 2.. below
      r >>= 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      const double fr =
          __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | rabs)), 4503599627370496.0);
      double x = __dmul_rn(fr, S.wi[idx]);
      if (r & 1) x = -x;
      const double u = u01(S.w[ZWS(j0 + 1)]);
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(S.fi[idx - 1], S.fi[idx]), u), S.fi[idx]);
      const int a = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x)) ? 1 : 0;
      S.qres[q] = (uint8_t)(2 | (a << 4));
      S.qx[q] = x;
    }
  } else {
    // exponential-tail entries, one warp each: the up to ZMMAX attempts
    // (pairs of words after the entry) are evaluated at once, one log1p per
    // lane, and the first accepted pair is kept -- the result of numpy's
    // sequential loop with one log1p latency instead of 2m
    constexpr int NTW = ZT / 32 - 2;
    int rank = 0;
    for (int base = 0; base < nqe; base += 32) {
      const int ql = base + lane;
      const bool tl = ql < nqe && (S.w[ZWS(S.qent[ql])] & 0xff) == 0;
      uint32_t tm = __ballot_sync(0xffffffffu, tl);
      while (tm) {
        const int q = base + __ffs(tm) - 1;
        tm &= tm - 1;
        if (rank++ % NTW != warp - 2) continue;
        const int j0 = S.qent[q];
        const uint64_t r = S.w[ZWS(j0)] >> 8;
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double lg = 0.0;
        if (lane < 2 * ZMMAX) lg = log1p_ool(-u01(S.w[ZWS(j0 + 1 + lane)]));
        // pair m = lane + 1: xx from word j0 + 2m - 1 (lane 2m - 2), yy from word j0 + 2m
        const double lx = __shfl_sync(0xffffffffu, lg, (2 * lane) & 31);
        const double ly = __shfl_sync(0xffffffffu, lg, (2 * lane + 1) & 31);
        const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R, lx);
        const double yy = -ly;
        const bool ok = lane < ZMMAX && __dadd_rn(yy, yy) > __dmul_rn(xx, xx);
        const uint32_t am = __ballot_sync(0xffffffffu, ok);
        const int first = am ? __ffs(am) - 1 : 0;
        const double xs = __shfl_sync(0xffffffffu, xx, first);
        if (lane == 0) {
          double x;
          int len = 0, a = 0;
          if (am) {
            x = ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xs) : __dadd_rn(RSV_ZIG_R, xs);
            len = 1 + 2 * (first + 1);
            a = 1;
          } else {  // no accept within ZMMAX loops: the exact serial walk redoes the draw
            const double fr =
                __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | rabs)), 4503599627370496.0);
            x = __dmul_rn(fr, S.wi[0]);
            if (r & 1) x = -x;
          }
          S.qres[q] = (uint8_t)(len | (a << 4));
          S.qx[q] = x;
        }
      }
    }
  }
  if (tid == 0 && nq > ZQ) atomicOr(&ctrl->zig_overflow, 1);  // never in practice: exact fallback
  __syncthreads();
  // attempt lengths (nibbles), accepts, non-unit-length starts
  uint32_t lens = 0x11111111u, acc = classify ? (~slow & 0xffu) : 0u, nu = 0;
  {
    uint32_t m = slow;
    int k = 0;
    while (m) {
      const int i = __ffs(m) - 1;
      m &= m - 1;
      const int q = qbase + k < ZQ ? qbase + k : ZQ - 1;
      const uint32_t res = S.qres[q];
      lens = (lens & ~(15u << (4 * i))) | ((res & 15u) << (4 * i));
      acc |= ((res >> 4) & 1u) << i;
      nu |= 1u << i;
      k++;
    }
  }
  ZSTAMP(3);

  // ---- speculative walk: in sync 16 words (two chunks) before my chunk.
  // Unit-length attempts are implicit; only the non-unit starts are visited
  // (usually none in the 24-word window), marking the words they cover.
  if (lane >= 30) {
    S.edge_lens[warp][lane - 30] = lens;
    S.edge_nu[warp][lane - 30] = nu;
  }
  uint32_t lm1 = __shfl_up_sync(0xffffffffu, lens, 1);
  uint32_t lm2 = __shfl_up_sync(0xffffffffu, lens, 2);
  uint32_t nm1 = __shfl_up_sync(0xffffffffu, nu, 1);
  uint32_t nm2 = __shfl_up_sync(0xffffffffu, nu, 2);
  __syncthreads();
  if (warp > 0) {
    if (lane == 0) {
      lm1 = S.edge_lens[warp - 1][1]; lm2 = S.edge_lens[warp - 1][0];
      nm1 = S.edge_nu[warp - 1][1]; nm2 = S.edge_nu[warp - 1][0];
    }
    if (lane == 1) { lm2 = S.edge_lens[warp - 1][1]; nm2 = S.edge_nu[warp - 1][1]; }
  }
  const bool counting = tid >= 2 && tid < ZT - 2;
  int entry = 0, exitst = 0, cnt = 0;
  uint32_t vis = 0, starts = 0;
  int ovf = 0;
  if (counting) {
    uint64_t cov = 0;  // window words inside an attempt that started earlier
    uint32_t m = nm2 | (nm1 << 8) | (nu << 16);
    while (m) {
      const int q = __ffs(m) - 1;
      m &= m - 1;
      if ((cov >> q) & 1) continue;
      const uint32_t src = q < 8 ? lm2 : q < 16 ? lm1 : lens;
      const int L = (int)((src >> (4 * (q & 7))) & 15u);
      if (L == 0) {
        if (q >= 16) ovf = 1;
        continue;
      }
      cov |= ((1ull << (L - 1)) - 1) << (q + 1);
    }
    const uint32_t free_mine = ~(uint32_t)(cov >> 16);
    entry = __ffs(free_mine) - 1;  // <= 14 (an attempt covers at most 14 more words)
    vis = free_mine & 0xffu & (0xffu << entry);
    starts = vis;  // attempt starts in my chunk (accepted or not)
    cnt = __popc(vis & acc);
    vis &= acc;
    exitst = __ffs(~(uint32_t)(cov >> 24)) - 1;
  }
  if (ovf) atomicOr(&ctrl->zig_overflow, 1);
  // verify: my entry == previous chunk's exit; block scan of the counts
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
  if (tid == 2) S.blk_entry = entry;
  if (tid == ZT - 3) S.blk_exit = exitst;
  __syncthreads();
  if (lane == 0 && warp > 0) prev_exit = S.warp_exit[warp - 1];
  if (tid > 2 && counting && prev_exit != entry) S.bad = 1;
  int woff = 0, btot = 0;
#pragma unroll
  for (int q = 0; q < ZT / 32; q++) {
    if (q < warp) woff += S.warp_tot[q];
    btot += S.warp_tot[q];
  }
  const int toff = woff + incl - cnt;  // exclusive offset of my normals in the CTA
  // publish the CTA's count now (look-back status word; with a co-resident
  // grid also the group sum and the release count): the normals below are
  // staged while the other CTAs publish theirs
  unsigned long long *grp = reinterpret_cast<unsigned long long *>(status) + 2 * (gridDim.x + 2);
  if (tid == 0) {
    volatile uint64_t *vst = status;
    vst[b] = zpack(b == 0 ? 2 : 1, S.blk_exit, S.epoch, (uint64_t)btot);
    if (coresident) {
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(grp + (b >> 5)), "l"((uint64_t)btot) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ctrl->zig_pub) : "memory");
    }
  }

  // ---- my normals into the CTA's output staging (block order); the global
  // offset only shifts the coalesced copy-out after the look-back
  if (vis) {
    int o = toff;
#pragma unroll
    for (int i = 0; i < ZW; i++) {
      if ((vis >> i) & 1) {
        double x;
        if ((slow >> i) & 1) {
          const int q = qbase + __popc(slow & ((1u << i) - 1));
          x = S.qx[q < ZQ ? q : ZQ - 1];
        } else {
          uint64_t r = S.w[ZWS(tid * ZW + i)];
          const int idx = (int)(r & 0xff);
          r >>= 8;
          const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
          const double fr =
              __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | rabs)), 4503599627370496.0);
          x = __dmul_rn(fr, S.wi[idx]);
          if (r & 1) x = -x;
        }
        RSV_CHECK(o >= 0 && o < ZB);
        S.xout[ZXS(o)] = x;
        o++;
      }
    }
  }

  ZSTAMP(4);
  // ---- global normal offset of this CTA.  Every CTA publishes its count;
  // when the grid is co-resident, the CTA that publishes last scans all
  // counts once and raises a flag (one cheap poll per waiting CTA instead of
  // hundreds of CTAs re-reading every predecessor).  Otherwise -- or if the
  // flag is late -- a decoupled look-back over the predecessors' counts,
  // which only depends on CTAs with smaller tickets (already running).
  if (warp == 0) {
    const int bexit = S.blk_exit;
    volatile uint64_t *vst = status;
    bool have = false, have_prev = false;
    uint64_t prev_word = 0;
    uint64_t accum = 0;
    if (coresident) {
      // every CTA counted itself into zig_pub (release reduction after its
      // status word and its 32-CTA group sum, above); once the count reaches
      // the grid size (acquire poll) one round of loads -- <= 31 status
      // words and the group sums -- gives the predecessors' total.  The CTA
      // that finishes last resets zig_pub and the group sums.
      bool flag = false;
      for (int it = 0; it < 4096 && !flag; it++) {
        unsigned f = 0;
        if (lane == 0) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(&ctrl->zig_pub) : "memory");
        flag = __shfl_sync(0xffffffffu, f, 0) == gridDim.x;
        if (!flag) __nanosleep(32);
      }
      if (flag) {
        if (dbg && lane == 0) dbg[(size_t)blockIdx.x * 8 + 7] = zgt();  // publication count complete, seen
        __syncwarp();  // the other lanes' loads follow lane 0's acquire
        // one round of independent loads: my group's predecessors' status
        // words (one per lane) and the sums of the groups before mine
        // (the previous CTA's word, needed by the verification below, is in
        // the same round: from its lane, or loaded by lane 0 when b opens a group)
        const int g = b >> 5, j = (g << 5) + lane;
        const bool opens = (b & 31) == 0;
        const unsigned long long *sw = reinterpret_cast<const unsigned long long *>(status);
        const uint64_t v = j < b                            ? __ldcg(sw + j)
                           : (opens && lane == 0 && b > 0) ? __ldcg(sw + b - 1)
                                                           : (uint64_t)S.epoch << 34 | 2ULL << 62;
        uint64_t part = 0;
        for (int k = lane; k < g; k += 32) part += __ldcg(grp + k);
        const bool ok = zready(v, S.epoch);
        part += j < b ? (v & ZCNT) : 0;
        prev_word = __shfl_sync(0xffffffffu, v, opens ? 0 : (b - 1) & 31);
        if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
          accum = part;
          have = true;
          have_prev = b > 0;
        }
      }
    }
    if (!have && b == 0) have = true;
    if (!have) {
      if (gridDim.x <= ZDIRECT) {
        // every CTA sums all its predecessors' aggregates in one round of
        // independent loads (no chain of published prefixes)
        for (;;) {
          uint64_t part = 0;
          bool ok = true;
          for (int base = 0; base < b; base += 256) {
            uint64_t v[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const int j = base + lane + 32 * q;
              v[q] = j < b ? vst[j] : (uint64_t)S.epoch << 34 | 2ULL << 62;
            }
#pragma unroll
            for (int q = 0; q < 8; q++) {
              ok &= zready(v[q], S.epoch);
              part += base + lane + 32 * q < b ? (v[q] & ZCNT) : 0;
            }
          }
          if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            accum = part;
            break;
          }
          __nanosleep(64);
        }
      } else {
        // look back 256 predecessors per round (8 independent loads per lane)
        int hi = b - 1;
        for (;;) {
          uint64_t sv[8];
          for (;;) {
            bool ok = true;
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const int j = hi - lane - 32 * q;
              sv[q] = j >= 0 ? vst[j] : (uint64_t)S.epoch << 34 | 2ULL << 62;  // before CTA 0: empty prefix
            }
#pragma unroll
            for (int q = 0; q < 8; q++) ok &= zready(sv[q], S.epoch);
            if (__all_sync(0xffffffffu, ok)) break;
            __nanosleep(200);  // back off: hundreds of CTAs poll the same lines
          }
          bool done = false;
          uint64_t mine = 0;
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (!done) {
              const unsigned pref = __ballot_sync(0xffffffffu, (sv[q] >> 62) == 2);
              const int stop = pref ? __ffs(pref) - 1 : 32;  // nearest predecessor holding a prefix
              if (lane <= stop) mine += sv[q] & ZCNT;
              done = pref != 0;
            }
          }
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
          accum += mine;
          if (done) break;
          hi -= 256;
        }
        // prefixes are only consumed by the chained look-back of large grids
        // (the direct sums need every CTA's own count to stay in place)
        if (lane == 0) {
          __threadfence();
          vst[b] = zpack(2, bexit, S.epoch, accum + (uint64_t)btot);
        }
      }
    }
    if (lane == 0) {
      S.blk_off = accum;
      if (b == 0) {
        // the draw's first block starts exactly at the stream position; a
        // window's first block is speculative (checked across shards)
        if (B == 0 && S.blk_entry != 0) S.bad = 1;
      } else {  // the previous CTA's exit must equal my block's entry (it has published)
        uint64_t prev = prev_word;
        if (!have_prev) do { prev = vst[b - 1]; } while (!zready(prev, S.epoch));
        if ((int)((prev >> 58) & 15) != S.blk_entry) S.bad = 1;
      }
      if (S.bad) atomicOr(&ctrl->zig_overflow, 2);
    }
  }
  __syncthreads();

  ZSTAMP(5);
  // ---- coalesced copy-out of the CTA's normals; the thread whose normal is
  // the draw's last (index T-1) records where the draw ended in the stream
  const uint64_t boff = S.blk_off;
  if (wmode) {
    RSV_CHECK(boff + (uint64_t)btot <= (uint64_t)win.cap);
    for (int j = tid; j < btot; j += ZT) {
      if (boff + (uint64_t)j < (uint64_t)win.cap) win.out[boff + j] = S.xout[ZXS(j)];
    }
    if (win.nend && vis) {  // where each of my normals' attempts ended
      int o = toff;
      for (int i = 0; i < ZW; i++) {
        if ((vis >> i) & 1) {
          const int L = (int)((lens >> (4 * i)) & 15u);
          if (boff + (uint64_t)o < (uint64_t)win.cap) win.nend[boff + o] = (uint32_t)(k_t - win.w0 + i + L);
          o++;
        }
      }
    }
    // anchors: the thread whose chunk holds the anchor word counts the
    // window's normals before it and finds the first attempt at or after it
    if (counting) {
      const int64_t an[2] = {win.a_lo, win.a_hi};
      for (int q = 0; q < 2; q++) {
        const int64_t a = an[q];
        if (a < k_t || a >= k_t + ZW) continue;
        const int off = (int)(a - k_t);
        const uint32_t before = (1u << off) - 1u;
        const int64_t c = (int64_t)boff + toff + __popc(vis & before);
        const uint32_t m = starts & ~before;
        const int64_t s = m ? k_t + __ffs(m) - 1 : k_t + ZW + exitst;
        if (q == 0) { win.info->cnt_lo = c; win.info->s_lo = s; }
        else { win.info->cnt_hi = c; win.info->s_hi = s; }
      }
    }
    if (tid == ZT - 1 && b == (int)gridDim.x - 1) {
      win.info->n_win = (int64_t)(S.blk_off + (uint64_t)btot);
      win.info->w0 = win.w0;
      if (win.a_hi < 0) { win.info->cnt_hi = (int64_t)(S.blk_off + (uint64_t)btot); win.info->s_hi = -1; }
    }
  } else {
    for (int j = tid; j < btot; j += ZT) {
      if (boff + (uint64_t)j < (uint64_t)T) normals[boff + j] = S.xout[ZXS(j)];
    }
  }
  if (!wmode && vis && boff + (uint64_t)toff <= (uint64_t)T - 1 && (uint64_t)T - 1 < boff + (uint64_t)toff + (uint64_t)cnt) {
    const int rank = (int)((uint64_t)T - 1 - boff - (uint64_t)toff);  // which of my normals
    uint32_t m = vis;
    for (int k = 0; k < rank; k++) m &= m - 1;
    const int i = __ffs(m) - 1;
    const int L = (int)((lens >> (4 * i)) & 15u);
    const int nxt = tid * ZW + i + L;  // local index of the next unread word
    ctrl->zig_used = (uint64_t)((int64_t)b * ZB - ZG + nxt);
    ctrl->u_word = S.w[ZWS(nxt)];
    if (KIND == PRNG_PCG32) ctrl->seq_next = pcg_advance(base, 2 * (uint64_t)(i + L), inc);
    else if (KIND == PRNG_MINSTD) ctrl->seq_next = mod31(minstd_pow(3 * (uint64_t)(i + L)) * base);
  }
  // the last CTA publishes how many normals the parse produced
  if (!wmode && tid == ZT - 1 && b == (int)gridDim.x - 1) ctrl->zig_avail = S.blk_off + (uint64_t)btot;
  ZSTAMP(6);
  // the CTA that finishes last re-arms the bookkeeping and, if the parallel
  // parse could not be trusted (p ~ 1e-12 per word), redoes it serially
  __syncthreads();
  if (tid == 0) {
    // acquire-release count: the CTA's writes (ordered by the barrier) are
    // released, and the last CTA acquires every other CTA's
    unsigned done;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(done) : "l"(&ctrl->zig_done) : "memory");
    if (done == gridDim.x - 1) {
      if (wmode) {
        win.info->err = 0;
        if (ctrl->zig_overflow != 0) zig_serial_window(ctrl, win, (int64_t)gridDim.x * ZB);
      } else if (ctrl->zig_overflow != 0 || ctrl->zig_avail < (uint64_t)T) {
        zig_serial(ctrl, words, nwords_buf, normals, T);
      }
      ctrl->zig_overflow = 0;
      ctrl->zig_ticket = 0;
      ctrl->zig_done = 0;
      ctrl->zig_pub = 0;
      if (coresident) {
        unsigned long long *grp = reinterpret_cast<unsigned long long *>(status) + 2 * (gridDim.x + 2);
        for (int k = 0; k < (int)(gridDim.x + 31) / 32; k++) grp[k] = 0;
      }
      ctrl->zig_epoch = ctrl->zig_epoch + 1;
      ctrl->t_stamp[1] = zgt();
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

// Exact serial walk of a momenta window (fallback of the window mode).  The
// walk assumes an attempt starts at the window's first word: exact for the
// draw's first window (word 0), and -- like the parallel parse's
// speculation -- in step with the true attempt chain within a few words
// elsewhere, long before the first anchor (checked across shards).
__device__ void zig_serial_window(DevControl *ctrl, const ZigWin &win, int64_t nwords) {
  const StreamState st = ctrl->stream;
  const int64_t w_end = win.w0 + nwords;
  uint64_t j = (uint64_t)win.w0;
  int64_t i = 0;
  bool lo_done = false, hi_done = win.a_hi < 0;
  while ((int64_t)j < w_end) {
    const uint64_t j0 = j;  // this attempt's start
    if (!lo_done && (int64_t)j0 >= win.a_lo) { win.info->cnt_lo = i; win.info->s_lo = (int64_t)j0; lo_done = true; }
    if (!hi_done && (int64_t)j0 >= win.a_hi) { win.info->cnt_hi = i; win.info->s_hi = (int64_t)j0; hi_done = true; }
    uint64_t r = word_at(st, st.pos + j);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, g_wi[idx]);
    if (sign) x = -x;
    j++;
    bool acc = rabs < g_ki[idx];
    if (!acc && idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R, glibc_log1p(-u01(word_at(st, st.pos + j))));
        const double yy = -glibc_log1p(-u01(word_at(st, st.pos + j + 1)));
        j += 2;
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          x = ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xx) : __dadd_rn(RSV_ZIG_R, xx);
          acc = true;
          break;
        }
      }
    } else if (!acc) {
      const double u = u01(word_at(st, st.pos + j));
      j++;
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(g_fi[idx - 1], g_fi[idx]), u), g_fi[idx]);
      acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
    }
    if (acc) {
      if (i < win.cap) {
        win.out[i] = x;
        if (win.nend) win.nend[i] = (uint32_t)(j - (uint64_t)win.w0);
      }
      i++;
    }
  }
  win.info->n_win = i;
  win.info->w0 = win.w0;
  if (win.a_hi < 0) { win.info->cnt_hi = i; win.info->s_hi = -1; }
  win.info->err = 2;
  ctrl->err |= 2;
}

// ---- ensemble: one numpy SFC64 stream per chain ------------------------------
// SFC64 has no jump-ahead, so a chain's raw words are inherently sequential.
// A CTA (16 warps) serves 29 chains with a pipeline over 64-word chunks, one
// CTA barrier per round.  The stages are placed so that the generator does
// not share its scheduler's issue slots (scheduler = warp id % 4).  In round r:
//   * warp 0 generates chunk r+2: lane j runs chain j's SFC64 into a 4-chunk
//     shared-memory ring and snapshots the state before each chunk.  The
//     generator is the critical path (64 sequential steps of 64-bit integer
//     work per lane and round), so it has scheduler 0 to itself;
//   * warps 1, 2, 9, 10 classify chunk r+1 (lane = chain; a quarter each):
//     one table compare per word gives the chunk's fast-path mask, the value
//     the word's attempt yields on the fast path (or the wedge) is staged, and
//     the few non-fast words (~1 %) go to the chunk's queue;
//   * warp 6 evaluates chunk r's queue (lane = queued word): the attempt a
//     non-fast word would start -- wedge: one more word and exp; exponential
//     tail: pairs of words and glibc log1p, up to ZE_MMAX loops into the next
//     chunk -- its length, whether it yields a normal, and a tail's value;
//   * warp 5 walks chunk r-1 (lane = chain): the attempts between two
//     non-fast starts are single-word normals, so the walk only stops at the
//     evaluated non-fast starts; it marks the attempts that yield normals and
//     finds where the chain's draw ends;
//   * warps 3, 7, 11, 13, 14, 15 emit chunk r-2 (lanes = words, two chains at
//     a time): each marked attempt's staged value goes to its place, coalesced.
// (Round 1 had one parse warp per chain with lanes = words; the generator
// shared its scheduler with five of them and every word was classified by a
// whole-warp pass: ~190 us for 4096 x 4096 against ~125 us now.)
// The draw is numpy's random_standard_normal on SFC64(SeedSequence([seed,
// c])) exactly; the stream states after the draw's words and after the
// Metropolis uniform are both kept for the trajectory kernel's decision.
constexpr int ZE_G = 29;      // chains per CTA (4096 chains = 142 CTAs, one wave)
constexpr int ZE_CH = 64;     // words per chunk
constexpr int ZE_RING = 256;  // ring words per chain (4 chunks)
constexpr int ZE_RS = ZE_RING + 1;  // padded rows: lanes of a chain-parallel access hit distinct banks
constexpr int ZE_XS = ZE_CH + 1;
constexpr int ZE_NT = 512;
constexpr int ZE_NE = 6;      // emitting warps
constexpr int ZE_QMAX = 512;  // queued non-fast words per chunk (expected ~20)
constexpr int ZE_MMAX = 30;   // tail loops resolvable inside the ring window
__device__ __forceinline__ int ze_emitter(int warp) {  // emitter index, -1: another role
  return (warp & 3) == 3 ? warp >> 2 : warp == 13 ? 4 : warp == 14 ? 5 : -1;
}
__device__ __forceinline__ int ze_classifier(int warp) {  // quarter of a chunk, -1: another role
  return warp == 1 ? 0 : warp == 2 ? 1 : warp == 9 ? 2 : warp == 10 ? 3 : -1;
}
__device__ __forceinline__ uint64_t ze_low(int n) { return n >= 64 ? ~0ull : ((1ull << n) - 1); }

// cycle counter that memory operations are not moved across (stamps only)
__device__ __forceinline__ long long ze_clk() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}

struct ZEnsShared {
  uint64_t ring[ZE_G * ZE_RS];
  uint64_t snap[ZE_G][4][4];     // generator state before each chunk (by chunk & 3)
  ulonglong2 kw[256];            // (ki, wi bits): one 16-byte lookup per classified word
  double wi[256], fi[256];
  double xs[4][ZE_G][ZE_XS];     // by chunk & 3: the value an attempt at each word yields
  uint64_t vis[2][ZE_G];         // by chunk & 1: attempt starts that yield a normal
  uint16_t fast[4][ZE_G][4];     // fast-path words
  uint32_t eacc[4][ZE_G][2];     // non-fast words whose attempt yields a normal
  int8_t elen[4][ZE_G][ZE_CH];   // ... their attempt's length in words (0: beyond the window)
  uint16_t qe[4][ZE_QMAX];       // queued non-fast words: chain << 6 | word
  int32_t qn[4];
  int32_t n0e[2][ZE_G], wr[2][ZE_G];  // by chunk & 1: normals before the chunk, the chunk walked
  int32_t n0[ZE_G], carry[ZE_G], done[ZE_G], ovf[ZE_G];
  int32_t ndone, last_round;
};

__global__ void __launch_bounds__(ZE_NT, 1) zig_ens_kernel(EnsChain *E, double *normals, int64_t Tc, int C,
                                                         unsigned long long *dbg, int advance, const int32_t *halt) {
  if (halt && *halt) return;  // blocked momenta of a stopped rsv_run_chain: streams untouched
  extern __shared__ __align__(16) unsigned char zesmem[];
  ZEnsShared &S = *reinterpret_cast<ZEnsShared *>(zesmem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.x * ZE_G;
  const int nch = min(ZE_G, C - c0);
  for (int i = tid; i < 256; i += ZE_NT) {
    S.kw[i] = make_ulonglong2(g_ki[i], (unsigned long long)__double_as_longlong(g_wi[i]));
    S.wi[i] = g_wi[i];
    S.fi[i] = g_fi[i];
  }
  if (tid < ZE_G) {
    S.n0[tid] = 0;
    S.carry[tid] = 0;
    S.done[tid] = tid >= nch;
    S.ovf[tid] = 0;
    S.wr[0][tid] = S.wr[1][tid] = -1;
  }
  if (tid < 4) S.qn[tid] = 0;
  if (tid == 0) {
    S.ndone = ZE_G - nch;
    S.last_round = -2;
  }
  // generator state (warp 0, lane j = chain c0 + j)
  uint64_t g[4] = {0, 0, 0, 0};
  const bool gen = warp == 0 && lane < nch;
  if (gen)
    for (int k = 0; k < 4; k++) g[k] = E[c0 + lane].st[k];
  auto gen_chunk = [&](int m) {
    uint64_t *row = S.ring + lane * ZE_RS;
    for (int k = 0; k < 4; k++) S.snap[lane][m & 3][k] = g[k];
    const int o = (m * ZE_CH) & (ZE_RING - 1);
#pragma unroll 8
    for (int k = 0; k < ZE_CH; k++) row[o + k] = sfc64_next(g);
  };
  // quarter h of chunk m (lane = chain): fast-path mask and values, the other words queued
  auto classify = [&](int m, int h) {
    if (lane >= nch || S.done[lane]) return;
    // words in, values computed, values out: no staging store between two
    // words' loads (the compiler cannot tell the ring, the tables and the
    // staging area apart, and would serialise every word)
    const uint64_t *row = S.ring + lane * ZE_RS + ((m * ZE_CH + h * 16) & (ZE_RING - 1));
    uint64_t wv[16];
#pragma unroll
    for (int k = 0; k < 16; k++) wv[k] = row[k];
    double xv[16];
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      uint64_t w = wv[k];
      const int idx = (int)(w & 0xff);
      w >>= 8;
      const uint64_t rabs = (w >> 1) & 0x000fffffffffffffULL;
      const double fr =
          __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | rabs)), 4503599627370496.0);
      const ulonglong2 kw = S.kw[idx];
      const double x = __dmul_rn(fr, __longlong_as_double((long long)kw.y));
      xv[k] = (w & 1) ? -x : x;
      bits |= (uint32_t)(rabs < kw.x) << k;
    }
    double *xr = S.xs[m & 3][lane] + h * 16;
#pragma unroll
    for (int k = 0; k < 16; k++) xr[k] = xv[k];
    S.fast[m & 3][lane][h] = (uint16_t)bits;
    if (h < 2) S.eacc[m & 3][lane][h] = 0;
    for (uint32_t sl = ~bits & 0xffffu; sl; sl &= sl - 1) {
      const int e = atomicAdd(&S.qn[m & 3], 1);
      if (e < ZE_QMAX) S.qe[m & 3][e] = (uint16_t)((lane << 6) | (h * 16 + __ffs(sl) - 1));
      else S.ovf[lane] = 1;  // never in practice: the draw is flagged (the proposal is rejected)
    }
  };
  // the attempts the queued words of chunk m would start (lane = queued word)
  auto evaluate = [&](int m) {
    const int n = min(S.qn[m & 3], ZE_QMAX);
    const int64_t base = (int64_t)m * ZE_CH;
    for (int e = lane; e < n; e += 32) {
      const int jq = S.qe[m & 3][e], j = jq >> 6, q = jq & 63;
      RSV_CHECK(j < nch);
      const uint64_t *row = S.ring + j * ZE_RS;
      uint64_t w = row[(base + q) & (ZE_RING - 1)];
      const int idx = (int)(w & 0xff);
      w >>= 8;
      const uint64_t rabs = (w >> 1) & 0x000fffffffffffffULL;
      int L = 0;
      bool acc = false;
      if (idx == 0) {  // exponential tail
        for (int mm = 1; mm <= ZE_MMAX; mm++) {
          const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R,
                                      glibc_log1p(-u01(row[(base + q + 2 * mm - 1) & (ZE_RING - 1)])));
          const double yy = -glibc_log1p(-u01(row[(base + q + 2 * mm) & (ZE_RING - 1)]));
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
            S.xs[m & 3][j][q] = ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xx) : __dadd_rn(RSV_ZIG_R, xx);
            L = 1 + 2 * mm;
            acc = true;
            break;
          }
        }
      } else {  // wedge (the staged value stands)
        const double fr =
            __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | rabs)), 4503599627370496.0);
        const double x = __dmul_rn(fr, S.wi[idx]);
        const double u = u01(row[(base + q + 1) & (ZE_RING - 1)]);
        const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(S.fi[idx - 1], S.fi[idx]), u), S.fi[idx]);
        acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
        L = 2;
      }
      S.elen[m & 3][j][q] = (int8_t)L;
      if (acc) atomicOr(&S.eacc[m & 3][j][q >> 5], 1u << (q & 31));
    }
  };
  // the attempt chain through chunk m (lane = chain)
  auto walk = [&](int m, int r) {
    const int j = lane;
    if (j >= nch || S.done[j]) return;
    const uint64_t fm = *reinterpret_cast<const uint64_t *>(S.fast[m & 3][j]);
    const uint64_t ea = (uint64_t)S.eacc[m & 3][j][0] | ((uint64_t)S.eacc[m & 3][j][1] << 32);
    const int64_t base = (int64_t)m * ZE_CH;
    const int64_t n0 = S.n0[j], need = Tc - n0;  // >= 1 normals still to draw
    int pos = S.carry[j];
    uint64_t vis = 0;
    int64_t used = -1;  // the draw's words, once it ends in this chunk
    bool ovf = false;
    while (pos < ZE_CH) {
      const uint64_t from = ~0ull << pos;
      const uint64_t slow = ~fm & from;
      const int q = slow ? __ffsll((long long)slow) - 1 : ZE_CH;
      const int have = __popcll(vis);
      if (have + (q - pos) >= need) {  // the draw ends at a single-word attempt in [pos, q)
        const int qe = pos + (int)(need - have) - 1;
        vis |= from & ze_low(qe + 1);
        used = base + qe + 1;
        break;
      }
      vis |= from & ze_low(q);
      if (q >= ZE_CH) {
        pos = ZE_CH;
        break;
      }
      int L = S.elen[m & 3][j][q];
      if (L <= 0) {  // a tail beyond the ring window (never in practice): flagged
        L = 1 + 2 * ZE_MMAX;
        ovf = true;
      }
      if ((ea >> q) & 1) {
        vis |= 1ull << q;
        if (have + (q - pos) + 1 >= need) {
          used = base + q + L;
          break;
        }
      }
      pos = q + L;
    }
    S.vis[m & 1][j] = vis;
    S.n0e[m & 1][j] = (int32_t)n0;
    S.wr[m & 1][j] = m;
    RSV_CHECK(pos <= 2 * ZE_CH && (used < 0 || (used > base && used <= base + 2 * ZE_CH)));
    if (used >= 0) {
      EnsChain &ec = E[c0 + j];
      const int mc = (int)(used / ZE_CH);
      uint64_t st[4];
      for (int k = 0; k < 4; k++) st[k] = S.snap[j][mc & 3][k];
      for (int64_t t = (int64_t)mc * ZE_CH; t < used; t++) sfc64_next(st);
      for (int k = 0; k < 4; k++) ec.st_used[k] = st[k];
      ec.used = (uint64_t)used;
      ec.u_word = sfc64_next(st);
      for (int k = 0; k < 4; k++) ec.st_used1[k] = st[k];
      if (advance)  // blocked momenta streams: no uniform is ever drawn from them
        for (int k = 0; k < 4; k++) ec.st[k] = ec.st_used[k];
      ec.overflow = (S.ovf[j] | (int)ovf) ? 1 : 0;
      S.done[j] = 1;
      atomicAdd(&S.ndone, 1);
      atomicMax(&S.last_round, r);
    } else {
      S.n0[j] = (int32_t)(n0 + __popcll(vis));
      S.carry[j] = pos - ZE_CH;
      S.ovf[j] |= (int)ovf;
    }
  };
  // the normals of chunk m (lanes = words; two chains at a time, all loads
  // before the stores)
  const int em = ze_emitter(warp);
  auto emit = [&](int m) {
    for (int j0 = em; j0 < nch; j0 += 2 * ZE_NE) {
      uint64_t vis[2];
      int64_t n0[2];
      double xv[2][2];
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const int j = min(j0 + t * ZE_NE, nch - 1);
        const bool ok = j0 + t * ZE_NE < nch && S.wr[m & 1][j] == m;
        vis[t] = ok ? S.vis[m & 1][j] : 0ull;
        n0[t] = S.n0e[m & 1][j];
#pragma unroll
        for (int h = 0; h < 2; h++) xv[t][h] = S.xs[m & 3][j][h * 32 + lane];
      }
#pragma unroll
      for (int t = 0; t < 2; t++) {
        double *out = normals + (int64_t)(c0 + j0 + t * ZE_NE) * Tc + n0[t];
        const int64_t lim = Tc - n0[t];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int q = h * 32 + lane;
          const int o = __popcll(vis[t] & ze_low(q));
          if (((vis[t] >> q) & 1) && o < lim) out[o] = xv[t][h];
        }
      }
    }
  };
  if (gen) {
    gen_chunk(0);
    gen_chunk(1);
  }
  __syncthreads();
  const int cq = ze_classifier(warp);
  if (cq >= 0) classify(0, cq);
  __syncthreads();
  long long cy_work = 0, cy_wait = 0, t_a = 0;
  int rounds = 0;
  const unsigned long long t_loop = dbg ? zgt() : 0ull;
  for (int r = 0;; r++) {
    // chains still drawing, or the last chunk walked still to be emitted
    if (S.ndone >= ZE_G && S.last_round + 1 < r) break;
    rounds++;
    if (dbg) t_a = ze_clk();
    if (warp == 0) {
      if (lane == 0) S.qn[(r + 2) & 3] = 0;  // chunk r+2's queue (its previous user, chunk r-2, is done)
      if (gen) gen_chunk(r + 2);
    } else if (cq >= 0) {
      classify(r + 1, cq);
    } else if (warp == 6) {
      evaluate(r);
    } else if (warp == 5) {
      if (r >= 1) walk(r - 1, r);
    } else if (em >= 0 && r >= 2) {
      emit(r - 2);
    }
    if (dbg) {
      const long long t_b = ze_clk();
      cy_work += t_b - t_a;
      __syncthreads();
      cy_wait += ze_clk() - t_b;
    } else {
      __syncthreads();
    }
  }
  // stamps: generator work / wait cycles, rounds, walk work / wait cycles,
  // and %globaltimer at entry, loop start, exit
  if (dbg && lane == 0 && warp == 0) {
    unsigned long long *d = dbg + (size_t)blockIdx.x * 8;
    d[0] = cy_work;
    d[4] = rounds;
    d[3] = t_loop;
    d[7] = zgt();
  }
  if (dbg && lane == 0 && (warp == 1 || warp == 3 || warp == 5 || warp == 6))  // classify, emit, walk, evaluate
    dbg[(size_t)blockIdx.x * 8 + (warp == 1 ? 1 : warp == 3 ? 2 : warp)] = cy_work;
}

int launch_momenta_ens(EnsChain *ens, double *normals, int64_t Tc, int n_chains, cudaStream_t s, int *launches,
                       unsigned long long *dbg, int advance, const int32_t *halt) {
  const size_t smem = sizeof(ZEnsShared);
  cudaFuncSetAttribute(zig_ens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  zig_ens_kernel<<<(n_chains + ZE_G - 1) / ZE_G, ZE_NT, smem, s>>>(ens, normals, Tc, n_chains, dbg, advance, halt);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---- run_chain on the device: the theta draws of one sweep -------------------
// One thread, after the proposal's Metropolis step: the five full
// conditionals of sampler.py:170-272 in run_chain's order (:339-344) from the
// statistics of the kept path, drawing from the same raw-word stream exactly
// as numpy's Generator would (ziggurat normals, next_double, and numpy's
// Marsaglia-Tsang gamma), every product / quotient rounded like the host's
// Python floats (no contraction).  Only exp / log differ from glibc (<= 1 ulp):
// a draw flips only if a uniform lands within an ulp of its threshold.
// The theta kernel is one long sequential chain executed by a single
// thread: its time is instruction-fetch latency, not arithmetic, so the
// generator, the ziggurat, log1p and the gamma sampler are out-of-line
// functions (one copy of each stays hot in the instruction cache) instead of
// being inlined at every call site.
constexpr int TH_NT = 256;
__global__ void __launch_bounds__(TH_NT) theta_sweep_kernel(DevControl *C, DevParams *P, TrajConsts *K, DevRun *R,
                                                            DevPrior pr, double dt, int64_t T,
                                                            const uint64_t *sfc_snaps) {
  // the draws are one sequential stream (thread 0); the CTA only stages the
  // ziggurat tables in shared memory so no draw waits on a global load
  __shared__ uint64_t s_ki[256];
  __shared__ double s_wi[256], s_fi[256];
  // programmatic dependent launch (rsv_run_chain): the next sweep's momenta
  // kernel may launch now; this kernel reads the trajectory's results only
  // after griddepcontrol.wait (both no-ops for a plain launch)
  asm volatile("griddepcontrol.launch_dependents;");
  for (int i = threadIdx.x; i < 256; i += TH_NT) {
    s_ki[i] = g_ki[i];
    s_wi[i] = g_wi[i];
    s_fi[i] = g_fi[i];
  }
  __syncthreads();
  // warp 0 runs the draws, every lane on the same values (theta_dev.cuh:
  // lane-parallel transcendentals); the identical stores of its lanes merge
  if (threadIdx.x >= 32 || blockIdx.x) return;
  (void)sfc_snaps;
  // while the trajectory kernel finishes: the draws at the position the
  // proposal will most likely leave the stream at -- after the momenta's
  // words (seq_next, written by the momenta kernel) and the uniform; the
  // chain checks the actual state before it uses any of them
  ThetaSpec sp;
  const int kind = C->stream.kind;
  const bool speculate = kind == PRNG_PCG32 || kind == PRNG_MINSTD;
  if (speculate) {
    const uint64_t inc = C->stream.s[1];
    uint64_t q = C->seq_next;
    if (kind == PRNG_PCG32) { q = q * PCG_MULT + inc; q = q * PCG_MULT + inc; }
    else q = mod31(mod31(mod31(q * MINSTD_A) * MINSTD_A) * MINSTD_A);
    theta_spec_fill(sp, kind, q, inc, __dadd_rn(pr.var_shape, __dmul_rn(0.5, (double)T)), s_ki, s_wi, s_fi);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  theta_sweep_body(C, P, K, R, pr, dt, T, s_ki, s_wi, s_fi, speculate ? &sp : nullptr);
}

int launch_theta_sweep(DevControl *ctrl, DevParams *prm, TrajConsts *kdev, DevRun *run, DevPrior prior, double dt,
                       int64_t T, const uint64_t *sfc_snaps, cudaStream_t s, int *launches, int pdl) {
  if (pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(TH_NT);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, theta_sweep_kernel, ctrl, prm, kdev, run, prior, dt, T, sfc_snaps) != cudaSuccess)
      return -1;
    (*launches)++;
    return 0;
  }
  theta_sweep_kernel<<<1, TH_NT, 0, s>>>(ctrl, prm, kdev, run, prior, dt, T, sfc_snaps);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
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

size_t momenta_scratch_bytes(int64_t T) {  // status words + CTA prefixes + 32-CTA group sums
  const int64_t nb = momenta_words(T) / ZB;
  return (size_t)(2 * (nb + 2) + (nb + 31) / 32 + 1) * sizeof(uint64_t) + 64;
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
int64_t momenta_blocks(int64_t T) { return momenta_words(T) / ZB; }

template <int KIND>
static void launch_zig(const MomentaBufs &b, const uint64_t *words, int64_t nbuf, int64_t T, uint64_t *status,
                       const uint64_t *bj, int nb, size_t smem, cudaStream_t s) {
  cudaFuncSetAttribute(zig_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(zig_kernel<KIND>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  // can every CTA of the draw be resident at once?  (flag-mode prefixes)
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zig_kernel<KIND>, ZT, smem);
  // (small grids poll their few predecessors directly: cheaper than the flag)
  const int coresident = nb >= 64 && nb <= per_sm * sms ? 1 : 0;
  if (b.pdl) {  // programmatic dependent of the preceding kernel (its griddepcontrol.wait orders the reads)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(ZT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, zig_kernel<KIND>, b.ctrl, words, nbuf, b.normals, T, status, bj, coresident, b.dbg, ZigWin{});
    return;
  }
  zig_kernel<KIND><<<nb, ZT, smem, s>>>(b.ctrl, words, nbuf, b.normals, T, status, bj, coresident, b.dbg, ZigWin{});
}

// Blocked layout (config 5): the momenta come from one SFC64 stream per block
// of sites; the main stream only supplies the Metropolis uniform (and the
// theta draws), so the proposal "uses" no main-stream words for momenta.
__global__ void main_uniform_kernel(DevControl *ctrl, uint64_t *snaps, int64_t T) {
  if (threadIdx.x || blockIdx.x || ctrl->halt) return;
  const StreamState st = ctrl->stream;
  ctrl->zig_used = 0;
  ctrl->zig_avail = (uint64_t)T;
  if (st.kind == PRNG_SFC64) {
    uint64_t q[4] = {st.s[0], st.s[1], st.s[2], st.s[3]};
    for (int k = 0; k < 4; k++) snaps[k] = q[k];  // state at the stream position (Metropolis rewinds from here)
    ctrl->u_word = sfc64_next(q);
  } else {
    ctrl->u_word = word_at(st, st.pos);
    ctrl->seq_next = ctrl->seq_state;
  }
}

int launch_momenta(const MomentaBufs &b, int kind, int64_t T, cudaStream_t s, int *launches) {
  if (b.blocks) {
    if (launch_momenta_ens(b.blocks, b.normals, b.block_len, b.n_blocks, s, launches, nullptr, 1, &b.ctrl->halt))
      return -1;
    main_uniform_kernel<<<1, 32, 0, s>>>(b.ctrl, b.sfc_snaps, T);
    (*launches)++;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
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
  // (the jump tables may cover more blocks than this draw: time-sharded contexts build them for windows)
  const uint64_t *bj = kind == PRNG_MINSTD ? b.bjump + 2 * (b.bjump_blocks ? b.bjump_blocks : nb) : b.bjump;
  const size_t smem = sizeof(ZigShared);
  switch (kind) {
    case PRNG_PHILOX: launch_zig<PRNG_PHILOX>(b, words, nbuf, T, status, bj, nb, smem, s); break;
    case PRNG_MINSTD: launch_zig<PRNG_MINSTD>(b, words, nbuf, T, status, bj, nb, smem, s); break;
    case PRNG_PCG32: launch_zig<PRNG_PCG32>(b, words, nbuf, T, status, bj, nb, smem, s); break;
    default: launch_zig<PRNG_SFC64>(b, words, nbuf, T, status, bj, nb, smem, s); break;
  }
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Window mode (time-sharded momenta): parse blocks [w.wb0, w.wb0 + nb) of the
// stream at the context's position into w.out, anchors into w.info.
int launch_momenta_window(const MomentaBufs &b, int kind, const ZigWin &w, int nb, cudaStream_t s, int *launches) {
  if (kind == PRNG_SFC64 || nb < 1) return -1;  // sequential generator: no window without the prefix
  uint64_t *status = (uint64_t *)b.scratch;
  const uint64_t *bj = kind == PRNG_MINSTD ? b.bjump + 2 * b.bjump_blocks : b.bjump;
  const size_t smem = sizeof(ZigShared);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ZT, smem);
    const int coresident = nb >= 64 && nb <= per_sm * sms ? 1 : 0;
    kern<<<nb, ZT, smem, s>>>(b.ctrl, nullptr, 0, nullptr, 0, status, bj, coresident, b.dbg, w);
  };
  switch (kind) {
    case PRNG_PHILOX: go(zig_kernel<PRNG_PHILOX>); break;
    case PRNG_MINSTD: go(zig_kernel<PRNG_MINSTD>); break;
    default: go(zig_kernel<PRNG_PCG32>); break;
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
