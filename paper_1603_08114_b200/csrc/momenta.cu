// momenta.cu -- bit-exact numpy momenta on the GPU.
//
// Replaces sampler.py:136-141 refresh_momenta = rng.standard_normal(T) with
// numpy's 256-layer ziggurat (random_standard_normal, numpy 2.3.5).  A
// ziggurat draw consumes a variable number of raw words (1 for the 98.9 %
// fast path, 2 for a wedge test, 1 + 2m for m exponential-tail loops), so
// normal i's position in the raw stream depends on every earlier draw.  We
// parse that in parallel:
//
//   Z1  every raw word k is classified as if an attempt started there:
//       (len_k, acc_k, x_k).  The parse is the automaton over states
//       s in {0..15} = "words still owed to the running attempt"; word k
//       maps s=0 -> len_k - 1 and s>0 -> s-1, emitting x_k when s=0 and
//       acc_k.  Each thread summarises its 8 words as a map
//       (exit state, #normals) for all 16 entry states by a backward DP;
//       blocks compose the 256 thread maps in a shared-memory tree.
//   Z2  one CTA scans the block maps from state 0 -> each block's entry
//       state and output offset.
//   Z3  each block re-derives its thread maps, runs the tree down from its
//       entry state and writes its normals to their global slots; the
//       thread that emits normal T-1 records how many words were used.
//
// Attempts needing more than ZMMAX tail loops (p ~ 1e-12 per word) set a
// flag and Z3 falls back to a serial walk, so results stay exact.
#include <math.h>

#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

__device__ const uint64_t g_ki[256] = RSV_KI_DOUBLE_INIT;
__device__ const double g_wi[256] = RSV_WI_DOUBLE_INIT;
__device__ const double g_fi[256] = RSV_FI_DOUBLE_INIT;

struct ZigTables {
  uint64_t ki[256];
  double wi[256];
};

__device__ __forceinline__ uint64_t look_word(const StreamState &st, const uint64_t *words, uint64_t pos0, uint64_t j) {
  return words ? words[j] : word_at(st, pos0 + j);
}

// Classify raw word j (relative to the draw's first word) as the first word
// of an attempt of numpy's random_standard_normal.
__device__ __forceinline__ void zig_classify(uint64_t r, uint64_t j, const StreamState &st, const uint64_t *words,
                                             uint64_t pos0, const uint64_t *ki, const double *wi, int mmax,
                                             int &len, int &acc, double &x) {
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const int sign = (int)(r & 0x1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  x = __dmul_rn((double)rabs, wi[idx]);
  if (sign) x = -x;
  if (rabs < ki[idx]) { len = 1; acc = 1; return; }
  if (idx == 0) {
    for (int m = 1; m <= mmax; m++) {
      const double xx = __dmul_rn(RSV_ZIG_NEG_INV_R, glibc_log1p(-u01(look_word(st, words, pos0, j + 2 * m - 1))));
      const double yy = -glibc_log1p(-u01(look_word(st, words, pos0, j + 2 * m)));
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        x = ((rabs >> 8) & 0x1) ? -__dadd_rn(RSV_ZIG_R, xx) : __dadd_rn(RSV_ZIG_R, xx);
        len = 1 + 2 * m;
        acc = 1;
        return;
      }
    }
    len = 0;  // overflow: resolved by the serial fallback
    acc = 0;
    return;
  }
  const double u = u01(look_word(st, words, pos0, j + 1));
  const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(g_fi[idx - 1], g_fi[idx]), u), g_fi[idx]);
  acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x)) ? 1 : 0;
  len = 2;
}

// Parse element over entry states 0..15: exit state (nibbles) + counts.
template <typename C>
struct ZElem {
  uint64_t exit;
  C cnt[ZS];
};

template <typename C, typename D>
__device__ __forceinline__ void zcompose(const ZElem<C> &f, const ZElem<D> &g, ZElem<C> &out) {
  uint64_t ex = 0;
  C cn[ZS];
#pragma unroll
  for (int e = 0; e < ZS; e++) {
    const int m = (int)((f.exit >> (4 * e)) & 15);
    ex |= ((g.exit >> (4 * m)) & 15ULL) << (4 * e);
    cn[e] = (C)(f.cnt[e] + (C)g.cnt[m]);
  }
  out.exit = ex;
#pragma unroll
  for (int e = 0; e < ZS; e++) out.cnt[e] = cn[e];
}

// Thread-level element from 8 (len, acc) pairs packed as nibbles / bits.
__device__ __forceinline__ void zthread_elem(uint32_t lens, uint32_t accs, ZElem<uint16_t> &el) {
  uint32_t exp_ = 0, cnp = 0;
#pragma unroll
  for (int p = ZW - 1; p >= 0; p--) {
    const int L = (int)((lens >> (4 * p)) & 15);
    const int a = (int)((accs >> p) & 1);
    const int nx = p + (L ? L : 1);
    int ex, cn;
    if (nx >= ZW) { ex = nx - ZW; cn = a; }
    else { ex = (int)((exp_ >> (4 * nx)) & 15); cn = a + (int)((cnp >> (4 * nx)) & 15); }
    exp_ |= (uint32_t)ex << (4 * p);
    cnp |= (uint32_t)cn << (4 * p);
  }
  uint64_t ex = 0;
#pragma unroll
  for (int e = 0; e < ZS; e++) {
    const uint64_t v = e < ZW ? ((exp_ >> (4 * e)) & 15) : (uint64_t)(e - ZW);
    ex |= v << (4 * e);
    el.cnt[e] = e < ZW ? (uint16_t)((cnp >> (4 * e)) & 15) : (uint16_t)0;
  }
  el.exit = ex;
}

__device__ __forceinline__ void load_tables(ZigTables &t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.ki[i] = g_ki[i];
    t.wi[i] = g_wi[i];
  }
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

// Z1: classify words [0, nb*ZB) of the draw, block maps -> agg.
__global__ void __launch_bounds__(ZT) z1_kernel(DevControl *ctrl, const uint64_t *words, double *xs,
                                                uint8_t *meta, ZElem<uint16_t> *agg) {
  __shared__ ZigTables tab;
  __shared__ ZElem<uint16_t> nodes[2 * ZT];
  load_tables(tab);
  const StreamState st = ctrl->stream;
  const uint64_t pos0 = st.pos;
  const uint64_t j0 = ((uint64_t)blockIdx.x * ZT + threadIdx.x) * ZW;
  uint64_t w[ZW];
  if (words) {
#pragma unroll
    for (int i = 0; i < ZW; i++) w[i] = words[j0 + i];
  } else {
    SeqGen g;
    g.init(st, pos0 + j0);
#pragma unroll
    for (int i = 0; i < ZW; i++) w[i] = g.next();
  }
  __syncthreads();
  uint32_t lens = 0, accs = 0;
  uint64_t m8 = 0;
  int ovf = 0;
  double xv[ZW];
#pragma unroll
  for (int i = 0; i < ZW; i++) {
    int len, acc;
    zig_classify(w[i], j0 + i, st, words, pos0, tab.ki, tab.wi, ZMMAX, len, acc, xv[i]);
    lens |= (uint32_t)len << (4 * i);
    accs |= (uint32_t)acc << i;
    m8 |= (uint64_t)(len | (acc << 7)) << (8 * i);
    ovf |= (len == 0);
  }
  *reinterpret_cast<uint64_t *>(meta + j0) = m8;
#pragma unroll
  for (int i = 0; i < ZW; i += 2) *reinterpret_cast<double2 *>(xs + j0 + i) = make_double2(xv[i], xv[i + 1]);
  if (ovf) atomicExch(&ctrl->zig_overflow, 1);
  ZElem<uint16_t> el;
  zthread_elem(lens, accs, el);
  nodes[ZT + threadIdx.x] = el;
  __syncthreads();
  for (int width = ZT / 2; width >= 1; width >>= 1) {
    if (threadIdx.x < width) {
      const int i = width + threadIdx.x;
      ZElem<uint16_t> o;
      zcompose(nodes[2 * i], nodes[2 * i + 1], o);
      nodes[i] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) agg[blockIdx.x] = nodes[1];
}

struct ZEntry {
  uint32_t state;
  uint32_t pad;
  uint64_t offset;
};

// Z2: scan block maps from (state 0, offset 0) -> per-block entries.
__global__ void __launch_bounds__(Z2T) z2_kernel(DevControl *ctrl, const ZElem<uint16_t> *agg, ZEntry *entries,
                                                 int nb) {
  __shared__ ZElem<uint32_t> nodes[2 * Z2T];
  __shared__ uint32_t in_state[2 * Z2T];
  __shared__ uint64_t in_off[2 * Z2T];
  const int per = (nb + Z2T - 1) / Z2T;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  ZElem<uint32_t> el;
  el.exit = 0xFEDCBA9876543210ULL;  // identity
#pragma unroll
  for (int e = 0; e < ZS; e++) el.cnt[e] = 0;
  for (int b = b0; b < b1; b++) {
    ZElem<uint16_t> g = agg[b];
    zcompose(el, g, el);
  }
  nodes[Z2T + threadIdx.x] = el;
  __syncthreads();
  for (int width = Z2T / 2; width >= 1; width >>= 1) {
    if (threadIdx.x < width) {
      const int i = width + threadIdx.x;
      ZElem<uint32_t> o;
      zcompose(nodes[2 * i], nodes[2 * i + 1], o);
      nodes[i] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { in_state[1] = 0; in_off[1] = 0; }
  __syncthreads();
  for (int width = 1; width < Z2T; width <<= 1) {
    if (threadIdx.x < width) {
      const int i = width + threadIdx.x;
      const uint32_t s = in_state[i];
      const uint64_t o = in_off[i];
      in_state[2 * i] = s;
      in_off[2 * i] = o;
      in_state[2 * i + 1] = (uint32_t)((nodes[2 * i].exit >> (4 * s)) & 15);
      in_off[2 * i + 1] = o + nodes[2 * i].cnt[s];
    }
    __syncthreads();
  }
  uint32_t s = in_state[Z2T + threadIdx.x];
  uint64_t o = in_off[Z2T + threadIdx.x];
  for (int b = b0; b < b1; b++) {
    entries[b].state = s;
    entries[b].offset = o;
    const ZElem<uint16_t> &g = agg[b];
    o += g.cnt[s];
    s = (uint32_t)((g.exit >> (4 * s)) & 15);
  }
  if (threadIdx.x == Z2T - 1) ctrl->zig_avail = o;
}

// Serial walk of the whole draw (exact fallback for parse overflow).
__device__ void zig_serial(DevControl *ctrl, const uint64_t *words, double *normals, int64_t T) {
  const StreamState st = ctrl->stream;
  uint64_t j = 0;
  for (int64_t i = 0; i < T;) {
    int len, acc;
    double x;
    const uint64_t r = words ? words[j] : word_at(st, st.pos + j);
    zig_classify(r, j, st, words, st.pos, g_ki, g_wi, 1 << 20, len, acc, x);
    if (acc) normals[i++] = x;
    j += (uint64_t)len;
  }
  ctrl->zig_used = j;
  ctrl->zig_avail = (uint64_t)T;
}

// Z3: emit normals.
__global__ void __launch_bounds__(ZT) z3_kernel(DevControl *ctrl, const uint64_t *words, const double *xs,
                                                const uint8_t *meta, const ZEntry *entries, double *normals,
                                                int64_t T) {
  __shared__ ZElem<uint16_t> nodes[2 * ZT];
  __shared__ uint8_t in_state[2 * ZT];
  __shared__ uint32_t in_off[2 * ZT];
  if (ctrl->zig_overflow) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      zig_serial(ctrl, words, normals, T);
      ctrl->err |= 2;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctrl->zig_avail < (uint64_t)T) ctrl->err |= 1;
  const uint64_t j0 = ((uint64_t)blockIdx.x * ZT + threadIdx.x) * ZW;
  const uint64_t m8 = *reinterpret_cast<const uint64_t *>(meta + j0);
  uint32_t lens = 0, accs = 0;
#pragma unroll
  for (int i = 0; i < ZW; i++) {
    const uint32_t m = (uint32_t)((m8 >> (8 * i)) & 0xff);
    lens |= (m & 15u) << (4 * i);
    accs |= (m >> 7) << i;
  }
  ZElem<uint16_t> el;
  zthread_elem(lens, accs, el);
  nodes[ZT + threadIdx.x] = el;
  __syncthreads();
  for (int width = ZT / 2; width >= 1; width >>= 1) {
    if (threadIdx.x < width) {
      const int i = width + threadIdx.x;
      ZElem<uint16_t> o;
      zcompose(nodes[2 * i], nodes[2 * i + 1], o);
      nodes[i] = o;
    }
    __syncthreads();
  }
  const ZEntry be = entries[blockIdx.x];
  if (threadIdx.x == 0) { in_state[1] = (uint8_t)be.state; in_off[1] = 0; }
  __syncthreads();
  for (int width = 1; width < ZT; width <<= 1) {
    if (threadIdx.x < width) {
      const int i = width + threadIdx.x;
      const uint32_t s = in_state[i];
      const uint32_t o = in_off[i];
      in_state[2 * i] = (uint8_t)s;
      in_off[2 * i] = o;
      in_state[2 * i + 1] = (uint8_t)((nodes[2 * i].exit >> (4 * s)) & 15);
      in_off[2 * i + 1] = o + nodes[2 * i].cnt[s];
    }
    __syncthreads();
  }
  int pos = in_state[ZT + threadIdx.x];
  uint64_t off = be.offset + in_off[ZT + threadIdx.x];
  if (off >= (uint64_t)T) return;
  while (pos < ZW) {
    const int L = (int)((lens >> (4 * pos)) & 15);
    if ((accs >> pos) & 1) {
      if (off < (uint64_t)T) {
        normals[off] = xs[j0 + pos];
        if (off == (uint64_t)T - 1) ctrl->zig_used = j0 + pos + L;
      }
      off++;
    }
    pos += L;
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
}

// ---------------------------------------------------------------------------
int64_t momenta_words(int64_t T) {
  const int64_t n = T + T / 16 + 512;
  return (n + ZB - 1) / ZB * ZB;
}

size_t momenta_scratch_bytes(int64_t T) {
  const int64_t N = momenta_words(T), nb = N / ZB;
  return (size_t)N * 8 + (size_t)N + (size_t)nb * sizeof(ZElem<uint16_t>) + (size_t)nb * sizeof(ZEntry) + 256;
}

int launch_momenta(const MomentaBufs &b, int kind, int64_t T, cudaStream_t s, int *launches) {
  const int64_t N = momenta_words(T);
  const int nb = (int)(N / ZB);
  char *base = (char *)b.scratch;
  double *xs = (double *)base;
  uint8_t *meta = (uint8_t *)(base + (size_t)N * 8);
  ZElem<uint16_t> *agg = (ZElem<uint16_t> *)(base + (size_t)N * 9);
  ZEntry *entries = (ZEntry *)(base + (size_t)N * 9 + (size_t)nb * sizeof(ZElem<uint16_t>));
  const uint64_t *words = nullptr;
  cudaMemsetAsync(&b.ctrl->zig_overflow, 0, sizeof(int32_t), s);
  if (kind == PRNG_SFC64) {
    z0_sfc64_kernel<<<1, 1, 0, s>>>(b.ctrl, b.sfc_words, b.sfc_snaps, N + 64);
    words = b.sfc_words;
    (*launches)++;
  }
  z1_kernel<<<nb, ZT, 0, s>>>(b.ctrl, words, xs, meta, agg);
  z2_kernel<<<1, Z2T, 0, s>>>(b.ctrl, agg, entries, nb);
  z3_kernel<<<nb, ZT, 0, s>>>(b.ctrl, words, xs, meta, entries, b.normals, T);
  *launches += 3;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_momenta_advance(const MomentaBufs &b, cudaStream_t s, int *launches) {
  zadvance_kernel<<<1, 1, 0, s>>>(b.ctrl, b.sfc_snaps);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace rsv
