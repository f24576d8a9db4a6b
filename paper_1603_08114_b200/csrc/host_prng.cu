// host_prng.cu -- host side of the bit generators: seeding, sequential draws
// and a numpy-compatible bitgen_t so numpy's own Generator (used for the
// scalar theta draws, sampler.py:170-272) continues exactly the stream the
// device consumed for the momenta.  Same formulas as prng.cuh (shared code).
#include <stdint.h>
#include <string.h>

#include "../../include/rsvhmc_b200.h"
#include "prng.cuh"

using namespace rsv;

namespace {
struct NpyBitgen {  // numpy/random/bitgen.h bitgen_t
  void *state;
  uint64_t (*next_uint64)(void *);
  uint32_t (*next_uint32)(void *);
  double (*next_double)(void *);
  uint64_t (*next_raw)(void *);
};

uint64_t stream_next(rsv_prng_state *st) {
  if (st->kind == PRNG_SFC64) {
    st->pos++;
    return sfc64_next(st->s);
  }
  StreamState s;
  s.kind = st->kind;
  for (int i = 0; i < 4; i++) s.s[i] = st->s[i];
  s.pos = st->pos;
  const uint64_t w = word_at(s, st->pos);
  st->pos++;
  return w;
}
uint64_t bg_u64(void *p) { return stream_next((rsv_prng_state *)p); }
uint32_t bg_u32(void *p) { return (uint32_t)(stream_next((rsv_prng_state *)p) >> 32); }
double bg_dbl(void *p) { return u01(stream_next((rsv_prng_state *)p)); }
}  // namespace

extern "C" {

/* Seed a stream from raw seed material (numpy SeedSequence words):
 * philox key = m[0..1]; minstd x0 = m[0] mod (2^31-1) (0 -> 1);
 * pcg32 = pcg32_srandom_r(initstate m[0], initseq m[1]);
 * sfc64 = numpy sfc64_set_seed(m[0], m[1], m[2]) (w = 1, 12 discards). */
int rsv_stream_seed(rsv_prng_state *st, int kind, const uint64_t *m) {
  if (!st || !m || kind < 0 || kind > 3) return RSV_E_INVALID;
  memset(st, 0, sizeof(*st));
  st->kind = kind;
  switch (kind) {
    case PRNG_PHILOX: st->s[0] = m[0]; st->s[1] = m[1]; break;
    case PRNG_MINSTD: { const uint64_t x = m[0] % MINSTD_M; st->s[0] = x ? x : 1; break; }
    case PRNG_PCG32: {
      const uint64_t inc = (m[1] << 1u) | 1u;
      uint64_t s = 0;
      s = s * PCG_MULT + inc;
      s += m[0];
      s = s * PCG_MULT + inc;
      st->s[0] = s;
      st->s[1] = inc;
      break;
    }
    default:
      st->s[0] = m[0]; st->s[1] = m[1]; st->s[2] = m[2]; st->s[3] = 1;
      for (int i = 0; i < 12; i++) sfc64_next(st->s);
      break;
  }
  return 0;
}

uint64_t rsv_stream_next_u64(rsv_prng_state *st) { return stream_next(st); }
double rsv_stream_next_double(rsv_prng_state *st) { return u01(stream_next(st)); }

/* Fill a numpy bitgen_t (struct of 5 pointers) drawing from *st. */
int rsv_stream_bitgen(rsv_prng_state *st, void *bitgen_out) {
  if (!st || !bitgen_out) return RSV_E_INVALID;
  NpyBitgen *b = (NpyBitgen *)bitgen_out;
  b->state = st;
  b->next_uint64 = bg_u64;
  b->next_uint32 = bg_u32;
  b->next_double = bg_dbl;
  b->next_raw = bg_u64;
  return 0;
}

/* numpy Philox block (for writing a position back into np.random.Philox). */
void rsv_philox_block(uint64_t blk, uint64_t k0, uint64_t k1, uint64_t out[4]) { philox_block(blk, k0, k1, out); }

}  // extern "C"
