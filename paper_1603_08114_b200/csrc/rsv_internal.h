// rsv_internal.h -- device data layout shared by the kernels and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "prng.cuh"

namespace rsv {

// ---- momenta (numpy ziggurat parse) geometry -------------------------------
constexpr int ZW = 8;            // raw words per thread
constexpr int ZT = 256;          // threads per block
constexpr int ZB = ZW * (ZT - 4); // words per block (threads 0,1: guard; ZT-2, ZT-1: look-ahead)
constexpr int ZS = 16;           // parse states: words still owed to the running attempt
constexpr int ZMMAX = 7;         // tail loops resolvable in the parallel parse (len <= 15)
constexpr int Z2T = 256;         // threads of the block-scan kernel
constexpr int SFC_SNAP = 64;     // sfc64 state snapshot stride (words)

// ---- trajectory tile geometry ----------------------------------------------
constexpr int TR_NT = 256;       // threads per tile
constexpr int TR_R = 4;          // consecutive sites per thread (registers)
constexpr int TR_MINB = 3;       // resident CTAs per SM (register budget 85/thread)
constexpr int TR_W = TR_NT * TR_R;
constexpr int TR_NW = TR_NT / 32;
constexpr int TR_NV = 17;        // 8-byte words of a tile / CTA partial record (see TilePart)

// ---- streamed (one step per pass) kernel ------------------------------------
constexpr int ES_NT = 256;
constexpr int ES_R = 4;

struct DevParams {
  double phi, mu, xi, se2, su2;
  // derived once on the host (rsv_set_params) so no tile recomputes them
  double inv_su2, inv_se2, emu, one_m_phi2;
  double hconst;   // theta-only part of H (model.py:134-163 log terms + 0.5*T*mu)
  int32_t n_lo, n_span;  // |h| <= 50  <=>  rint(-2048 (h - mu)/ln2) - n_lo in [0, n_span]
};

// Per-CTA partial record of the trajectory kernel.  dh, H_old and H_new are
// exact sums of per-group values (a group = 4 consecutive sites 4-aligned in
// the global series, summed in site order) rounded to 128-bit fixed point
// (value * 2^64, fix128 in leapfrog.cu): integer addition is associative, so
// the totals do not depend on the tile shape, the tile -> CTA assignment or
// how the series is split across GPUs (bitwise the same dH for any world
// size).  The theta moments stay fixed-order FP64 sums.
struct TilePart {
  long long dh[2], hold[2], hnew[2];  // int128 as {low word, high word}
  double so[5];    // old path: sum d, sum d^2, sum d_t d_{t-1}, sum e, sum e^2
  double sn[5];    // proposal: same
  double flag;     // > 0 if any core site left [-50, 50] (or NaN) at a kick
};
static_assert(sizeof(TilePart) == TR_NV * 8, "TilePart is TR_NV 8-byte words");

// ---- time-sharded chains: one shard's record, all-gathered per proposal
// (mirrors rsv_shard_totals of the C ABI: 23 8-byte words)
struct ShardRec {
  TilePart part;       // over the shard's owned sites
  double ends[4];      // d_0 old, d_{T-1} old, d_0 new, d_{T-1} new (0 unless this shard owns the end)
  uint64_t u_word;     // raw word after the momenta (the Metropolis uniform)
  uint64_t words_used; // raw words the momenta consumed
};
constexpr int SHARD_W = (int)(sizeof(ShardRec) / 8);
static_assert(SHARD_W == 23, "rsv_shard_totals layout");

// ---- time-sharded momenta: each shard parses only a window of the raw-word
// stream around its sites.  Anchor words a_r (the expected
// start of shard r's first owned normal) split the stream; a shard counts
// the normals whose attempts start in [a_r, a_{r+1}), the counts are
// all-gathered and their exclusive prefix gives every window its global
// normal index.  Neighbouring windows overlap around each anchor: both
// shards report the first attempt start at or after it, which must agree
// (the check that the speculative start of a window has synchronised).
struct WinInfo {           // one shard's window, all-gathered (8 words)
  int64_t cnt_lo, cnt_hi;  // window normals whose attempts start before a_lo / a_hi
  int64_t s_lo, s_hi;      // first attempt start at or after a_lo / a_hi (words past the stream position)
  int64_t n_win;           // normals the window produced
  int64_t w0;              // first word of the window
  int64_t err;             // bit 1: the exact serial walk redid the window
  int64_t pad;
};
// Peer-memory exchange of the sharded chain's per-proposal records: every
// shard context owns one box; each shard writes its record into slot
// [epoch & 1][rank] of every shard's box over NVLink (P2P stores) and then
// the slot's flag (the epoch, release at system scope); a shard reads the
// records once all flags of its box carry its own epoch.  Two slots: a rank
// can run at most one exchange ahead of the slowest (its next record needs
// everyone's current one).
constexpr int P2P_MAXW = 16;
constexpr int P2P_KINDS = 2;  // 0: shard records (ShardRec, 23 words), 1: window records (WinInfo, 8 words)
constexpr int P2P_WORDS = 24;
struct P2PBox {
  unsigned long long flag[P2P_KINDS][2][P2P_MAXW];
  double rec[P2P_KINDS][2][P2P_MAXW][P2P_WORDS];
};
struct ZigWin {            // window mode of the momenta kernel
  int64_t wb0;             // first block: CTA b of the window parses block wb0 + b of the full stream
  int64_t w0;              // wb0 * ZB
  int64_t cap;             // capacity of out / nend (normals)
  int64_t a_lo, a_hi;      // anchors (words past the stream position); a_hi < 0: the last shard
  double *out;             // the window's normals, in stream order
  uint32_t *nend;          // optional: per normal, the word after its attempt (relative to w0)
  WinInfo *info;
};

// ---- ensemble of independent chains (rsv_ens_*) ------------------------------
struct EnsPart {  // per trajectory tile: partials of the (<= 2) chains its core touches
  double dh, hold, hnew, flag;
};
struct EnsChain {  // per chain: sfc64 stream and the last proposal's bookkeeping
  uint64_t st[4];        // stream state for the next draw (a, b, c, counter)
  uint64_t st_used[4];   // state after the momenta's words (no uniform drawn)
  uint64_t st_used1[4];  // ... and after the Metropolis uniform
  uint64_t u_word, used;
  double last_dh;        // +inf when the proposal diverged
  int32_t last_accept, n_accept, n_diverged, overflow;
};

// ---- run_chain on the device (theta draws by one device thread) --------------
struct DevPrior {  // mirrors rsv_prior / PriorSpec (sampler.py:43-63)
  double mu_mean, mu_var, xi_mean, xi_var, var_shape, var_scale, phi_a, phi_b;
};
constexpr int RUN_STORM_WINDOW = 100, RUN_STORM_LIMIT = 50;  // sampler.py:36-37
struct DevRun {
  int64_t sweep;        // sweeps done
  int64_t n_burnin, thin, n_store, stored;
  double *params;       // n_store x 5: phi, mu, xi, sigma_eta_sq, sigma_u_sq
  int32_t *accept;      // n_store
  double *delta_h;      // n_store
  int64_t *iters;       // n_store
  int64_t storm_sweep;  // first sweep at which the storm guard fired (-1: none)
  int32_t ring_n, ring_pos, ring_div;  // divergence flags of the last RUN_STORM_WINDOW proposals
  uint8_t ring[RUN_STORM_WINDOW];
  int32_t degenerate;   // a full conditional had a non-positive precision (ValueError in the reference)
};

struct DevResult {  // mirrors rsv_result
  int32_t accept, diverged;
  double delta_h, h_old, h_new;
  uint64_t words_used;
  double u;
};

struct DevControl {
  StreamState stream;   // stream position / state for the next draw
  int32_t cur;          // index of the h buffer holding the current path
  int32_t err;          // bit 0: momenta shortfall, bit 1: parse overflow (serial fallback ran)
  uint64_t zig_used;    // raw words consumed by the last momenta draw
  uint64_t zig_avail;   // normals the parallel parse produced
  int32_t zig_overflow; // an attempt needed > ZMMAX tail loops
  int32_t pad;
  double ends_old[2], ends_new[2];  // d_0, d_{T-1} (shifted by mu)
  double stats[7];      // statistics of the kept path (shift mu, xi of the params used)
  DevResult res;
  uint64_t u_word;      // raw word right after the momenta (the Metropolis uniform)
  uint32_t tiles_done;  // trajectory CTAs finished (last one runs the Metropolis step)
  uint32_t tile_next;   // dynamic tile scheduling: tiles handed out beyond the first wave
  // sequential state of jump-ahead generators at the stream position (pcg32:
  // LCG state before output 2*pos; minstd: x_{3*pos}); seq_next = at pos + used
  uint64_t seq_state, seq_next;
  // momenta kernel bookkeeping (reset by its last CTA: no memsets per draw)
  uint32_t zig_ticket, zig_done, zig_epoch, zig_pub;
  // rsv_run_chain stopped (divergence storm or degenerate precision): every
  // later kernel of the run leaves the stream, the path and the parameters
  // exactly as they were at that sweep (sampler.py:331-337 raises there)
  int32_t halt;
  uint32_t pad5;
  double shard_parts[TR_NV];  // time-sharded chains: this shard's totals (TilePart order)
  // trajectory kernel: every CTA adds its fixed-point dH, H_old, H_new as
  // three 42-bit limbs each (fx[3 v + l]; <= 2^22 CTAs cannot carry out of a
  // 64-bit word) and ORs its flag into fx[9]; the last CTA reads and clears
  unsigned long long fx[10];
  // peer-memory record exchange of a time-sharded chain (rsv_shard_p2p_*):
  // epochs of this shard's pushes (shard records, window records)
  unsigned long long p2p_seq[2];
  // %globaltimer stamps (ns) of the last proposal: momenta kernel first-CTA
  // entry / last-CTA exit, trajectory kernel CTA-0 entry / last-CTA exit,
  // and the previous proposal's trajectory exit
  unsigned long long t_stamp[5];
};

}  // namespace rsv
