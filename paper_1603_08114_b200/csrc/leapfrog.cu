// leapfrog.cu -- the fused HMC trajectory and its Metropolis test on sm_100a.
//
// Replaces (paths relative to the reference's pkg/src/rsvhmc/):
//   integrator.py:149-179 integrate_trajectory and :139-146 elementary_step
//     (kernels 1-3, _kernels.py:37-54, force _kernels.py:23-34),
//   model.py:134-182 log_posterior / hamiltonian (H_old, H_new),
//   sampler.py:155-167 (dH, divergence sentinel, Metropolis),
//   the sums inside sampler.py:170-272 (theta sufficient statistics).
//
// traj_persistent_kernel: a persistent grid (2 CTAs per SM) walks tiles of
// `core` consecutive sites, each with a halo of n_steps + 1 sites on either
// side; each thread keeps R = 4 consecutive sites (x = K (h - mu), p, and
// the per-site force constants) in registers for the whole trajectory.
// Neighbour values move by warp shuffles and, across warps, through
// ghost lanes refreshed via shared memory every R steps.  Because the
// stencil is nearest-neighbour, L steps on a tile with an L-site halo give
// the core sites exactly the values a global step-by-step sweep gives, so
// the whole trajectory is one launch with no grid-wide synchronisation.
// HBM traffic per trajectory is 32 B/site (h, p, (y/2)y, lnRV in; h' out);
// the FP64 pipe is the bound.
#include <math.h>

#include "exp_table.h"
#include "rsv_check.h"
#include "traj_dev.cuh"
#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

// Ghost-lane refresh slots of one thread (see ghost_lanes below): `w` the
// slot this lane writes (lanes 1 / 30), `r` the slot it reads (lanes 0 / 31
// with a neighbour warp), null otherwise; the two parities alternate.
struct GhostSlots {
  double *w;
  const double *r;
};

template <int R, int NT>
__device__ __forceinline__ void ghost_refresh(double (&d)[R], double (&p)[R], const GhostSlots &g, int parity);

// The L leapfrog steps of a tile (integrator.py:149-179), unrolled by the
// ghost-refresh period R: loop control and the refresh test once per R
// steps.  EDGE is warp-uniform (masked kick for partially live / end / mixed
// core threads).  cf / cl: ensemble chain boundaries cut the coupling.
// The drifts between two kicks are one full drift (K3 of a step and K1 of
// the next, integrator.py:161-179, act on the same p) whether or not the
// caller asked for fuse_half_steps: the same map in real arithmetic, one
// FP64 instruction per site-update less; the last half drift is taken as a
// full one minus a half (no per-step select in the unrolled loop, measured
// 3.5 % faster than either alternative).
template <bool EDGE, int R, int NT, bool ENS>
__device__ __forceinline__ void run_steps(double (&d)[R], double (&p)[R], const double (&Ad)[R],
                                          const double (&Cd)[R], const TrajConsts &s,
                                          const unsigned long long *tab, uint32_t live, uint32_t endm,
                                          const unsigned (&cm)[R], bool cf, bool cl, int L, const GhostSlots &gs,
                                          unsigned &nmax) {
  constexpr int NW = NT / 32;
  int gpar = 0;
  auto one = [&]() {
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
    drift(d, p, s.xc_full);
  };
  drift(d, p, s.xc_half);
  int step = 0;
  for (; step + R <= L; step += R) {
#pragma unroll
    for (int u = 0; u < R; u++) one();
    if (NW > 1 && step + R < L) {
      ghost_refresh<R, NT>(d, p, gs, gpar);
      gpar ^= 1;
    }
  }
  for (; step < L; step++) one();
  drift(d, p, -s.xc_half);
  if (NW > 1) ghost_refresh<R, NT>(d, p, gs, gpar);
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
__device__ __forceinline__ GhostSlots ghost_lanes(double *s_gx, int lane, int warp) {
  constexpr int NW = NT / 32;
  // s_gx layout: [parity][warp][side 0: lane 30 -> right neighbour's lane 0,
  //                                side 1: lane 1 -> left neighbour's lane 31][2R]
  GhostSlots g;
  g.w = (lane == 30 || lane == 1) ? s_gx + (warp * 2 + (lane == 1)) * 2 * R : nullptr;
  g.r = (lane == 0 && warp > 0)        ? s_gx + ((warp - 1) * 2 + 0) * 2 * R
        : (lane == 31 && warp < NW - 1) ? s_gx + ((warp + 1) * 2 + 1) * 2 * R
                                        : nullptr;
  return g;
}
template <int R, int NT>
__device__ __forceinline__ void ghost_refresh(double (&d)[R], double (&p)[R], const GhostSlots &g, int parity) {
  constexpr int PO = (NT / 32) * 4 * R;  // doubles per parity
  static_assert(R % 2 == 0, "16-byte slot accesses");
  if (g.w) {
    double2 *dst = reinterpret_cast<double2 *>(g.w + parity * PO);
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      dst[r / 2] = make_double2(d[r], d[r + 1]);
      dst[R / 2 + r / 2] = make_double2(p[r], p[r + 1]);
    }
  }
  __syncthreads();
  if (g.r) {
    const double2 *src = reinterpret_cast<const double2 *>(g.r + parity * PO);
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const double2 a = src[r / 2], b = src[R / 2 + r / 2];
      d[r] = a.x; d[r + 1] = a.y;
      p[r] = b.x; p[r + 1] = b.y;
    }
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
template <int W, bool HEADK = false>
__device__ __forceinline__ void stage_tile(const TrajArgs &A, const double *hsrc, int tile, double *stage,
                                           uint64_t *bar, int part = 3) {
  const int64_t g = (int64_t)tile * A.g.core - A.g.halo;
  const int64_t lo = g < 0 ? 0 : g, hi = min(g + W, A.Tpad);
  const uint32_t bytes = (uint32_t)((hi - lo) * 8);
  const int off = (int)(lo - g);
  RSV_CHECK(tile >= 0 && tile < A.g.n_tiles && lo < hi && off >= 0 && off + (hi - lo) <= W);
  RSV_CHECK(bytes % 16 == 0 && off % 2 == 0 && lo % 2 == 0);
  RSV_CHECK((((uintptr_t)(hsrc + lo)) & 15) == 0 && (((uintptr_t)(A.p_in + lo)) & 15) == 0);
  mbar_expect_tx(bar, (part == 3 ? 4 : part == 1 ? 3 : 1) * bytes);
  if (part & 1) {
    // (a separate instantiation: the branch alone costs the device-resident
    // kernel ~1 us at 2^20 through the step loop's schedule, measured)
    const double *hs = (HEADK && hi <= A.head_end) ? A.h_head : hsrc;
    tma_load_1d(stage + 0 * W + off, hs + lo, bytes, bar);
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
  RSV_CHECK(tile >= 0 && tile < A.g.n_tiles && lo < hi && off >= 0 && off + (hi - lo) <= W && bytes % 16 == 0);
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

template <int R, int NT, bool STATS>
struct PersistSmem {
  static constexpr int NW = NT / 32;
  static constexpr int W = NW > 1 ? NW * 30 * R + 2 * R : 32 * R;
  static constexpr int NM = STATS ? 10 : 1;
  union {
    double stage[2][4 * W];     // double-buffered tile windows
    double red[NW * TR_NV];     // after the last tile: warp totals of the CTA reduction
  };
  __int128 acc3[3][NT];         // per-thread fixed-point dh, H_old, H_new across tiles
  double accm[NM][NT];          // per-thread theta moments across tiles (old 5, new 5)
  double gx[2 * NW * 4 * R];    // ghost-lane refresh slots
  double v[NW * TR_NV + TR_NV];
  alignas(16) unsigned long long tab[RSV_EXP_TAB_N];
  double epart[2][NW][8];  // ensemble: per-warp chain partials of a tile (by staging buffer)
  uint64_t bar[4];  // two staging buffers, the exp table, the first tile's momenta
  int last;
  int next[2];     // the CTA's next tile (by staging buffer: read after the tile, rewritten two tiles later)
};

template <int R, int NT, int MINB, bool STATS, bool ENS = false, bool DEVK = false, bool HEADK = false>
__global__ void __launch_bounds__(NT, MINB) traj_persistent_kernel(TrajArgs A) {
  using SM = PersistSmem<R, NT, STATS>;
  constexpr int NW = SM::NW, W = SM::W;
  // Without statistics every reduced value is a fixed-point integer sum, so
  // tiles can go to whichever CTA is free (dynamic scheduling: the two CTAs
  // of an SM do not finish a tile apart); the FP64 moments of the statistics
  // variant keep the static, fixed-order assignment.
  constexpr bool DYN = !STATS;
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
    sk.xg_int = q.xg_int; sk.xg_end = q.xg_end; sk.xbphi = q.xbphi;
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
  for (int k = 0; k < 3; k++) S.acc3[k][tid] = 0;
  for (int k = 0; k < SM::NM; k++) S.accm[k][tid] = 0.0;
  bool bad = false;  // a core site flagged at a kick / an energy beyond the fixed-point range
  int n_done = 0;
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
    if (!ENS && tile < n_tiles) stage_tile<W, HEADK>(A, hsrc, tile, S.stage[0], &S.bar[0], 1);
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
  const int64_t core_len = A.g.core;
  const bool own_lane = (lane >= 1 && lane <= 30) || (lane == 0 && warp == 0) || (lane == 31 && warp == NW - 1);
  const int lw = warp * WSTEP + lane * R;  // my first site inside the window
  const GhostSlots gs = ghost_lanes<R, NT>(S.gx, lane, warp);
  RSV_CHECK(lw >= 0 && lw + R <= W && lw % 2 == 0);
  RSV_CHECK((!gs.w || (gs.w >= S.gx && gs.w + 2 * R <= S.gx + NW * 4 * R)) &&
            (!gs.r || (gs.r >= S.gx && gs.r + 2 * R <= S.gx + NW * 4 * R)));
  // Interior tiles (window inside the local range, core fully owned, no
  // global end site and no chain boundary in the window) need no per-site
  // masks: every window site is live (sites past the halo only ever feed
  // sites outside the core) and the thread's core mask is the same for every
  // such tile (H and the core are multiples of R: all of a thread's sites
  // are core or none), so it is computed once here.
  uint32_t core_int = 0;
#pragma unroll
  for (int r = 0; r < R; r++) core_int |= (uint32_t)(own_lane && lw + r >= H && lw + r < H + core_len) << r;
  unsigned parity = 0;  // bit b: mbarrier phase of staging buffer b
  int buf = 0;
  long long cyc_wait = 0, cyc_pre = 0, cyc_loop = 0, cyc_post = 0, c0 = 0, c1 = 0;
  const bool stamps = A.dbg != nullptr;
  bool first = !ENS;  // first tile of a single chain: momenta not yet readable
  for (; tile < n_tiles; buf ^= 1) {
    if (stamps) c0 = clock64();
    // the CTA's next tile (thread 0; everyone reads S.next after the tile's
    // closing barrier) -- its staging starts now, into the other buffer,
    // released at the end of the previous tile (first tile: after the wait)
    if (tid == 0) S.next[buf] = DYN ? (int)gridDim.x + (int)atomicAdd(&A.ctrl->tile_next, 1u) : tile + (int)gridDim.x;
    const int next = tid == 0 ? S.next[buf] : 0;
    if (tid == 0 && !first && next < n_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (ENS) stage_tile_ens<W>(A, next, S.stage[buf ^ 1], &S.bar[buf ^ 1]);
      else stage_tile<W, HEADK>(A, hsrc, next, S.stage[buf ^ 1], &S.bar[buf ^ 1]);
    }
    const double *stg = S.stage[buf];
    const int64_t t0 = (int64_t)tile * core_len;
    const int64_t t1 = min(t0 + core_len, T);
    const int64_t g0 = t0 - H + lw;
    const bool interior = !ENS && t0 >= H && t0 + core_len + H <= T && t0 >= A.own_lo && t0 + core_len <= A.own_hi &&
                          goff + t0 - H > 0 && goff + t0 - H + W < Tg;

    // ---- tile data from the staging buffer ----
    mbar_wait(&S.bar[buf], (parity >> buf) & 1);
    parity ^= 1u << buf;
    if (stamps) { c1 = clock64(); cyc_wait += c1 - c0; c0 = c1; }
    double d[R], p[R], Ad[R], Cd[R], av[R], lv[R];
    uint32_t live, core, wcore, endm = 0, firstm = 0;
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
    bool warp_edge = false;
    if (interior) {
      live = (1u << R) - 1;
      core = wcore = core_int;
#pragma unroll
      for (int r = 0; r < R; r++) {
        cm[r] = ~0u;
        d[r] = d[r] - s.mu;
        Ad[r] = s.dt * (s.emu * av[r]);
        Cd[r] = fma(-s.alpha, lv[r] - s.xm, s.half_dt);
      }
    } else {
      if (ENS) {
        const int64_t m = ((g0 % A.Tc) + A.Tc) % A.Tc;
        cf = m == 0;
        cl = m + R == A.Tc;
        chain = g0 >= 0 ? g0 / A.Tc : -1;
      }
      const int64_t lo_live = max((int64_t)0, t0 - H), hi_live = min(T, t1 + H);
      // only a lane whose sites include global site 0 or Tg-1 has end sites
      const bool near_end =
          (g0 + goff <= 0 && g0 + goff + R > 0) || (g0 + goff <= Tg - 1 && g0 + goff + R > Tg - 1);
      live = core = wcore = 0;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const int64_t gi = g0 + r;
        const bool in = gi >= lo_live && gi < hi_live;
        // wcore: tile-core sites of the local range (written back; a shard
        // keeps its margins evolving too); core: those this context owns
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
      warp_edge = __any_sync(0xffffffffu, edge || !any_live || mixed_core);
      if (!ENS && edge && !A.h_src) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          if ((core >> r) & 1) {
            if (g0 + r + goff == 0) A.ctrl->ends_old[0] = d[r];
            if (g0 + r + goff == Tg - 1) A.ctrl->ends_old[1] = d[r];
          }
        }
      }
    }
    // H_old of the owned core sites while a / lnRV are at hand
    double vold[6] = {0, 0, 0, 0, 0, 0};
    {
      const double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
      tile_energy<R, STATS>(d, av, lv, dl, core, firstm, s, S.tab, vold);
    }
    if (!ENS && first) {
      // the momenta kernel's normals: wait for it (everything above
      // overlapped its tail), stage this tile's momenta and the next tile
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (tid == 0) {
        stage_tile<W, HEADK>(A, hsrc, tile, S.stage[buf], &S.bar[3], 2);
        if (next < n_tiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          stage_tile<W, HEADK>(A, hsrc, next, S.stage[buf ^ 1], &S.bar[buf ^ 1]);
        }
      }
      mbar_wait(&S.bar[3], 0);
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        const double2 p2 = *reinterpret_cast<const double2 *>(stg + 1 * W + lw + r);
        p[r] = ((live >> r) & 1) ? p2.x : 0.0;
        p[r + 1] = ((live >> (r + 1)) & 1) ? p2.y : 0.0;
      }
      first = false;
    }
    const double hold = vold[0] + kinetic<R>(p, core);  // the thread's group: H_old of its core sites
    if (STATS) {
#pragma unroll
      for (int k = 0; k < 5; k++) S.accm[k][tid] += vold[1 + k];
    }

    // ---- the trajectory, on x = K (h - mu) ----
    if (stamps) { c1 = clock64(); cyc_pre += c1 - c0; c0 = c1; }
#pragma unroll
    for (int r = 0; r < R; r++) d[r] *= s.kx;
    unsigned nmax = 0;
    const int L = A.n_steps;
    if (warp_edge) {
      run_steps<true, R, NT, ENS>(d, p, Ad, Cd, s, S.tab, live, endm, cm, cf, cl, L, gs, nmax);
    } else {
      run_steps<false, R, NT, ENS>(d, p, Ad, Cd, s, S.tab, live, endm, cm, cf, cl, L, gs, nmax);
      nmax = core ? nmax : 0u;
    }
#pragma unroll
    for (int r = 0; r < R; r++) d[r] *= s.kxinv;
    __syncthreads();  // refresh slots reused by the next tile
    if (stamps) { c1 = clock64(); cyc_loop += c1 - c0; c0 = c1; }

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
      tile_energy<R, STATS>(d, av, lv, dl, core, firstm, s, S.tab, vnew);
    }
    const double hnew = vnew[0] + kinetic<R>(p, core);
    double *hd = hdst;
    if (ENS && core) {
      RSV_CHECK(chain >= 0 && chain < A.n_chains);
      hd = A.ens_cur[chain] ? A.hbuf0 : A.hbuf1;
    }
    RSV_CHECK(!wcore || (g0 >= 0 && g0 + R <= A.Tpad));
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
    if (!ENS && !interior && !A.h_src) {
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
      const double dhv = hnew - hold;
      double w8[8] = {right ? 0.0 : dhv, right ? 0.0 : hold, right ? 0.0 : hnew, right ? 0.0 : fl,
                      right ? dhv : 0.0, right ? hold : 0.0, right ? hnew : 0.0, right ? fl : 0.0};
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
    } else if (core) {
      const double dhv = hnew - hold;
      bad |= nmax > (unsigned)s.n_span || !(fabs(hold) < FIX_MAX) || !(fabs(hnew) < FIX_MAX);
      S.acc3[0][tid] += fix128(dhv);
      S.acc3[1][tid] += fix128(hold);
      S.acc3[2][tid] += fix128(hnew);
      if (STATS) {
#pragma unroll
        for (int k = 0; k < 5; k++) S.accm[5 + k][tid] += vnew[1 + k];
      }
    }
    __syncthreads();  // all reads of this tile's buffer done before it is refilled
    if (ENS && warp == 0 && lane < 8) {  // the tile's two chain records, warps summed in order
      double v = S.epart[buf][0][lane];
#pragma unroll
      for (int w = 1; w < NW; w++) v += S.epart[buf][w][lane];
      double *q = reinterpret_cast<double *>(A.ens_parts + 2 * (size_t)tile);
      q[lane] = v;  // EnsPart {dh, hold, hnew, flag} x 2
    }
    if (stamps) { c1 = clock64(); cyc_post += c1 - c0; }
    tile = S.next[buf];  // written by thread 0 before this tile's barriers
    n_done++;
  }
  if (A.dbg && tid == 0) {
    A.dbg[(size_t)blockIdx.x * 8 + 0] = cyc_wait;
    A.dbg[(size_t)blockIdx.x * 8 + 1] = cyc_pre;
    A.dbg[(size_t)blockIdx.x * 8 + 2] = cyc_loop;
    A.dbg[(size_t)blockIdx.x * 8 + 3] = cyc_post;
    A.dbg[(size_t)blockIdx.x * 8 + 4] = n_done;  // tiles processed
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
  // ---- one reduction per CTA: the fixed-point sums in any order (exact),
  // the moments by warp butterflies and warp totals in warp order ----
  __int128 q3[3] = {S.acc3[0][tid], S.acc3[1][tid], S.acc3[2][tid]};
  double m[10];
#pragma unroll
  for (int k = 0; k < 10; k++) m[k] = 0.0;
  if (STATS) {
#pragma unroll
    for (int k = 0; k < 10; k++) m[k] = S.accm[STATS ? k : 0][tid];
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 3; k++) q3[k] += shfl_xor_128(q3[k], o);
    if (STATS) {
#pragma unroll
      for (int k = 0; k < 10; k++) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
    }
  }
  const bool wbad = __any_sync(0xffffffffu, bad);
  __syncthreads();  // the stage buffers (aliased by red) are no longer read
  if (lane == 0) {
    TilePart &w = *reinterpret_cast<TilePart *>(S.red + warp * TR_NV);
    st128(w.dh, q3[0]);
    st128(w.hold, q3[1]);
    st128(w.hnew, q3[2]);
#pragma unroll
    for (int k = 0; k < 5; k++) { w.so[k] = m[k]; w.sn[k] = m[5 + k]; }
    w.flag = wbad ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    const TilePart *w = reinterpret_cast<const TilePart *>(S.red);
    TilePart o = w[0];
    __int128 a0 = ld128(o.dh), a1 = ld128(o.hold), a2 = ld128(o.hnew);
    for (int q = 1; q < NW; q++) {
      a0 += ld128(w[q].dh);
      a1 += ld128(w[q].hold);
      a2 += ld128(w[q].hnew);
      for (int k = 0; k < 5; k++) { o.so[k] += w[q].so[k]; o.sn[k] += w[q].sn[k]; }
      o.flag = fmax(o.flag, w[q].flag);
    }
    // the fixed-point sums go straight into the grid totals (64-bit atomic
    // limbs); only the statistics variant leaves a per-CTA record, for the
    // fixed-order sums of its FP64 moments
    fx_add(A.ctrl->fx + 0, a0);
    fx_add(A.ctrl->fx + 3, a1);
    fx_add(A.ctrl->fx + 6, a2);
    if (o.flag > 0.0) atomicOr(A.ctrl->fx + 9, 1ull);
    if (STATS) A.parts[blockIdx.x] = o;
    // acquire-release count: this CTA's partials are released; the last CTA
    // acquires everyone's
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
// Persistent, TMA-staged shapes (R sites per thread, threads per CTA, CTAs
// per SM).  The index is the RSV_TRAJ_VARIANT development switch; 11 is the
// long-series shape, 12..14 the small windows for short series, 17 one
// 512-thread CTA per SM.  Retired indices (round-1 experiments: the
// non-persistent kernel and R = 6 / 8 shapes, all measured slower) fall back
// to the automatic choice.
static const TrajVariant kVariants[] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0},
                                        {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0},
                                        {4, 256, 2}, {4, 128, 3}, {4, 64, 5}, {4, 32, 8},
                                        {0, 0, 0}, {0, 0, 0}, {4, 512, 1}};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
static bool variant_available(int v) { return v >= 0 && v < kNumVariants && kVariants[v].R > 0; }

int traj_num_variants() { return kNumVariants; }

static TrajGeom traj_geometry_v(int64_t T, int n_steps, int sm_count, int variant) {
  TrajGeom g;
  if (!variant_available(variant)) variant = 11;
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
  g.grid = (int)((int64_t)g.n_tiles < slots ? (int64_t)g.n_tiles : slots);
  return g;
}

// variant < 0: automatic shape.  Long series use the 256-thread persistent
// kernel (11); when that leaves SMs idle, the CTA window shrinks (128 / 64 /
// 32 threads) so a short series still spreads over the whole GPU -- at small
// T the trajectory is latency-bound per step, and more, smaller tiles
// shorten it even though the halo share grows.
TrajGeom traj_geometry(int64_t T, int n_steps, int sm_count, int variant) {
  if (variant_available(variant)) return traj_geometry_v(T, n_steps, sm_count, variant);
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

template <int R, int NT, int MINB, bool STATS, bool ENS = false, bool DEVK = false, bool HEADK = false>
static void launch_p2(const TrajArgs &a, cudaStream_t s) {
  const size_t smem = sizeof(PersistSmem<R, NT, STATS>);
  cudaFuncSetAttribute(traj_persistent_kernel<R, NT, MINB, STATS, ENS, DEVK, HEADK>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // same (maximal) shared-memory carveout as the momenta kernel: no L1/shared
  // reconfiguration of the SMs between the two kernels of a proposal
  cudaFuncSetAttribute(traj_persistent_kernel<R, NT, MINB, STATS, ENS, DEVK, HEADK>,
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
    cudaLaunchKernelEx(&cfg, traj_persistent_kernel<R, NT, MINB, STATS, ENS, DEVK, HEADK>, a);
  } else {
    traj_persistent_kernel<R, NT, MINB, STATS, ENS, DEVK, HEADK><<<a.g.grid, NT, smem, s>>>(a);
  }
}

// run_chain on the device: the statistics variant with device-resident
// theta constants (persistent shapes of the automatic geometry only)
template <int R, int NT, int MINB>
static void launch_pd(const TrajArgs &a, cudaStream_t s) {
  launch_p2<R, NT, MINB, true, false, true>(a, s);
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
const void *traj_kernel_fn_devk(int variant, int) {
#define RSV_FN(R, NT, MB) ((const void *)traj_persistent_kernel<R, NT, MB, true, false, true>)
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
  if (a.stats) launch_p2<R, NT, MINB, true>(a, s);
  else launch_p2<R, NT, MINB, false>(a, s);
}

const void *traj_kernel_fn_head() { return (const void *)traj_persistent_kernel<4, 256, 2, false, false, false, true>; }

const void *traj_kernel_fn(int variant, int, int stats) {
#define RSV_FN(R, NT, MB)                                                     \
  (stats ? (const void *)traj_persistent_kernel<R, NT, MB, true>              \
         : (const void *)traj_persistent_kernel<R, NT, MB, false>)
  switch (variant) {
    case 12: return RSV_FN(4, 128, 3);
    case 13: return RSV_FN(4, 64, 5);
    case 14: return RSV_FN(4, 32, 8);
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

const void *traj_kernel_fn_ens(int) {
  return (const void *)traj_persistent_kernel<4, 256, 2, false, true>;
}

__global__ void ens_decide_kernel(TrajArgs A);

int launch_trajectory(const TrajArgs &a, cudaStream_t s, int *launches) {
  if (a.kdev) {
    if (!launch_devk(a, s)) return -1;
    (*launches)++;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  if (a.Tc > 0) {
    launch_p2<4, 256, 2, false, true>(a, s);
    ens_decide_kernel<<<(a.n_chains + 127) / 128, 128, 0, s>>>(a);
    (*launches) += 2;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  if (a.h_head && a.g.variant == 11 && !a.stats) {  // zero-copy input with a copied head
    launch_p2<4, 256, 2, false, false, false, true>(a, s);
    (*launches)++;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  switch (a.g.variant) {
    case 12: launch_p<4, 128, 3>(a, s); break;
    case 13: launch_p<4, 64, 5>(a, s); break;
    case 14: launch_p<4, 32, 8>(a, s); break;
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
  TilePart tp;
  if (STATS) {
    // the moments: CTA records in the plain loop's order (part j, then
    // j + NT, ...), then warp butterflies and warp totals in warp order
    double mm[10];
#pragma unroll
    for (int k = 0; k < 10; k++) mm[k] = 0.0;
    for (int j = threadIdx.x; j < n_parts; j += NT) {
      const TilePart &t = A.parts[j];
#pragma unroll
      for (int k = 0; k < 5; k++) { mm[k] += t.so[k]; mm[5 + k] += t.sn[k]; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
      for (int k = 0; k < 10; k++) mm[k] += __shfl_xor_sync(0xffffffffu, mm[k], o);
    }
    if (lane == 0)
      for (int k = 0; k < 10; k++) s_v[warp * TR_NV + k] = mm[k];
    __syncthreads();
    if (threadIdx.x) return;
    for (int k = 0; k < 5; k++) { tp.so[k] = s_v[k]; tp.sn[k] = s_v[5 + k]; }
    for (int q = 1; q < NW; q++)
      for (int k = 0; k < 5; k++) { tp.so[k] += s_v[q * TR_NV + k]; tp.sn[k] += s_v[q * TR_NV + 5 + k]; }
  } else {
    if (threadIdx.x) return;
    for (int k = 0; k < 5; k++) tp.so[k] = tp.sn[k] = 0.0;
  }
  // every control word the decision needs, loaded in one round with the
  // fixed-point totals (acquired with the CTA count; a value first read after
  // the branches below would cost an L2 round trip each)
  DevControl *C = A.ctrl;
  const int halt = C->halt, cur = C->cur, kind = C->stream.kind;
  const uint64_t used = C->zig_used, u_word = C->u_word, seq_next = C->seq_next;
  const uint64_t pos = C->stream.pos, inc = C->stream.s[1];
  const double e_old0 = C->ends_old[0], e_old1 = C->ends_old[1], e_new0 = C->ends_new[0], e_new1 = C->ends_new[1];
  const int ring_i = A.ring ? *A.ring_count : 0;
  const double cst = A.kdev ? A.kdev->hconst : A.k.hconst;
  // the fixed-point totals, then cleared for the next launch
  unsigned long long *fx = A.ctrl->fx;
  const __int128 a0 = fx_total(fx + 0), a1 = fx_total(fx + 3), a2 = fx_total(fx + 6);
  tp.flag = fx[9] ? 1.0 : 0.0;
  for (int k = 0; k < 10; k++) fx[k] = 0;
  st128(tp.dh, a0);
  st128(tp.hold, a1);
  st128(tp.hnew, a2);
  // tot: dH, H_old, H_new (variable parts), the moments (old 3..7, new 8..12), the flag (13)
  double tot[14];
  tot[0] = unfix128(a0);
  tot[1] = unfix128(a1);
  tot[2] = unfix128(a2);
  for (int k = 0; k < 5; k++) { tot[3 + k] = tp.so[k]; tot[8 + k] = tp.sn[k]; }
  tot[13] = tp.flag;
  C->tiles_done = 0;  // re-arm for the next launch
  C->tile_next = 0;
  C->t_stamp[3] = gtimer();
  if (halt) return;  // rsv_run_chain stopped at an earlier sweep: stream, path and statistics untouched
  if (A.shard) {  // time-sharded chain: the shards' records are combined by the decision
    *reinterpret_cast<TilePart *>(C->shard_parts) = tp;
    return;
  }
  DevResult r;
  r.h_old = tot[1] + cst;
  r.h_new = tot[2] + cst;
  r.accept = 0;
  r.u = __longlong_as_double(0x7ff8000000000000LL);
  r.words_used = 0;
  const bool flagged = tot[13] > 0.0;
  if (A.integrate_only) {
    // a non-finite final state only arises from a kick the reference flags
    // (NaN / inf are absorbing under the leapfrog map, _kernels.py:50-51);
    // the flag also covers energies beyond the fixed-point range
    r.diverged = flagged;
    r.delta_h = tot[0];
    C->res = r;
    return;
  }
  bool drew = false;
  const double dh = tot[0];
  if (flagged || !isfinite(dh) || fabs(dh) > 1000.0) {
    r.diverged = 1;
    r.delta_h = __longlong_as_double(0x7ff0000000000000LL);
  } else {
    r.diverged = 0;
    r.delta_h = dh;
    r.u = u01(u_word);  // raw word at stream position pos0 + used (momenta kernel)
    drew = true;
    r.accept = (dh <= 0.0) || (r.u < exp(-dh));
  }
  const uint64_t consumed = used + (drew ? 1 : 0);
  r.words_used = consumed;
  if (kind == PRNG_SFC64) {
    const uint64_t *q = A.sfc_snaps + 4 * (consumed / SFC_SNAP);
    uint64_t st[4] = {q[0], q[1], q[2], q[3]};
    for (uint64_t i = 0; i < consumed % SFC_SNAP; i++) sfc64_next(st);
    for (int i = 0; i < 4; i++) C->stream.s[i] = st[i];
  }
  C->stream.pos = pos + consumed;
  if (kind == PRNG_PCG32) {
    uint64_t q = seq_next;
    if (drew) { q = q * PCG_MULT + inc; q = q * PCG_MULT + inc; }
    C->seq_state = q;
  } else if (kind == PRNG_MINSTD) {
    uint64_t q = seq_next;
    if (drew) q = mod31(mod31(mod31(q * MINSTD_A) * MINSTD_A) * MINSTD_A);
    C->seq_state = q;
  }
  if (r.accept) C->cur = cur ^ 1;
  const double *sm = r.accept ? tot + 8 : tot + 3;
  C->stats[0] = r.accept ? e_new0 : e_old0;
  C->stats[1] = r.accept ? e_new1 : e_old1;
  for (int k = 0; k < 5; k++) C->stats[2 + k] = sm[k];
  C->res = r;
  if (A.ring) {  // batched proposals: the result ring (as ring_store_kernel)
    if (ring_i < A.ring_cap) A.ring[ring_i] = r;
    *A.ring_count = ring_i + 1;
  }
}

// Metropolis step of every chain of an ensemble (sampler.py:155-167 per
// chain), one thread per chain: sum the chain's tile records in tile order,
// decide with the chain's own uniform, keep the matching stream state, flip
// its buffer.
__global__ void ens_decide_kernel(TrajArgs A) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) {
    A.ctrl->t_stamp[3] = gtimer();
    A.ctrl->tile_next = 0;  // re-arm the trajectory kernel's dynamic tile counter
  }
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
