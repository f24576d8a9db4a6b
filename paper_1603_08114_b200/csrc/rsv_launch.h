// rsv_launch.h -- host-side launch wrappers of the kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "exp_table.h"
#include "rsv_internal.h"

namespace rsv {

struct MomentaBufs {
  DevControl *ctrl;
  void *scratch;        // momenta_scratch_bytes(T)
  uint64_t *sfc_words;  // SFC64 only: momenta_words(T) + 64 words
  uint64_t *sfc_snaps;  // SFC64 only: 4 * ((momenta_words(T) + 64) / SFC_SNAP + 1) words
  double *normals;      // T doubles
  const uint64_t *bjump;  // momenta_jump_bytes(T): per-CTA jump-ahead constants
  int64_t bjump_blocks = 0;  // blocks of the full draw the tables were built for (minstd's half follows pcg's)
  unsigned long long *dbg;  // optional per-CTA %globaltimer stamps (development aid)
  // blocked layout (config 5): one SFC64 stream per block of block_len sites
  EnsChain *blocks = nullptr;
  int64_t block_len = 0;
  int n_blocks = 0;
  int pdl = 0;  // launch the draw kernel as a programmatic dependent of the preceding kernel
};

int64_t momenta_words(int64_t T);
int momenta_init(cudaStream_t s, uint64_t *bjump, int64_t T);  // builds the jump-ahead tables
size_t momenta_jump_bytes(int64_t T);
size_t momenta_scratch_bytes(int64_t T);
int launch_momenta(const MomentaBufs &b, int kind, int64_t T, cudaStream_t s, int *launches);
int launch_momenta_advance(const MomentaBufs &b, cudaStream_t s, int *launches);
int launch_momenta_window(const MomentaBufs &b, int kind, const ZigWin &w, int nb, cudaStream_t s, int *launches);
int64_t momenta_blocks(int64_t T);  // CTAs (blocks of ZB words) of a full draw of T normals

// Tile geometry of the fused trajectory kernel for (T, n_steps).
struct TrajGeom {
  int64_t core;   // core sites per tile
  int halo;       // n_steps + 1
  int n_tiles;
  int ok;         // 0 if n_steps is too large for one tile (falls back to per-step passes)
  int variant;    // (sites/thread, threads/CTA, CTAs/SM) configuration, see leapfrog.cu
  int grid;       // CTAs launched (== n_tiles, or the persistent grid)
};
TrajGeom traj_geometry(int64_t T, int n_steps, int sm_count, int variant);
TrajGeom traj_geometry_ens(int64_t T, int64_t Tc, int n_steps, int sm_count);
const void *traj_kernel_fn_ens(int fuse);
const void *traj_kernel_fn_devk(int variant, int fuse);
int traj_num_variants();

// Trajectory constants derived on the host from (params, dt): passed by
// value in the kernel's parameter block so the hot loop reads them as
// constant-bank operands instead of holding ~30 registers.
struct TrajConsts {
  double mu, phi, dt, c_half, c_full, half_dt, alpha, bphi, g_int, g_end, emu, xm, inv2su, inv2se, one_m_phi2;
  double hconst;
  // The step loop runs on x = K (h - mu), K = 2048 / ln 2: the
  // drift and the kick's linear terms take their constants pre-scaled, and
  // e^{-d} = 2^{-x/2048} needs no Cody-Waite split (f = -x - rint(-x) is exact)
  double xc_half, xc_full, xg_int, xg_end, xbphi, kx, kxinv;
  double ex1, ex2, ex3;  // e^{f ln2/2048} - 1 = f (ex1 + f (ex2 + f ex3))
  int32_t n_lo, n_span;
};
__host__ __device__ inline TrajConsts traj_consts(const DevParams &P, double dt) {
  TrajConsts s;
  s.mu = P.mu;
  s.phi = P.phi;
  s.dt = dt;
  s.c_half = 0.5 * dt;
  s.c_full = dt;
  s.half_dt = 0.5 * dt;
  s.alpha = dt * P.inv_su2;
  const double beta = dt * P.inv_se2;
  s.bphi = beta * P.phi;
  s.g_int = s.alpha + beta * (2.0 - P.one_m_phi2);
  s.g_end = s.alpha + beta;
  s.emu = P.emu;
  s.xm = P.xi + P.mu;
  s.inv2su = 0.5 * P.inv_su2;
  s.inv2se = 0.5 * P.inv_se2;
  s.one_m_phi2 = P.one_m_phi2;
  s.hconst = P.hconst;
  s.kx = RSV_INV_LN2_N;
  s.kxinv = RSV_LN2_N_HI + RSV_LN2_N_LO;
  s.xc_half = s.c_half * s.kx;
  s.xc_full = s.c_full * s.kx;
  s.xg_int = s.g_int * s.kxinv;
  s.xg_end = s.g_end * s.kxinv;
  s.xbphi = s.bphi * s.kxinv;
  s.ex1 = s.kxinv;
  s.ex2 = 0.5 * s.kxinv * s.kxinv;
  s.ex3 = s.kxinv * s.kxinv * s.kxinv / 6.0;
  s.n_lo = P.n_lo;
  s.n_span = P.n_span;
  return s;
}


struct TrajArgs {
  TrajConsts k;
  int64_t T;            // local series length
  int64_t Tpad;         // arrays are allocated (and zero padded) to Tpad = roundup(T, 8)
  int64_t goff, Tg;     // global index of local site 0, global length (time sharding)
  int64_t own_lo, own_hi;  // local sites this context owns (reductions, write-back)
  int shard;            // 1: publish totals to ctrl->shard_parts instead of the Metropolis step
  int n_steps;
  int fuse;
  double dt;
  TrajGeom g;
  const double *h_src;  // if null: h buffers selected by ctrl->cur
  double *h_dst;
  // zero-copy input: sites [0, head_end) of h_src were copied to h_head by a
  // copy-engine node that ran beside the momenta kernel; windows inside it
  // are staged from there instead of over the link
  const double *h_head;
  int64_t head_end;
  double *hbuf0, *hbuf1;
  const double *p_in;
  double *p_out;        // optional
  const double *a;      // 0.5 y^2
  const double *lrv;
  const DevParams *prm;
  DevControl *ctrl;
  TilePart *parts;
  // Metropolis step folded into the last tile
  const uint64_t *sfc_snaps;
  int integrate_only;   // 1: only reduce (rsv_integrate): no Metropolis, no stream update
  int stats;            // compute the theta statistics of both paths (persistent kernel)
  unsigned long long *dbg;  // optional per-tile %globaltimer stamps (8 per tile), development aid
  // ensemble of independent chains: T = n_chains * Tc sites, chain-major;
  // Tc == 0 for a single chain
  int64_t Tc;
  int n_chains;
  int8_t *ens_cur;      // per chain: which h buffer holds its current path
  EnsPart *ens_parts;   // per tile: [2] partials
  EnsChain *ens;        // per chain bookkeeping
  // run_chain on the device: theta-dependent constants read from here (written
  // by the theta kernel); null: all constants from the parameter block
  const TrajConsts *kdev;
  int pdl;  // launched as a programmatic dependent of the momenta kernel
  // batched proposals (rsv_hmc_update_many): the Metropolis step appends its
  // result to this ring (null: the caller stores it)
  DevResult *ring;
  int32_t *ring_count;
  int ring_cap;
};
int launch_trajectory(const TrajArgs &a, cudaStream_t s, int *launches);
// ensemble: per-chain sfc64 momenta (numpy SFC64 + ziggurat, one thread per chain)
int launch_momenta_ens(EnsChain *ens, double *normals, int64_t Tc, int n_chains, cudaStream_t s, int *launches,
                       unsigned long long *dbg = nullptr, int advance = 0, const int32_t *halt = nullptr);
const void *traj_kernel_fn(int variant, int fuse, int stats);  // for locating the node in a captured graph
const void *traj_kernel_fn_head();  // the zero-copy instantiation that stages a copied head


// one streamed leapfrog step over all sites (integrator.py:139-146)
int launch_elementary_step(const double *h, const double *p, double *ho, double *po, const double *a,
                           const double *lrv, const DevParams *prm, double dt, int64_t T, int32_t *flag,
                           cudaStream_t s, int *launches, int pdl = 0);

// kernel-level plug-in (the reference's backend.run protocol)
int launch_position_update(double *h, const double *p, double c, int64_t lo, int64_t hi, cudaStream_t s,
                           int *launches);
struct PackedScal {  // model.py:185-199 scalar_pack
  double v[7];
};
int launch_momentum_update(const double *h, double *p, const double *y, const double *lrv, double dt,
                           PackedScal sc, int64_t n, int64_t lo, int64_t hi, int32_t *flag, cudaStream_t s,
                           int *launches);
int launch_gradient(const double *h, const double *y, const double *lrv, PackedScal sc, double *out, int64_t n,
                    int64_t lo, int64_t hi, int32_t *flag, cudaStream_t s, int *launches);

// deterministic reductions for hamiltonian / log_posterior / suff_stats
// out[0..7): see rsv_suff_stats; out for energy: {kinetic, -log f}
int launch_energy(const double *h, const double *p, const double *y, const double *lrv, const DevParams *prm,
                  int64_t T, double *partials, double *out, cudaStream_t s, int *launches);
int launch_suff_stats(const double *h, const double *lrv, int64_t T, double c_mu, double c_xi, double *partials,
                      double *out, cudaStream_t s, int *launches);
int reduce_partials_count(int64_t T);
// statistics shifted by the device-held parameters (mu, xi)
int launch_suff_stats_dev(const double *h, const double *lrv, int64_t T, const DevParams *prm, double *partials,
                          double *out, cudaStream_t s, int *launches);

// one Gibbs sweep's theta draws on the device (sampler.py:170-272, run_chain
// :327-344) after a proposal: updates *prm and *kdev, stores the sample
int launch_theta_sweep(DevControl *ctrl, DevParams *prm, TrajConsts *kdev, DevRun *run, DevPrior prior,
                       double dt, int64_t T, const uint64_t *sfc_snaps, cudaStream_t s, int *launches, int pdl = 0);

// data.py:72-95 simulate_rsv from 3T numpy normals already on the device;
// work: T + 2 * ceil((T-1)/256) doubles
int launch_simulate(const double *normals, int64_t T, double phi, double mu, double xi, double se2, double su2,
                    double *h, double *y, double *lrv, double *work, cudaStream_t s, int *launches);

}  // namespace rsv
