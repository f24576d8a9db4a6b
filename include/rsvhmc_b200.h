/*
 * rsvhmc_b200.h -- C ABI of the B200-native HMC volatility update of the
 * realized stochastic volatility (RSV) model (arXiv 1603.08114).
 *
 * This is the drop-in boundary for the reference's hot path.  Each entry
 * point names the reference interface it replaces (paths relative to the
 * reference tree, pkg/src/rsvhmc/...).  Plain pointers and sizes only; no
 * torch types.  All functions return 0 on success and a negative
 * RSV_E_* code on failure; rsv_last_error() returns the message.
 *
 * Pointers flagged `on_device` are CUDA device pointers (e.g. a torch
 * tensor's data_ptr()); otherwise they are host pointers and the call
 * copies synchronously.  One host thread per context.
 */
#ifndef RSVHMC_B200_H
#define RSVHMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSV_OK 0
#define RSV_E_INVALID -1   /* contract violation -> Python ValueError   */
#define RSV_E_CUDA -2      /* CUDA runtime failure -> RuntimeError      */
#define RSV_E_STATE -3     /* call order / missing data -> RuntimeError */
#define RSV_E_STORM -4     /* divergence storm in rsv_run_chain -> DivergenceStormError (sampler.py:39) */

/* Bit generator kinds.  Raw 64-bit words, numpy next_double convention
 * (word >> 11) * 2^-53 for every kind.
 *   PHILOX: numpy Philox4x64-10; s[0..1] = key, pos = words drawn.
 *   MINSTD: std::minstd_rand (a=48271, m=2^31-1); s[0] = x0;
 *           word n = x_{3n+1}<<33 | x_{3n+2}<<2 | x_{3n+3}>>29.
 *   PCG32 : pcg_basic pcg32; s[0] = LCG state after seeding, s[1] = inc;
 *           word n = out_{2n}<<32 | out_{2n+1}.
 *   SFC64 : numpy SFC64; s[0..3] = a, b, c, w at the current position. */
#define RSV_PRNG_PHILOX 0
#define RSV_PRNG_MINSTD 1
#define RSV_PRNG_PCG32 2
#define RSV_PRNG_SFC64 3

typedef struct {
  int32_t kind;
  int32_t reserved;
  uint64_t s[4];
  uint64_t pos; /* raw words drawn since seeding (informational for SFC64) */
} rsv_prng_state;

/* model.py:78-94 Params */
typedef struct {
  double phi, mu, xi, sigma_eta_sq, sigma_u_sq;
} rsv_params;

/* Outcome of one HMC proposal (sampler.py:144-167). */
typedef struct {
  int32_t accept;        /* proposal accepted                                  */
  int32_t diverged;      /* trajectory flagged (|h|>50 or NaN) or dH rejected  */
  double delta_h;        /* H_new - H_old, or +inf (sampler.py:31 sentinel)    */
  double h_old, h_new;   /* hamiltonian() before / after (model.py:178-182)    */
  uint64_t words_used;   /* raw words consumed: momenta (+1 uniform if drawn)  */
  double u;              /* the Metropolis uniform (NaN if none drawn)         */
} rsv_result;

/* sampler.py:43-63 PriorSpec */
typedef struct {
  double mu_mean, mu_var, xi_mean, xi_var, var_shape, var_scale, phi_a, phi_b;
} rsv_prior;

typedef struct rsv_ctx rsv_ctx;

const char *rsv_last_error(const rsv_ctx *ctx);
const char *rsv_version(void);

/* Context for one chain of length T on one CUDA device.  Owns device
 * buffers, a stream and cached CUDA graphs.  Replaces the implicit state of
 * sampler.py:291-358 run_chain (latent path, rng) for the device path. */
int rsv_create(rsv_ctx **out, int device, int64_t T);
int rsv_destroy(rsv_ctx *ctx);

/* Dataset (model.py:34-75): returns y_t and log realized variances. */
int rsv_set_data(rsv_ctx *ctx, const double *y, const double *log_rv, int on_device);
/* Params (model.py:78-94); validated like Params.__post_init__. */
int rsv_set_params(rsv_ctx *ctx, const rsv_params *p);
/* Latent path h (sampler.py:291-314 run_chain's h). */
int rsv_set_latent(rsv_ctx *ctx, const double *h, int on_device);
int rsv_get_latent(rsv_ctx *ctx, double *h, int on_device);
/* Bit-generator state (sampler.py:131-133 make_rng).  SFC64 states are
 * advanced on the device; the others are counter/jump-ahead based. */
int rsv_set_prng_state(rsv_ctx *ctx, const rsv_prng_state *st);
int rsv_get_prng_state(rsv_ctx *ctx, rsv_prng_state *st);

/* sampler.py:136-141 refresh_momenta: T standard normals, bit-exact with
 * numpy's Generator.standard_normal on the same stream; advances it. */
int rsv_refresh_momenta(rsv_ctx *ctx, double *p_out, int on_device);

/* sampler.py:144-167 hmc_update_volatility on the context's latent path:
 * momenta -> H_old -> L leapfrog steps -> H_new -> Metropolis, all on
 * device.  fuse != 0 selects integrate_trajectory(fuse_half_steps=True). */
int rsv_hmc_update(rsv_ctx *ctx, double step_size, int n_steps, int fuse, rsv_result *out);
/* sampler.py:144-167 in one call from host memory (the reference-facing
 * fast path of hmc_update_volatility): h_in (T doubles) and *stream in; when
 * the proposal is accepted it is written to h_out (otherwise h_out is left
 * untouched: the kept path is h_in); *stream advanced.  The theta statistics
 * are not evaluated.  When T >= 2^16, T % 8 == 0 and h_in is page-locked and
 * 16-byte aligned, the trajectory kernel reads h_in in place over PCIe
 * (zero copy, overlapped with its tiles) instead of one copy in ahead of the
 * proposal; rsv_last_update_zero_copy tells which way the last call went.
 * The context's own latent path afterwards: h_out when accepted; after a
 * rejected zero-copy call it holds none (rsv_set_latent before any
 * device-resident call such as rsv_hmc_update).  h_in == NULL proposes from
 * the path the context holds (RSV_E_STATE when it holds none): a chain driven
 * through this call then moves only its stream state in and, when accepted,
 * the proposal out. */
int rsv_hmc_update_host(rsv_ctx *ctx, const double *h_in, double *h_out, rsv_prng_state *stream, double step_size,
                        int n_steps, int fuse, rsv_result *out);
int rsv_last_update_zero_copy(const rsv_ctx *ctx);
/* n back-to-back proposals with fixed params (one CUDA graph per proposal,
 * no host round trip in between); results (n entries) optional.  Like the
 * reference's hmc_update_volatility these proposals do not evaluate the theta
 * statistics (rsv_last_stats is only valid after rsv_hmc_update). */
int rsv_hmc_update_many(rsv_ctx *ctx, double step_size, int n_steps, int fuse, int n, rsv_result *out);

/* integrator.py:149-179 integrate_trajectory from (h_in, p_in).
 * h_out/p_out may alias the inputs.  *diverged as the reference's flag. */
int rsv_integrate(rsv_ctx *ctx, const double *h_in, const double *p_in, double step_size, int n_steps, int fuse,
                  double *h_out, double *p_out, int32_t *diverged, int on_device);
/* integrator.py:139-146 elementary_step (K1 -> K2 -> K3 fused into one
 * streamed kernel), in place on (h, p). */
int rsv_elementary_step(rsv_ctx *ctx, double *h, double *p, double step_size, int32_t *diverged, int on_device);

/* Paper protocol (bench.py:121-190 time_elementary_step): n_steps streamed
 * elementary steps on a device-resident state (set by rsv_bench_state from
 * host arrays -- null keeps that half -- or left by the previous call /
 * rsv_elementary_step); *ms = device time of the n_steps launches,
 * *diverged = any step flagged |h| > 50 (may be null). */
int rsv_bench_state(rsv_ctx *ctx, const double *h, const double *p);
int rsv_bench_elementary(rsv_ctx *ctx, double step_size, int n_steps, float *ms, int32_t *diverged);
/* The same n steps fused into one launch of the persistent trajectory kernel
 * (state as for rsv_bench_elementary; device time of the launch in *ms). */
int rsv_bench_fused(rsv_ctx *ctx, double step_size, int n_steps, float *ms, int32_t *diverged);
/* The proposal's trajectory kernel alone, n launches back to back between
 * one CUDA event pair (integrate-only on the current path and momenta):
 * the per-launch duration bench.py's roofline divides by. */
int rsv_bench_trajectory(rsv_ctx *ctx, double step_size, int n_steps, int n, float *ms_per_launch);

/* Kernel-level plug-in (integrator.py:50-65 backend.run protocol):
 * _kernels.py:37-41 position_update, :44-54 momentum_update,
 * :57-67 gradient_fill on the index range [lo, hi) of length-n arrays.
 * scal[7] is model.py:185-199 scalar_pack order:
 * (half, phi, mu, xi, 1/sigma_u_sq, 1/sigma_eta_sq, 1 - phi^2). */
int rsv_position_update(rsv_ctx *ctx, double *h, const double *p, double c, int64_t n, int64_t lo, int64_t hi,
                        int on_device);
int rsv_momentum_update(rsv_ctx *ctx, const double *h, double *p, const double *y, const double *lrv, double dt,
                        const double *scal, int64_t n, int64_t lo, int64_t hi, int32_t *flag, int on_device);
int rsv_gradient(rsv_ctx *ctx, const double *h, const double *y, const double *lrv, const double *scal,
                 double *out, int64_t n, int64_t lo, int64_t hi, int32_t *flag, int on_device);

/* model.py:178-182 hamiltonian / :134-163 log_posterior of (h, p) against
 * the context's data and params. */
int rsv_hamiltonian(rsv_ctx *ctx, const double *h, const double *p, double *out, int on_device);
int rsv_log_posterior(rsv_ctx *ctx, const double *h, double *out, int on_device);

/* Sufficient statistics of the context's latent path for the theta full
 * conditionals (sampler.py:170-272), shifted by (c_mu, c_xi):
 *   out = {d_0, d_{T-1}, sum d, sum d^2, sum_{t>=1} d_t d_{t-1}, sum e, sum e^2}
 * with d = h - c_mu, e = log_rv - h - c_xi. */
int rsv_suff_stats(rsv_ctx *ctx, double c_mu, double c_xi, double out[7]);

/* Last proposal's statistics (computed inside the fused trajectory kernel
 * for whichever path was kept), shifted by the params' (mu, xi). */
int rsv_last_stats(rsv_ctx *ctx, double out[7]);

/* Device timing helpers for the benchmark: average duration (ms) of the
 * whole proposal (level 1: one CUDA event pair per proposal on the context's
 * stream around the proposal) and, at level 2, of its momenta and trajectory
 * parts (event nodes inside the proposal graph, which add their own latency)
 * over the last rsv_hmc_update_many call.  Level 0 disables timing. */
int rsv_set_timing(rsv_ctx *ctx, int level);
int rsv_get_timing(rsv_ctx *ctx, double *traj_ms, double *momenta_ms, double *total_ms);
/* Device-side orchestration of a sharded chain (no host synchronisation per
 * proposal; the host only enqueues): rsv_set_stream puts the context on an
 * external CUDA stream (e.g. the one NCCL collectives are ordered on; NULL
 * restores its own).  rsv_shard_propose_async writes this shard's 23-word totals
 * (rsv_shard_totals layout, u_word / words_used as bit patterns) to device
 * memory; after an all-gather of every rank's totals, rsv_shard_decide_async
 * takes the Metropolis decision on the device (exact integer sums of the
 * fixed-point dH / H parts, fixed-order compensated sums of the moments: the
 * same decision on every rank, and the same dH bits for any world size) and advances the stream / flips the path;
 * rsv_shard_halo_async packs the owned boundary sites of the current path
 * (unpack = 0: left gets [own_lo, own_lo + nl), right [own_hi - nr, own_hi))
 * or writes received margins (unpack = 1); rsv_shard_results returns the
 * decisions recorded since the last call. */
int rsv_set_stream(rsv_ctx *ctx, void *cuda_stream);
int rsv_shard_propose_async(rsv_ctx *ctx, double step_size, int n_steps, int fuse, int stats, double *totals_dev);
int rsv_shard_decide_async(rsv_ctx *ctx, const double *gathered_dev, int world);
/* builds the cached proposal graph ahead (before a caller-side stream capture
 * of the per-proposal sequence; inside a capture rsv_shard_propose_async
 * enqueues that graph's kernels directly) */
int rsv_shard_prepare(rsv_ctx *ctx, double step_size, int n_steps, int fuse, int stats);
int rsv_shard_halo_async(rsv_ctx *ctx, double *left, int64_t n_left, double *right, int64_t n_right, int unpack);
int rsv_shard_results(rsv_ctx *ctx, rsv_result *out, int max_n, int *n_out);

/* Time-sharded momenta (replaces sampler.py:136-141
 * refresh_momenta for one shard).  rsv_shard_set_momenta(ctx, 1) switches a
 * shard from drawing the whole series to parsing only a window of the
 * raw-word stream around its own sites (jump-ahead generators: philox,
 * pcg32, minstd; sfc64 uses rsv_shard_set_blocked_streams).  Per proposal:
 * rsv_shard_momenta_async writes this shard's 8-word window record to
 * device memory; after an all-gather of the records (rank order),
 * rsv_shard_place_async gives the window its global normal indices (the
 * exclusive prefix of the counts between anchor words), checks that
 * neighbouring windows agree on the attempt boundary at each anchor, and
 * places the shard's normals; then rsv_shard_propose_async runs the
 * trajectory only.  The normals are bit for bit those of the whole-series
 * draw. */
int rsv_shard_set_momenta(rsv_ctx *ctx, int windowed);
int rsv_shard_momenta_async(rsv_ctx *ctx, double *window_record_dev);
int rsv_shard_place_async(rsv_ctx *ctx, const double *gathered_records_dev, int world, int rank);
/* Peer-memory exchange of the per-proposal records (replaces the two NCCL
 * all-gathers of the protocol above by NVLink stores between the GPUs; the
 * reference's ΔH / statistics reduction, sampler.py:155-167 over the whole
 * series): every shard owns a small receive box.  rsv_shard_p2p_init
 * allocates it and returns its 64-byte CUDA IPC handle (and its device
 * address, for shards of the same process); rsv_shard_p2p_connect maps
 * every shard's box (boxes[q] != 0: that address, same device; otherwise
 * handles[64 q..] is opened over NVLink).  Per exchange (words = 23: shard
 * totals, 8: window records) every shard calls rsv_shard_p2p_push_async
 * with its own record, then rsv_shard_p2p_collect_async, which waits for
 * every shard's record of this exchange (flags written with release
 * semantics after the record; a missing peer raises an error after 5 s,
 * RSV_P2P_TIMEOUT_MS, instead of hanging) and copies the records out in rank order -- the
 * layout the all-gather produced, so rsv_shard_decide_async /
 * rsv_shard_place_async read it unchanged.  Shards of one process push all
 * before any of them collects. */
int rsv_shard_p2p_init(rsv_ctx *ctx, int world, int rank, unsigned char handle[64], uint64_t *box_dev);
int rsv_shard_p2p_connect(rsv_ctx *ctx, const unsigned char *handles, const uint64_t *boxes);
int rsv_shard_p2p_push_async(rsv_ctx *ctx, const double *record_dev, int words);
int rsv_shard_p2p_collect_async(rsv_ctx *ctx, double *records_out_dev, int words);
/* Blocked layout of a shard (config 5): the streams of the blocks
 * [first_block, first_block + n_blocks) its local range touches. */
int rsv_shard_set_blocked_streams(rsv_ctx *ctx, int64_t block_len, int64_t first_block, int64_t n_blocks,
                                  const uint64_t *states);
/* run_chain of a time-sharded chain (sampler.py:291-358): begin (prior,
 * schedule; theta constants move to device memory), then per sweep the
 * proposal protocol above with stats = 1, rsv_shard_decide_async, and
 * rsv_shard_theta_async (the theta draws of sampler.py:339-344 from the
 * all-gathered statistics of the kept path -- identical on every shard);
 * end copies the stored samples out (storm -> RSV_E_STORM as rsv_run_chain). */
int rsv_shard_run_begin(rsv_ctx *ctx, double step_size, const rsv_prior *prior, int64_t n_burnin, int64_t n_samples,
                        int64_t thin);
int rsv_shard_theta_async(rsv_ctx *ctx);
int rsv_shard_run_end(rsv_ctx *ctx, int64_t *iters, double *params, int32_t *accept, double *delta_h,
                      int64_t *n_stored, int64_t *storm_sweep);

/* data.py:72-95 simulate_rsv on the device: the reference's 3T normals
 * (initial deviation, innovations, return shocks, measurement noise) drawn
 * from *stream bit for bit (the stream is advanced), the AR(1) path by a
 * parallel affine scan (agrees with the sequential recursion to rounding),
 * h, returns and log_rv written to host (on_device = 0) or device buffers. */
int rsv_simulate(int device, const rsv_params *params, int64_t T, rsv_prng_state *stream, double *h, double *returns,
                 double *log_rv, int on_device);

/* Blocked momenta layout (BASELINE config 5; NOT the reference's single-stream
 * layout): SFC64 has no jump-ahead, so for very long series the
 * momenta of sites [j*block_len, (j+1)*block_len) come from their own numpy
 * SFC64 stream j (states: n_blocks x 4 words, the benchmark seeds stream j
 * with SeedSequence([seed, j])), continued from proposal to proposal; the
 * context's own stream then supplies only the Metropolis uniforms (and the
 * theta draws).  n_blocks * block_len must equal T.  states = NULL restores
 * the single-stream layout. */
int rsv_set_blocked_streams(rsv_ctx *ctx, int64_t block_len, int64_t n_blocks, const uint64_t *states);
int rsv_get_blocked_streams(rsv_ctx *ctx, uint64_t *states);

/* sampler.py:291-358 run_chain with the whole sweep on the device: starting
 * from the context's params, latent path and stream, n_burnin + n_samples *
 * thin sweeps of [hmc_update_volatility, update_mu, update_phi,
 * update_sigma_eta_sq, update_xi, update_sigma_u_sq] -- the theta draws by a
 * device thread on the same raw-word stream (numpy's normal / next_double /
 * gamma restated), no host round trip per sweep.  Stores every thin-th sweep
 * after the burn-in: iters[n_samples], params[n_samples x 5] (phi, mu, xi,
 * sigma_eta_sq, sigma_u_sq), accept[n_samples], delta_h[n_samples] (+inf:
 * divergent).  On a divergence storm (> 50 of 100 proposals, sampler.py:
 * 329-337) returns RSV_E_STORM with the sweep in *storm_sweep.  Afterwards the
 * context holds the final params, path and stream position. */
int rsv_run_chain(rsv_ctx *ctx, double step_size, int n_steps, int fuse, const rsv_prior *prior, int64_t n_burnin,
                  int64_t n_samples, int64_t thin, int64_t *iters, double *params, int32_t *accept,
                  double *delta_h, int64_t *storm_sweep);
int rsv_get_params(rsv_ctx *ctx, rsv_params *out);

/* ---- ensemble of independent chains (BASELINE config 4) ----
 * n_chains chains of T_chain sites each (chain-major arrays of
 * n_chains * T_chain doubles for rsv_set_data / rsv_set_latent /
 * rsv_get_latent), one shared parameter set, one numpy SFC64 stream per chain
 * (state words a, b, c, counter: chain c of the benchmark uses
 * SFC64(SeedSequence([seed, c]))).  One round = one hmc_update_volatility
 * (sampler.py:144-167) of every chain: momenta from the chain's own stream,
 * trajectory, per-chain dH and Metropolis test with the chain's own uniform.
 * The reference has no ensemble driver (SURVEY §2 K-ens); per chain the
 * result is exactly the reference's single-chain update. */
int rsv_ens_create(rsv_ctx **out, int device, int n_chains, int64_t T_chain);
int rsv_ens_set_streams(rsv_ctx *ctx, const uint64_t *states /* n_chains x 4 */);
int rsv_ens_get_streams(rsv_ctx *ctx, uint64_t *states /* n_chains x 4 */);
/* one momenta draw per chain (sampler.py:136-141); normals may be null */
int rsv_ens_refresh_momenta(rsv_ctx *ctx, double *normals /* n_chains x T_chain, host */);
/* n_rounds proposals of every chain; accept / delta_h (+inf: diverged) of
 * the last round per chain, either may be null */
int rsv_ens_hmc_update(rsv_ctx *ctx, double step_size, int n_steps, int fuse, int n_rounds, int32_t *accept,
                       double *delta_h);
/* accepted / diverged proposals per chain since rsv_ens_set_streams */
int rsv_ens_counts(rsv_ctx *ctx, int32_t *n_accept, int32_t *n_diverged);

/* %globaltimer stamps (ns) of the last proposal, taken inside the kernels:
 * [0] momenta kernel entry (first CTA), [1] its exit (last CTA), [2]
 * trajectory kernel entry (CTA 0), [3] its exit (Metropolis step), [4] the
 * previous proposal's trajectory exit.  No events, no added latency. */
int rsv_kernel_stamps(rsv_ctx *ctx, uint64_t out[5]);
/* Benchmark hygiene: with bytes > 0, rsv_hmc_update_many writes a
 * scratch buffer of that size between proposals (outside the timed events)
 * so each proposal starts with a cold L2. */
int rsv_set_l2_flush(rsv_ctx *ctx, int64_t bytes);
/* Measured FP64 FMA throughput of this device (DFMA microbenchmark),
 * in TFLOP/s (2 flops per FMA); *sm_mhz_est = implied average SM clock. */
int rsv_measure_fp64_peak(rsv_ctx *ctx, double *tflops);
/* Kernel launches issued by the context so far (gpu_launches evidence). */
int64_t rsv_launch_count(const rsv_ctx *ctx);

/* ---- time sharding: one chain split over several contexts / GPUs ----
 * (SURVEY §8e).  A shard context holds the global sites [local_start,
 * local_start + local_len) = the owned sites [lo, hi) plus a margin of at
 * least n_steps + 1 sites on each side (clamped at the series ends); the
 * margins are refreshed from the neighbours' owned sites before each
 * proposal.  rsv_set_data / rsv_set_latent take the local slices.  Every
 * shard draws the momenta of the whole series (same stream, same normals),
 * runs the trajectory on its local range and publishes its totals; the host
 * combines the shards' totals in rank order (bitwise independent of the
 * shard count's scheduling), decides (same u on every shard) and applies. */
typedef struct {
  int64_t dh[2];       /* dH over the owned sites: sum of per-group values (4-aligned groups of 4 global sites)
                          as 128-bit fixed point, value * 2^64 rounded toward zero, {low, high} words */
  int64_t h_old[2];    /* the variable part of H_old, same encoding */
  int64_t h_new[2];    /* the variable part of H_new, same encoding */
  double stats_old[5]; /* theta moments of the current path (sum d, d^2, d_t d_{t-1}, e, e^2) */
  double stats_new[5]; /* ... of the proposal */
  double flag;         /* > 0: a kick flagged |h| > 50 (or an energy beyond the fixed-point range) */
  double ends[4];      /* d_0 old, d_{T-1} old, d_0 new, d_{T-1} new (0 unless owned) */
  uint64_t u_word;     /* raw word after the momenta: the Metropolis uniform */
  uint64_t words_used; /* raw words consumed by the momenta */
} rsv_shard_totals;
int rsv_create_shard(rsv_ctx **out, int device, int64_t T_global, int64_t lo, int64_t hi, int64_t margin,
                     int64_t *local_start, int64_t *local_len);
int rsv_shard_propose(rsv_ctx *ctx, double step_size, int n_steps, int fuse, int stats, rsv_shard_totals *out);
int rsv_shard_apply(rsv_ctx *ctx, int accept, int drew_uniform);
/* copy [offset, offset + n) of the current local path to (to_ctx = 0) or
 * from (to_ctx = 1) buf -- the halo exchange of a sharded chain */
int rsv_latent_slice(rsv_ctx *ctx, int64_t offset, int64_t n, double *buf, int to_ctx, int on_device);

/* ---- host side of the bit generators (no device needed) ----
 * Seeding from raw seed material (numpy.SeedSequence words), sequential
 * draws, and a numpy bitgen_t so numpy.random.Generator continues the same
 * stream for the scalar theta draws (sampler.py:170-272).  Replaces
 * sampler.py:131-133 make_rng for the non-Philox kinds. */
int rsv_stream_seed(rsv_prng_state *st, int kind, const uint64_t *material);
uint64_t rsv_stream_next_u64(rsv_prng_state *st);
double rsv_stream_next_double(rsv_prng_state *st);
int rsv_stream_bitgen(rsv_prng_state *st, void *numpy_bitgen_out);
void rsv_philox_block(uint64_t block, uint64_t key0, uint64_t key1, uint64_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* RSVHMC_B200_H */
