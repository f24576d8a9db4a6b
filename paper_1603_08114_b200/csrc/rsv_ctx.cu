// rsv_ctx.cu -- the C ABI (include/rsvhmc_b200.h): device buffers, streams,
// CUDA-graph launch orchestration of one HMC proposal.
//
// One proposal (sampler.py:144-167 hmc_update_volatility) is the launch
// sequence  [SFC64 words] -> Z1 -> Z2 -> Z3 (momenta) -> trajectory -> accept,
// entirely device-resident: the stream position, the index of the current
// path buffer and the proposal outcome live in DevControl, so the sequence is
// captured once per (prng kind, dt, L, fuse) into a CUDA graph and replayed
// with no host round trip between proposals.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/rsvhmc_b200.h"
#include "exp_table.h"
#include "rsv_internal.h"
#include "rsv_launch.h"

using namespace rsv;

namespace {

struct GraphKey {
  int kind, n_steps, fuse, timing, stats;
  double dt;
  int zc = 0;     // zero-copy input (rsv_hmc_update_host): the trajectory reads h from host memory
  int nomom = 0;  // time-sharded windowed momenta: the normals are placed before the graph runs
  int devk = 0;   // theta constants from device memory (sharded run_chain)
  bool operator<(const GraphKey &o) const {
    return std::tie(kind, n_steps, fuse, timing, stats, dt, zc, nomom, devk) <
           std::tie(o.kind, o.n_steps, o.fuse, o.timing, o.stats, o.dt, o.zc, o.nomom, o.devk);
  }
};

// rsv_hmc_update_host reads a page-locked path in place from this length on
// (below it one copy in is as fast)
constexpr int64_t ZC_MIN_T = 1 << 16;
// share (in eighths) of a zero-copy path copied in by the copy engine, beside
// the momenta kernel, ahead of the trajectory (which reads the rest in place):
// the copy engine moves bytes faster than the kernel's in-place reads and
// the link is otherwise idle under the momenta kernel.  Measured at 2^20
// (tools/e2e_head_ab.py): 257 us per call without, 252 / 248 / 241 / 242 us
// with 1/16, 1/4, 3/8, 1/2 of the path.
constexpr int64_t ZC_HEAD_EIGHTHS = 3;
// host threads copying a pageable path into the page-locked staging buffer
constexpr int HOST_STAGE_THREADS = 8;

__global__ void prep_data_kernel(const double *y, double *a, int64_t T) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < T) a[i] = __dmul_rn(__dmul_rn(0.5, y[i]), y[i]);  // (half * y) * y, _kernels.py:27
}

// FP64 peak probe: 8 independent DFMA chains per thread, grid = 8 CTAs/SM.
__global__ void __launch_bounds__(256) dfma_peak_kernel(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void ring_store_kernel(DevControl *ctrl, DevResult *ring, int cap, int32_t *count) {
  if (threadIdx.x || blockIdx.x) return;
  const int i = *count;
  if (i < cap) ring[i] = ctrl->res;
  *count = i + 1;
}

__global__ void ens_gather_kernel(const double *h0, const double *h1, const int8_t *cur, int64_t Tc, int64_t T,
                                  double *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < T) out[i] = cur[i / Tc] ? h1[i] : h0[i];
}

__global__ void ens_advance_kernel(EnsChain *E, int C) {  // refresh_momenta alone: no uniform drawn
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C)
    for (int k = 0; k < 4; k++) E[c].st[k] = E[c].st_used[k];
}

}  // namespace

struct rsv_ctx {
  int device = 0;
  int64_t T = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  cudaStream_t own_stream = nullptr;  // set when an external stream is in use (rsv_set_stream)
  bool has_data = false, has_params = false, has_latent = false;
  int kind = PRNG_PHILOX;
  // time sharding: this context holds global sites [goff, goff + T) of a
  // series of Tg sites and owns [goff + own_lo, goff + own_hi)
  int64_t Tg = 0, goff = 0, own_lo = 0, own_hi = 0;
  bool shard = false;
  int64_t jump_T = 0;  // length the momenta jump tables cover (time-sharded: the windows' reach)
  // time-sharded windowed momenta (rsv_shard_set_momenta): this shard's window
  // of the raw-word stream, its anchors, and the parse outputs
  int win_mode = 0;
  // peer-memory record exchange (rsv_shard_p2p_*)
  P2PBox *p2p_box = nullptr;         // mine (receives every shard's records)
  P2PBox **p2p_peers = nullptr;      // device array: every shard's box, as this device sees it
  std::vector<void *> p2p_opened;    // boxes opened from IPC handles (closed on destroy)
  int p2p_world = 0, p2p_rank = 0;
  unsigned long long p2p_timeout_ns = 5000000000ull;  // RSV_P2P_TIMEOUT_MS (read at rsv_shard_p2p_init)
  int64_t win_wb0 = 0, win_nb = 0, win_cap = 0, win_a_lo = 0, win_a_hi = -1;
  double *win_out = nullptr;
  uint32_t *win_nend = nullptr;
  // sharded run_chain (rsv_shard_run_begin / _theta_async / _run_end)
  DevPrior run_prior{};
  double run_dt = 0.0;
  int run_active = 0;
  int variant = -1;  // automatic: persistent, TMA-staged, window size by T (traj_geometry in leapfrog.cu)
  unsigned long long *dbg = nullptr;  // RSV_TRAJ_STAMPS=1: per-tile timestamps

  double *hbuf[2] = {nullptr, nullptr};
  double *y = nullptr, *a = nullptr, *lrv = nullptr, *normals = nullptr;
  double *sh = nullptr, *sp = nullptr, *sh2 = nullptr, *sp2 = nullptr;  // scratch T each
  void *zscratch = nullptr;
  uint64_t *sfc_words = nullptr, *sfc_snaps = nullptr, *bjump = nullptr;
  TilePart *parts = nullptr;
  int max_tiles = 0;
  double *rpart = nullptr;  // reduction partials
  double *rout = nullptr;   // reduction outputs (8 doubles)
  double *fb = nullptr;     // long-trajectory fallback: energies and statistics (24 doubles)
  int zc_last = 0;  // the last rsv_hmc_update_host read h_in in place
  double *h_stage = nullptr;  // page-locked staging of a pageable path (rsv_hmc_update_host)
  int32_t *dflag = nullptr;
  int32_t *ring_count = nullptr;
  DevResult *ring = nullptr;
  int ring_cap = 0;
  DevControl *ctrl = nullptr;
  DevParams *prm = nullptr;
  // pinned host mirrors
  DevControl *h_ctrl = nullptr;
  DevParams *h_prm = nullptr;
  double *h_out = nullptr;  // 8 doubles
  int32_t *h_flag = nullptr;
  DevResult *h_ring = nullptr;
  int h_ring_cap = 0;
  // plug-in scratch (arbitrary n)
  double *pl[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t pl_n = 0;

  void *flush_buf = nullptr;
  int64_t flush_bytes = 0;
  struct Cached {
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    cudaGraphNode_t traj_node;
    cudaKernelNodeParams traj_params;
    cudaGraphNode_t head_node = nullptr;  // zero-copy graphs: the path's head, copied in beside the momenta
    const void *head_src = nullptr;
    size_t head_bytes = 0;
    TrajArgs args;
    double dt;
    std::vector<cudaGraphNode_t> ev;  // timing event-record nodes
    int launches = 0;                 // kernels per launch of the graph
  };
  std::map<GraphKey, Cached *> graphs;
  // rsv_hmc_update_many without per-proposal timing or L2 flush: one graph of
  // UPDATE_BATCH proposals (rebuilt when its key, its ring or the parameters change)
  Cached *batched = nullptr;
  GraphKey batched_key{};
  const DevResult *batched_ring = nullptr;
  int batched_ring_cap = 0;
  int timing = 0;  // 0 off, 1 per-proposal total, 2 with momenta / trajectory breakdown
  std::vector<cudaEvent_t> evpool;
  std::vector<double> last_traj_ms, last_mom_ms, last_total_ms;
  // ensemble of independent chains (rsv_ens_create): T = ens_C * ens_Tc
  int ens_C = 0;
  int64_t ens_Tc = 0;
  bool ens_streams = false;
  int8_t *ens_cur = nullptr;
  EnsPart *ens_parts = nullptr;
  EnsChain *ens = nullptr, *h_ens = nullptr;
  std::map<GraphKey, Cached *> ens_graphs;
  // blocked momenta streams (config 5): one SFC64 stream per block
  EnsChain *blocks = nullptr, *h_blocks = nullptr;
  int64_t block_len = 0;
  int n_blocks = 0;
  int64_t block_first = 0;  // time-sharded: the series block of this context's first block
  // run_chain on the device
  TrajConsts *kdev = nullptr;
  DevRun *run = nullptr;
  void *run_store = nullptr;
  int64_t run_cap = 0;
};

static std::string g_err;

static int fail(rsv_ctx *c, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_err = buf;
  return code;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(c, RSV_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define LK(call)                                                                                   \
  do {                                                                                             \
    if ((call) != 0)                                                                               \
      return fail(c, RSV_E_CUDA, "launch %s: %s", #call, cudaGetErrorString(cudaGetLastError())); \
  } while (0)

extern "C" {

const char *rsv_last_error(const rsv_ctx *c) { return c ? c->err.c_str() : g_err.c_str(); }
const char *rsv_version(void) { return "paper_1603_08114_b200 0.1.0 (sm_100a)"; }
int64_t rsv_launch_count(const rsv_ctx *c) { return c ? c->launches : 0; }

int rsv_destroy(rsv_ctx *c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto *m : {&c->graphs, &c->ens_graphs}) {
    for (auto &kv : *m) {
      cudaGraphExecDestroy(kv.second->exec);
      cudaGraphDestroy(kv.second->graph);
      delete kv.second;
    }
  }
  if (c->batched) {
    cudaGraphExecDestroy(c->batched->exec);
    cudaGraphDestroy(c->batched->graph);
    delete c->batched;
  }
  if (c->blocks) cudaFree(c->blocks);
  if (c->h_blocks) cudaFreeHost(c->h_blocks);
  if (c->win_out) cudaFree(c->win_out);
  if (c->win_nend) cudaFree(c->win_nend);
  for (void *q : c->p2p_opened) cudaIpcCloseMemHandle(q);
  if (c->p2p_peers) cudaFree(c->p2p_peers);
  if (c->p2p_box) cudaFree(c->p2p_box);
  if (c->kdev) cudaFree(c->kdev);
  if (c->run) cudaFree(c->run);
  if (c->run_store) cudaFree(c->run_store);
  if (c->ens_cur) cudaFree(c->ens_cur);
  if (c->ens_parts) cudaFree(c->ens_parts);
  if (c->ens) cudaFree(c->ens);
  if (c->h_ens) cudaFreeHost(c->h_ens);
  if (c->flush_buf) cudaFree(c->flush_buf);
  if (c->dbg) cudaFree(c->dbg);
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  void *dev[] = {c->hbuf[0], c->hbuf[1], c->y, c->a, c->lrv, c->normals, c->sh, c->sp, c->sh2, c->sp2,
                 c->zscratch, c->sfc_words, c->sfc_snaps, c->parts, c->rpart, c->rout, c->dflag, c->ring_count,
                 c->ring, c->ctrl, c->prm, c->pl[0], c->pl[1], c->pl[2], c->pl[3], c->bjump, c->fb};
  for (void *p : dev)
    if (p) cudaFree(p);
  void *host[] = {c->h_ctrl, c->h_prm, c->h_out, c->h_flag, c->h_ring};
  for (void *p : host)
    if (p) cudaFreeHost(p);
  if (c->own_stream) c->stream = c->own_stream;
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}

// Time-sharded windowed momenta: raw words per normal of numpy's ziggurat
// (1.0225 on average) and the slack around a shard's expected word range --
// the position of normal i wanders ~0.11 sqrt(i) words from i * rho, so the
// slack covers > 30 standard deviations at any length.
constexpr double WIN_RHO = 1.0225;
static int64_t shard_slack(int64_t Tg) { return 8192 + (int64_t)(4.0 * sqrt((double)Tg)); }
static int64_t shard_anchor(int64_t site) { return (int64_t)llround((double)site * WIN_RHO); }

// T: local series length; Tg: global length (== T unless time-sharded: the
// momenta are drawn for the whole series so every shard sees the same stream)
static int create_impl(rsv_ctx *c, int device, int64_t T, int64_t Tg) {
  c->device = device;
  c->T = T;
  c->Tg = Tg;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(c, RSV_E_CUDA, "built for sm_100a (B200); device is sm_%d%d", prop.major, prop.minor);
  c->sm_count = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  // zero-padded to a multiple of 8 doubles so tiles can be bulk-copied in 64 B units
  const size_t tb = sizeof(double) * (size_t)((T + 7) / 8 * 8);
  for (int i = 0; i < 2; i++) {
    CK(cudaMalloc(&c->hbuf[i], tb));
    CK(cudaMemset(c->hbuf[i], 0, tb));
  }
  double **bufs[] = {&c->y, &c->a, &c->lrv, &c->sh, &c->sp, &c->sh2, &c->sp2};
  for (double **b : bufs) {
    CK(cudaMalloc(b, tb));
    CK(cudaMemset(*b, 0, tb));
  }
  const size_t tbg = sizeof(double) * (size_t)((Tg + 7) / 8 * 8);
  CK(cudaMalloc(&c->normals, tbg));
  CK(cudaMemset(c->normals, 0, tbg));
  CK(cudaMalloc(&c->zscratch, momenta_scratch_bytes(Tg)));
  CK(cudaMemset(c->zscratch, 0, momenta_scratch_bytes(Tg)));  // look-back status words (epoch-tagged)
  const int64_t nw = momenta_words(Tg) + 64;
  CK(cudaMalloc(&c->sfc_words, sizeof(uint64_t) * nw));
  CK(cudaMalloc(&c->sfc_snaps, sizeof(uint64_t) * 4 * (nw / SFC_SNAP + 2)));
  c->max_tiles = (int)(T / 64 + 16 * c->sm_count + 8);
  if (c->max_tiles < (int)(momenta_words(Tg) / ZB) + 8) c->max_tiles = (int)(momenta_words(Tg) / ZB) + 8;
  if (const char *v = getenv("RSV_TRAJ_VARIANT")) c->variant = atoi(v);
  if (getenv("RSV_TRAJ_STAMPS") || getenv("RSV_ZIG_STAMPS") || getenv("RSV_ENS_STAMPS")) {
    CK(cudaMalloc(&c->dbg, sizeof(unsigned long long) * 8 * c->max_tiles));
    CK(cudaMemset(c->dbg, 0, sizeof(unsigned long long) * 8 * c->max_tiles));
  }
  CK(cudaMalloc(&c->parts, sizeof(TilePart) * c->max_tiles));
  CK(cudaMalloc(&c->rpart, sizeof(double) * 8 * (reduce_partials_count(T) + 1)));
  CK(cudaMalloc(&c->rout, sizeof(double) * 8));
  CK(cudaMalloc(&c->fb, sizeof(double) * 24));
  CK(cudaMalloc(&c->dflag, sizeof(int32_t)));
  CK(cudaMalloc(&c->ring_count, sizeof(int32_t)));
  CK(cudaMemset(c->ring_count, 0, sizeof(int32_t)));
  CK(cudaMalloc(&c->ctrl, sizeof(DevControl)));
  CK(cudaMalloc(&c->prm, sizeof(DevParams)));
  CK(cudaMallocHost(&c->h_ctrl, sizeof(DevControl)));
  CK(cudaMallocHost(&c->h_prm, sizeof(DevParams)));
  CK(cudaMallocHost(&c->h_out, sizeof(double) * 8));
  CK(cudaMallocHost(&c->h_flag, sizeof(int32_t)));
  memset(c->h_ctrl, 0, sizeof(DevControl));
  c->h_ctrl->stream.kind = PRNG_PHILOX;
  CK(cudaMemcpy(c->ctrl, c->h_ctrl, sizeof(DevControl), cudaMemcpyHostToDevice));
  // time-sharded contexts parse windows that reach a little past the
  // expected end of the draw (shard_window): their jump tables cover it
  c->jump_T = c->shard ? Tg + 2 * shard_slack(Tg) + 4 * (int64_t)ZB : Tg;
  CK(cudaMalloc(&c->bjump, momenta_jump_bytes(c->jump_T)));
  if (momenta_init(c->stream, c->bjump, c->jump_T)) return fail(c, RSV_E_CUDA, "momenta table init failed");
  c->launches += 2;
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int rsv_create(rsv_ctx **out, int device, int64_t T) {
  if (!out) return fail(nullptr, RSV_E_INVALID, "out is null");
  *out = nullptr;
  if (T < 2) return fail(nullptr, RSV_E_INVALID, "need at least 2 sites, got %lld", (long long)T);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, RSV_E_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, RSV_E_INVALID, "device %d out of range", device);
  rsv_ctx *c = new rsv_ctx();
  c->own_lo = 0;
  c->own_hi = T;
  const int r = create_impl(c, device, T, T);
  if (r) {
    g_err = c->err;
    rsv_destroy(c);
    return r;
  }
  *out = c;
  return 0;
}

static int copy_in(rsv_ctx *c, double *dst, const double *src, int64_t n, int on_device) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     c->stream));
  return 0;
}
static int copy_out(rsv_ctx *c, double *dst, const double *src, int64_t n, int on_device) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     c->stream));
  return 0;
}
static int sync(rsv_ctx *c) {
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}
static int pull_ctrl(rsv_ctx *c) {
  CK(cudaMemcpyAsync(c->h_ctrl, c->ctrl, sizeof(DevControl), cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

int rsv_set_data(rsv_ctx *c, const double *y, const double *log_rv, int on_device) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!y || !log_rv) return fail(c, RSV_E_INVALID, "null data pointer");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = copy_in(c, c->y, y, c->T, on_device))) return r;
  if ((r = copy_in(c, c->lrv, log_rv, c->T, on_device))) return r;
  prep_data_kernel<<<(unsigned)((c->T + 255) / 256), 256, 0, c->stream>>>(c->y, c->a, c->T);
  c->launches++;
  CK(cudaGetLastError());
  c->has_data = true;
  return sync(c);
}

static int check_params(rsv_ctx *c, const rsv_params *p) {
  if (!p) return fail(c, RSV_E_INVALID, "null params");
  if (!(fabs(p->phi) < 1.0)) return fail(c, RSV_E_INVALID, "|phi| must be < 1 for stationarity, got %g", p->phi);
  if (!(p->sigma_eta_sq > 0.0)) return fail(c, RSV_E_INVALID, "sigma_eta_sq must be positive, got %g", p->sigma_eta_sq);
  if (!(p->sigma_u_sq > 0.0)) return fail(c, RSV_E_INVALID, "sigma_u_sq must be positive, got %g", p->sigma_u_sq);
  return 0;
}

static int refresh_graph_params(rsv_ctx *c);

int rsv_set_params(rsv_ctx *c, const rsv_params *p) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  int r = check_params(c, p);
  if (r) return r;
  CK(cudaSetDevice(c->device));
  // the previous graph replays may still read *prm: order the update on the stream
  CK(cudaStreamSynchronize(c->stream));
  DevParams &q = *c->h_prm;
  q.phi = p->phi;
  q.mu = p->mu;
  q.xi = p->xi;
  q.se2 = p->sigma_eta_sq;
  q.su2 = p->sigma_u_sq;
  q.inv_su2 = 1.0 / q.su2;
  q.inv_se2 = 1.0 / q.se2;
  q.emu = exp(-q.mu);
  q.one_m_phi2 = 1.0 - q.phi * q.phi;
  const double Td = (double)(c->shard ? c->Tg : c->T);  // a shard's H constant is the whole series'
  q.hconst = 0.5 * Td * q.mu + 0.5 * Td * log(q.su2) + 0.5 * log(q.se2 / (1.0 - q.phi * q.phi)) +
             0.5 * (Td - 1.0) * log(q.se2);
  q.n_lo = (int32_t)floor((q.mu - 50.0) * RSV_INV_LN2_N);
  q.n_span = (int32_t)ceil((q.mu + 50.0) * RSV_INV_LN2_N) - q.n_lo;
  CK(cudaMemcpyAsync(c->prm, c->h_prm, sizeof(DevParams), cudaMemcpyHostToDevice, c->stream));
  c->has_params = true;
  return refresh_graph_params(c);
}

// the trajectory reads the derived constants from its parameter block:
// update the kernel node of every cached graph after a parameter change
static void drop_batched(rsv_ctx *c) {
  if (!c->batched) return;
  cudaGraphExecDestroy(c->batched->exec);
  cudaGraphDestroy(c->batched->graph);
  delete c->batched;
  c->batched = nullptr;
}

static int refresh_graph_params(rsv_ctx *c) {
  drop_batched(c);  // its trajectory nodes carry the old constants: rebuilt on demand
  const DevParams &q = *c->h_prm;
  for (auto *m : {&c->graphs, &c->ens_graphs}) {
    for (auto &kv : *m) {
      auto *g = kv.second;
      if (!g->traj_node) continue;  // graphs without a trajectory node (paper protocol)
      g->args.k = traj_consts(q, g->dt);
      void *kp[] = {&g->args};
      cudaKernelNodeParams np = g->traj_params;
      np.kernelParams = kp;
      CK(cudaGraphExecKernelNodeSetParams(g->exec, g->traj_node, &np));
    }
  }
  return sync(c);
}

int rsv_set_latent(rsv_ctx *c, const double *h, int on_device) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!h) return fail(c, RSV_E_INVALID, "null latent pointer");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = copy_in(c, c->hbuf[0], h, c->T, on_device))) return r;
  CK(cudaMemsetAsync(&c->ctrl->cur, 0, sizeof(int32_t), c->stream));
  if (c->ens_cur) CK(cudaMemsetAsync(c->ens_cur, 0, (size_t)c->ens_C, c->stream));
  c->has_latent = true;
  return sync(c);
}

int rsv_get_latent(rsv_ctx *c, double *h, int on_device) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!c->has_latent) return fail(c, RSV_E_STATE, "latent path not set");
  CK(cudaSetDevice(c->device));
  int r;
  if (c->ens_C) {  // ensemble: every chain's current buffer
    double *dst = h;
    if (!on_device) dst = c->sh;
    ens_gather_kernel<<<(unsigned)((c->T + 255) / 256), 256, 0, c->stream>>>(c->hbuf[0], c->hbuf[1], c->ens_cur,
                                                                           c->ens_Tc, c->T, dst);
    c->launches++;
    CK(cudaGetLastError());
    if (!on_device && (r = copy_out(c, h, c->sh, c->T, 0))) return r;
    return sync(c);
  }
  if ((r = pull_ctrl(c))) return r;
  if ((r = copy_out(c, h, c->hbuf[c->h_ctrl->cur & 1], c->T, on_device))) return r;
  return sync(c);
}

int rsv_set_prng_state(rsv_ctx *c, const rsv_prng_state *st) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!st || st->kind < 0 || st->kind > 3) return fail(c, RSV_E_INVALID, "invalid bit generator state");
  if (st->kind == PRNG_MINSTD && (st->s[0] == 0 || st->s[0] >= MINSTD_M))
    return fail(c, RSV_E_INVALID, "minstd state must be in [1, 2^31-2]");
  CK(cudaSetDevice(c->device));
  StreamState s;
  s.kind = st->kind;
  s.reserved = 0;
  for (int i = 0; i < 4; i++) s.s[i] = st->s[i];
  s.pos = st->pos;
  CK(cudaStreamSynchronize(c->stream));
  c->h_ctrl->stream = s;
  CK(cudaMemcpyAsync(&c->ctrl->stream, &c->h_ctrl->stream, sizeof(StreamState), cudaMemcpyHostToDevice, c->stream));
  uint64_t seq = 0;
  if (s.kind == PRNG_PCG32) seq = pcg_advance(s.s[0], 2 * s.pos, s.s[1]);
  else if (s.kind == PRNG_MINSTD) seq = mod31(minstd_pow(3 * s.pos) * s.s[0]);
  c->h_ctrl->seq_state = seq;
  CK(cudaMemcpyAsync(&c->ctrl->seq_state, &c->h_ctrl->seq_state, sizeof(uint64_t), cudaMemcpyHostToDevice,
                     c->stream));
  c->kind = st->kind;
  return sync(c);
}

int rsv_get_prng_state(rsv_ctx *c, rsv_prng_state *st) {
  if (!c || !st) return fail(c, RSV_E_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = pull_ctrl(c))) return r;
  st->kind = c->h_ctrl->stream.kind;
  st->reserved = 0;
  for (int i = 0; i < 4; i++) st->s[i] = c->h_ctrl->stream.s[i];
  st->pos = c->h_ctrl->stream.pos;
  return 0;
}

static MomentaBufs mbufs(rsv_ctx *c) {
  MomentaBufs b;
  b.ctrl = c->ctrl;
  b.scratch = c->zscratch;
  b.sfc_words = c->sfc_words;
  b.sfc_snaps = c->sfc_snaps;
  b.normals = c->normals;
  b.bjump = c->bjump;
  b.bjump_blocks = momenta_blocks(c->jump_T ? c->jump_T : c->Tg);
  b.dbg = getenv("RSV_ZIG_STAMPS") ? c->dbg : nullptr;
  b.blocks = c->blocks;
  if (c->blocks) b.normals = c->normals + c->block_first * c->block_len;  // a shard's first block
  b.block_len = c->block_len;
  b.n_blocks = c->n_blocks;
  return b;
}

static void drop_graphs(rsv_ctx *c) {  // the momenta layout changed: recapture
  drop_batched(c);
  for (auto &kv : c->graphs) {
    cudaGraphExecDestroy(kv.second->exec);
    cudaGraphDestroy(kv.second->graph);
    delete kv.second;
  }
  c->graphs.clear();
}

static int check_err_bits(rsv_ctx *c) {
  if (c->h_ctrl->err & 1) return fail(c, RSV_E_CUDA, "momenta word budget exhausted (ziggurat shortfall)");
  if (c->h_ctrl->err & 16)
    return fail(c, RSV_E_CUDA, "sharded momenta: neighbouring windows disagree on an attempt boundary");
  if (c->h_ctrl->err & 32) return fail(c, RSV_E_CUDA, "sharded momenta: a window does not cover its shard");
  if (c->h_ctrl->err & 4) return fail(c, RSV_E_CUDA, "ensemble momenta: a tail draw needed > 30 loops");
  if (c->h_ctrl->err & 64)
    return fail(c, RSV_E_CUDA, "sharded chain: a peer's record did not arrive within the timeout (peer exchange)");
  return 0;
}

int rsv_refresh_momenta(rsv_ctx *c, double *p_out, int on_device) {
  if (!c || !p_out) return fail(c, RSV_E_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  int l = 0;
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  if (launch_momenta(mbufs(c), c->kind, c->Tg, c->stream, &l)) return fail(c, RSV_E_CUDA, "momenta launch failed");
  if (launch_momenta_advance(mbufs(c), c->stream, &l)) return fail(c, RSV_E_CUDA, "advance launch failed");
  c->launches += l;
  int r;
  if ((r = copy_out(c, p_out, c->normals, c->Tg, on_device))) return r;
  if ((r = pull_ctrl(c))) return r;
  return check_err_bits(c);
}

static TrajArgs traj_args(rsv_ctx *c, double dt, int n_steps, int fuse, const TrajGeom &g) {
  TrajArgs a;
  memset(&a, 0, sizeof(a));
  a.k = traj_consts(*c->h_prm, dt);
  a.T = c->T;
  a.Tpad = (c->T + 7) / 8 * 8;
  a.n_steps = n_steps;
  a.fuse = fuse;
  a.dt = dt;
  a.g = g;
  a.hbuf0 = c->hbuf[0];
  a.hbuf1 = c->hbuf[1];
  a.p_in = c->normals + c->goff;
  a.goff = c->goff;
  a.Tg = c->Tg;
  a.own_lo = c->own_lo;
  a.own_hi = c->own_hi;
  a.shard = c->shard ? 1 : 0;
  a.a = c->a;
  a.lrv = c->lrv;
  a.prm = c->prm;
  a.ctrl = c->ctrl;
  a.parts = c->parts;
  a.sfc_snaps = c->sfc_snaps;
  a.integrate_only = 0;
  a.dbg = getenv("RSV_TRAJ_STAMPS") ? c->dbg : nullptr;
  return a;
}

static int check_md(rsv_ctx *c, double dt, int n_steps) {
  if (!(dt > 0.0)) return fail(c, RSV_E_INVALID, "step_size must be positive, got %g", dt);
  if (n_steps < 1) return fail(c, RSV_E_INVALID, "n_steps must be >= 1, got %d", n_steps);
  return 0;
}

static int ensure_events(rsv_ctx *c, size_t n) {
  while (c->evpool.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->evpool.push_back(e);
  }
  return 0;
}

// ---- trajectories longer than a tile's halo allows (L > ~360 at 256
// threads): the proposal as streamed elementary steps (the reference's
// K1-K2-K3 grouping, integrator.py:139-146), H by the deterministic
// reductions, and a one-thread Metropolis step (sampler.py:155-167).  Every
// parameter is read from device memory, so device-side theta updates work too.
__global__ void fb_take_current_kernel(const DevControl *C, const double *h0, const double *h1, double *dst,
                                       int64_t T) {
  const double *src = C->cur ? h1 : h0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void fb_put_proposal_kernel(const DevControl *C, const double *src, double *h0, double *h1, int64_t T) {
  double *dst = C->cur ? h0 : h1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__device__ void shard_advance(DevControl *C, int drew, const uint64_t *snaps);
// e: [0..1] old {kinetic, log f}, [2..3] new, [4..10] old statistics, [11..17] new statistics
__global__ void fb_metropolis_kernel(DevControl *C, const double *e, const int32_t *flag, const uint64_t *snaps,
                                     int stats) {
  if (threadIdx.x || blockIdx.x) return;
  DevResult r;
  r.h_old = e[0] - e[1];
  r.h_new = e[2] - e[3];
  r.accept = 0;
  r.u = __longlong_as_double(0x7ff8000000000000LL);
  const double dh = r.h_new - r.h_old;
  bool drew = false;
  if (*flag || !isfinite(dh) || fabs(dh) > 1000.0) {
    r.diverged = 1;
    r.delta_h = __longlong_as_double(0x7ff0000000000000LL);
  } else {
    r.diverged = 0;
    r.delta_h = dh;
    r.u = u01(C->u_word);
    drew = true;
    r.accept = (dh <= 0.0) || (r.u < exp(-dh));
  }
  r.words_used = C->zig_used + (drew ? 1 : 0);
  shard_advance(C, drew, snaps);
  if (r.accept) C->cur ^= 1;
  if (stats)
    for (int k = 0; k < 7; k++) C->stats[k] = r.accept ? e[11 + k] : e[4 + k];
  C->res = r;
}

static bool enqueue_fallback(rsv_ctx *c, double dt, int n_steps, int stats, int *l) {
  bool ok = cudaMemsetAsync(c->dflag, 0, sizeof(int32_t), c->stream) == cudaSuccess;
  const unsigned nb = (unsigned)((c->T + 255) / 256 < 4096 ? (c->T + 255) / 256 : 4096);
  fb_take_current_kernel<<<nb, 256, 0, c->stream>>>(c->ctrl, c->hbuf[0], c->hbuf[1], c->sh, c->T);
  ok &= launch_energy(c->sh, c->normals, c->y, c->lrv, c->prm, c->T, c->rpart, c->fb + 0, c->stream, l) == 0;
  if (stats) ok &= launch_suff_stats_dev(c->sh, c->lrv, c->T, c->prm, c->rpart, c->fb + 4, c->stream, l) == 0;
  const double *hin = c->sh, *pin = c->normals;
  double *ho = c->sh2, *po = c->sp2;
  for (int k = 0; k < n_steps; k++) {
    ok &= launch_elementary_step(hin, pin, ho, po, c->a, c->lrv, c->prm, dt, c->T, c->dflag, c->stream, l, 1) == 0;
    hin = ho;
    pin = po;
    ho = (ho == c->sh2) ? c->sh : c->sh2;
    po = (po == c->sp2) ? c->sp : c->sp2;
  }
  ok &= launch_energy(hin, pin, c->y, c->lrv, c->prm, c->T, c->rpart, c->fb + 2, c->stream, l) == 0;
  if (stats) ok &= launch_suff_stats_dev(hin, c->lrv, c->T, c->prm, c->rpart, c->fb + 11, c->stream, l) == 0;
  fb_put_proposal_kernel<<<nb, 256, 0, c->stream>>>(c->ctrl, hin, c->hbuf[0], c->hbuf[1], c->T);
  fb_metropolis_kernel<<<1, 1, 0, c->stream>>>(c->ctrl, c->fb, c->dflag, c->sfc_snaps, stats);
  *l += 3;
  return ok && cudaGetLastError() == cudaSuccess;
}

// Capture one proposal into a graph.  With timing, 4 event-record nodes
// (start, trajectory begin, trajectory end, end) are added; their events are
// re-pointed per launch with cudaGraphExecEventRecordNodeSetEvent.
static bool variant_is_persistent(int v) { return v >= 9; }

static int build_graph(rsv_ctx *c, const GraphKey &k, rsv_ctx::Cached **out, const void *head_src = nullptr) {
  const TrajGeom g = traj_geometry(c->T, k.n_steps, c->sm_count, c->variant);
  if (!g.ok && c->shard) return fail(c, RSV_E_INVALID, "n_steps=%d too large for a sharded trajectory", k.n_steps);
  if (g.ok && g.n_tiles > c->max_tiles) return fail(c, RSV_E_CUDA, "tile count %d exceeds buffer", g.n_tiles);
  int r;
  if ((r = ensure_events(c, 4))) return r;
  auto *cg = new rsv_ctx::Cached();
  cg->dt = k.dt;
  cg->args = traj_args(c, k.dt, k.n_steps, k.fuse, g);
  cg->args.stats = k.stats;
  if (k.devk) {
    if (!g.ok || g.variant < 11 || g.variant > 14 || !c->kdev)
      return fail(c, RSV_E_STATE, "sharded run_chain needs a persistent trajectory shape");
    cg->args.kdev = c->kdev;
  }
  if (k.zc && g.ok) {  // h_src is re-pointed at the caller's page-locked path per call
    cg->args.h_src = c->hbuf[0];
    cg->args.h_dst = c->hbuf[1];
    if (head_src) {
      const int64_t head = getenv("RSV_ZC_HEAD") ? atoll(getenv("RSV_ZC_HEAD")) : c->T * ZC_HEAD_EIGHTHS / 8;
      const int64_t he = std::min<int64_t>(head, c->T) / 8 * 8;
      const bool use = he > 0 && g.variant == 11 && !k.stats;  // the instantiation that has the head
      cg->args.h_head = use ? c->hbuf[0] : nullptr;
      cg->args.head_end = use ? he : 0;
    }
  }
  // programmatic dependent launch of the trajectory after the momenta kernel
  // (not with timing event nodes between them)
  cg->args.pdl = (k.timing == 0 && !k.nomom && variant_is_persistent(g.variant) && !getenv("RSV_NO_PDL")) ? 1 : 0;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int l = 0;
  bool ok = true;
  if (k.timing) cudaEventRecordWithFlags(c->evpool[0], c->stream, cudaEventRecordExternal);
  if (!k.nomom) ok &= launch_momenta(mbufs(c), k.kind, c->Tg, c->stream, &l) == 0;
  if (k.timing) cudaEventRecordWithFlags(c->evpool[1], c->stream, cudaEventRecordExternal);
  if (g.ok) ok &= launch_trajectory(cg->args, c->stream, &l) == 0;
  else ok &= enqueue_fallback(c, k.dt, k.n_steps, k.stats, &l);
  if (k.timing) cudaEventRecordWithFlags(c->evpool[2], c->stream, cudaEventRecordExternal);
  if (k.timing) cudaEventRecordWithFlags(c->evpool[3], c->stream, cudaEventRecordExternal);
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (!ok || e != cudaSuccess) {
    delete cg;
    return fail(c, RSV_E_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
  }
  cg->graph = graph;
  size_t n = 0;
  CK(cudaGraphGetNodes(graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CK(cudaGraphGetNodes(graph, nodes.data(), &n));
  const void *fn = !g.ok                ? nullptr
                   : k.devk             ? traj_kernel_fn_devk(g.variant, k.fuse)
                   : cg->args.h_head    ? traj_kernel_fn_head()
                                        : traj_kernel_fn(g.variant, k.fuse, k.stats);
  cg->traj_node = nullptr;
  cg->launches = l;
  cg->ev.assign(4, nullptr);
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) {
      cudaKernelNodeParams kp;
      CK(cudaGraphKernelNodeGetParams(nd, &kp));
      if (fn && kp.func == fn) {
        cg->traj_node = nd;
        cg->traj_params = kp;
      }
    } else if (t == cudaGraphNodeTypeEventRecord) {
      cudaEvent_t ev;
      cudaGraphEventRecordNodeGetEvent(nd, &ev);
      for (int i = 0; i < 4; i++)
        if (ev == c->evpool[i]) cg->ev[i] = nd;
    }
  }
  if (g.ok && !cg->traj_node) return fail(c, RSV_E_CUDA, "trajectory node not found in the captured graph");
  if (k.zc && g.ok && head_src && cg->args.head_end > 0) {
    // the copy engine brings the path's first sites in while the momenta
    // kernel runs (the link is otherwise idle then); the trajectory kernel
    // (a full dependent of the copy) stages windows inside it from device memory
    cg->head_bytes = sizeof(double) * (size_t)cg->args.head_end;
    cg->head_src = head_src;
    CK(cudaGraphAddMemcpyNode1D(&cg->head_node, graph, nullptr, 0, c->hbuf[0], head_src, cg->head_bytes,
                                cudaMemcpyHostToDevice));
    CK(cudaGraphAddDependencies(graph, &cg->head_node, &cg->traj_node, 1));
  }
  if (k.timing)
    for (int i = 0; i < 4; i++)
      if (!cg->ev[i]) return fail(c, RSV_E_CUDA, "timing graph: event node %d not found", i);
  CK(cudaGraphInstantiate(&cg->exec, graph, 0));
  *out = cg;
  return 0;
}

static int get_graph(rsv_ctx *c, double dt, int n_steps, int fuse, int stats, rsv_ctx::Cached **out,
                     int *kernels, int zc = 0, const void *head_src = nullptr) {
  GraphKey k{c->kind, n_steps, fuse ? 1 : 0, c->timing == 2 ? 1 : 0, stats ? 1 : 0, dt, zc};
  k.nomom = c->shard && c->win_mode && !c->blocks ? 1 : 0;
  k.devk = c->shard && c->run_active && stats ? 1 : 0;
  auto it = c->graphs.find(k);
  if (it == c->graphs.end()) {
    rsv_ctx::Cached *cg = nullptr;
    int r = build_graph(c, k, &cg, head_src);
    if (r) return r;
    it = c->graphs.emplace(k, cg).first;
  }
  *out = it->second;
  *kernels = it->second->launches;
  return 0;
}

static int ready(rsv_ctx *c) {
  if (!c->has_data) return fail(c, RSV_E_STATE, "data not set (rsv_set_data)");
  if (!c->has_params) return fail(c, RSV_E_STATE, "params not set (rsv_set_params)");
  if (!c->has_latent) return fail(c, RSV_E_STATE, "latent path not set (rsv_set_latent)");
  return 0;
}

static void to_result(const DevResult &d, rsv_result *o) {
  o->accept = d.accept;
  o->diverged = d.diverged;
  o->delta_h = d.delta_h;
  o->h_old = d.h_old;
  o->h_new = d.h_new;
  o->words_used = d.words_used;
  o->u = d.u;
}

// UPDATE_BATCH proposals as one graph: momenta (a programmatic dependent of
// the previous trajectory from the second proposal on) and trajectory, the
// result ring written by the Metropolis step -- no graph-to-graph gap and no
// ring-store kernel between proposals.
constexpr int UPDATE_BATCH = 8;
static int get_batched(rsv_ctx *c, double dt, int n_steps, int fuse, bool results, rsv_ctx::Cached **out) {
  *out = nullptr;
  GraphKey k{c->kind, n_steps, fuse ? 1 : 0, 0, 0, dt};
  const DevResult *ring = results ? c->ring : nullptr;
  // (the ring's capacity too: a reallocated ring can come back at the same address)
  if (c->batched && !(c->batched_key < k) && !(k < c->batched_key) && c->batched_ring == ring &&
      c->batched_ring_cap == (ring ? c->ring_cap : 0)) {
    *out = c->batched;
    return 0;
  }
  drop_batched(c);
  const TrajGeom g = traj_geometry(c->T, n_steps, c->sm_count, c->variant);
  if (!g.ok || !variant_is_persistent(g.variant) || getenv("RSV_NO_PDL")) return 0;  // per-proposal graphs
  if (g.n_tiles > c->max_tiles) return fail(c, RSV_E_CUDA, "tile count %d exceeds buffer", g.n_tiles);
  auto *cg = new rsv_ctx::Cached();
  cg->dt = dt;
  cg->args = traj_args(c, dt, n_steps, fuse, g);
  cg->args.pdl = 1;
  cg->args.ring = const_cast<DevResult *>(ring);
  cg->args.ring_count = ring ? c->ring_count : nullptr;
  cg->args.ring_cap = ring ? c->ring_cap : 0;
  cg->traj_node = nullptr;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int l = 0;
  bool ok = true;
  for (int j = 0; j < UPDATE_BATCH; j++) {
    MomentaBufs mb = mbufs(c);
    mb.pdl = j > 0 ? 1 : 0;
    ok &= launch_momenta(mb, k.kind, c->Tg, c->stream, &l) == 0;
    ok &= launch_trajectory(cg->args, c->stream, &l) == 0;
  }
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (!ok || e != cudaSuccess) {
    delete cg;
    return fail(c, RSV_E_CUDA, "batched graph capture failed: %s", cudaGetErrorString(e));
  }
  cg->graph = graph;
  cg->launches = l;
  CK(cudaGraphInstantiate(&cg->exec, graph, 0));
  c->batched = cg;
  c->batched_key = k;
  c->batched_ring = ring;
  c->batched_ring_cap = ring ? c->ring_cap : 0;
  *out = cg;
  return 0;
}

int rsv_hmc_update_many(rsv_ctx *c, double dt, int n_steps, int fuse, int n, rsv_result *out) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  if (n < 1) return fail(c, RSV_E_INVALID, "n must be >= 1");
  CK(cudaSetDevice(c->device));
  if (out && n > c->ring_cap) {
    if (c->ring) cudaFree(c->ring);
    if (c->h_ring) cudaFreeHost(c->h_ring);
    c->ring_cap = n;
    CK(cudaMalloc(&c->ring, sizeof(DevResult) * n));
    CK(cudaMallocHost(&c->h_ring, sizeof(DevResult) * n));
  }
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  CK(cudaMemsetAsync(c->ring_count, 0, sizeof(int32_t), c->stream));
  rsv_ctx::Cached *cg = nullptr;
  int kpl = 0;
  // HMC-only proposals (the reference's hmc_update_volatility): no theta statistics
  if ((r = get_graph(c, dt, n_steps, fuse, 0, &cg, &kpl))) return r;
  cudaGraphExec_t exec = cg->exec;
  // timing 1: one event pair per proposal on the stream around the graph
  // launch (the L2 flush stays outside); timing 2: the graph's own four
  // event-record nodes give the momenta / trajectory breakdown as well
  std::vector<cudaGraphNode_t> *evn = nullptr;
  if (c->timing) {
    if (c->timing == 2) evn = &cg->ev;
    if ((r = ensure_events(c, 4 * (size_t)n + 4))) return r;
  }
  rsv_ctx::Cached *bg = nullptr;  // batches of UPDATE_BATCH proposals (no per-proposal timing / flush)
  if (!c->timing && c->flush_bytes == 0 && !c->shard && !c->ens_C && n >= UPDATE_BATCH && !getenv("RSV_NO_BATCH"))
    if ((r = get_batched(c, dt, n_steps, fuse, out != nullptr, &bg))) return r;
  for (int i = 0; i < n; i++) {
    if (bg && n - i >= UPDATE_BATCH) {
      CK(cudaGraphLaunch(bg->exec, c->stream));
      c->launches += bg->launches;
      i += UPDATE_BATCH - 1;
      continue;
    }
    if (evn) {
      for (int j = 0; j < 4; j++) CK(cudaGraphExecEventRecordNodeSetEvent(exec, (*evn)[j], c->evpool[4 + 4 * i + j]));
    }
    if (c->flush_bytes > 0) CK(cudaMemsetAsync(c->flush_buf, i & 0xff, (size_t)c->flush_bytes, c->stream));
    if (c->timing == 1) CK(cudaEventRecord(c->evpool[4 + 4 * i], c->stream));
    CK(cudaGraphLaunch(exec, c->stream));
    if (c->timing == 1) CK(cudaEventRecord(c->evpool[4 + 4 * i + 3], c->stream));
    c->launches += kpl;
    if (out) {
      ring_store_kernel<<<1, 1, 0, c->stream>>>(c->ctrl, c->ring, c->ring_cap, c->ring_count);
      c->launches++;
    }
  }
  if (out) CK(cudaMemcpyAsync(c->h_ring, c->ring, sizeof(DevResult) * n, cudaMemcpyDeviceToHost, c->stream));
  if ((r = pull_ctrl(c))) return r;
  if ((r = check_err_bits(c))) return r;
  if (out)
    for (int i = 0; i < n; i++) to_result(c->h_ring[i], out + i);
  if (c->timing) {
    c->last_traj_ms.assign(n, 0.0);
    c->last_mom_ms.assign(n, 0.0);
    c->last_total_ms.assign(n, 0.0);
    for (int i = 0; i < n; i++) {
      float t0 = 0, t1 = 0, t2 = 0;
      cudaEvent_t *e = &c->evpool[4 + 4 * i];
      if (evn) {
        CK(cudaEventElapsedTime(&t0, e[0], e[1]));
        CK(cudaEventElapsedTime(&t1, e[1], e[2]));
      }
      CK(cudaEventElapsedTime(&t2, e[0], e[3]));
      c->last_mom_ms[i] = t0;
      c->last_traj_ms[i] = t1;
      c->last_total_ms[i] = t2;
    }
  }
  return 0;
}

int rsv_hmc_update(rsv_ctx *c, double dt, int n_steps, int fuse, rsv_result *out) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  CK(cudaSetDevice(c->device));
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  rsv_ctx::Cached *cg = nullptr;
  int kpl = 0;
  if ((r = get_graph(c, dt, n_steps, fuse, 1, &cg, &kpl))) return r;
  CK(cudaGraphLaunch(cg->exec, c->stream));
  c->launches += kpl;
  if ((r = pull_ctrl(c))) return r;
  if ((r = check_err_bits(c))) return r;
  if (out) to_result(c->h_ctrl->res, out);
  return 0;
}

// sampler.py:144-167 in one call from host memory: the path and the stream
// state go in with asynchronous copies, the proposal runs as one graph, and
// one synchronisation returns the result (a second one copies the proposal
// out when it was accepted).  The theta statistics are not evaluated.
// h_in == NULL: propose from the path the context holds (a chain driven
// through this call keeps its path resident: only the stream state goes in).
int rsv_hmc_update_host(rsv_ctx *c, const double *h_in, double *h_out, rsv_prng_state *st, double dt, int n_steps,
                        int fuse, rsv_result *out) {
  if (!c || !h_out || !st || !out) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_md(c, dt, n_steps))) return r;
  if (!h_in && !c->has_latent) return fail(c, RSV_E_STATE, "no resident latent path (h_in is NULL)");
  if (!c->has_data) return fail(c, RSV_E_STATE, "data not set (rsv_set_data)");
  if (!c->has_params) return fail(c, RSV_E_STATE, "params not set (rsv_set_params)");
  if (c->shard || c->ens_C) return fail(c, RSV_E_STATE, "rsv_hmc_update_host needs a single-chain context");
  if (st->kind < 0 || st->kind > 3) return fail(c, RSV_E_INVALID, "invalid bit generator state");
  if (st->kind == PRNG_MINSTD && (st->s[0] == 0 || st->s[0] >= MINSTD_M))
    return fail(c, RSV_E_INVALID, "minstd state must be in [1, 2^31-2]");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));  // h_ctrl is the staging area below
  StreamState ss;
  ss.kind = st->kind;
  ss.reserved = 0;
  for (int i = 0; i < 4; i++) ss.s[i] = st->s[i];
  ss.pos = st->pos;
  c->h_ctrl->stream = ss;
  c->h_ctrl->seq_state = ss.kind == PRNG_PCG32    ? pcg_advance(ss.s[0], 2 * ss.pos, ss.s[1])
                         : ss.kind == PRNG_MINSTD ? mod31(minstd_pow(3 * ss.pos) * ss.s[0])
                                                  : 0;
  if (ss.kind != c->kind) c->kind = ss.kind;
  // stream state, cur = 0 and err = 0 are contiguous: one copy (plus seq_state)
  c->h_ctrl->cur = 0;
  c->h_ctrl->err = 0;
  static_assert(offsetof(DevControl, err) + sizeof(int32_t) - offsetof(DevControl, stream) ==
                    sizeof(StreamState) + 2 * sizeof(int32_t),
                "stream, cur, err are contiguous");
  if (h_in) {
    CK(cudaMemcpyAsync(&c->ctrl->stream, &c->h_ctrl->stream, sizeof(StreamState) + 2 * sizeof(int32_t),
                       cudaMemcpyHostToDevice, c->stream));
  } else {  // the resident path stays where it is: cur untouched
    CK(cudaMemcpyAsync(&c->ctrl->stream, &c->h_ctrl->stream, sizeof(StreamState), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  }
  CK(cudaMemcpyAsync(&c->ctrl->seq_state, &c->h_ctrl->seq_state, sizeof(uint64_t), cudaMemcpyHostToDevice,
                     c->stream));
  c->has_latent = true;
  const TrajGeom g = traj_geometry(c->T, n_steps, c->sm_count, c->variant);
  // zero copy: the trajectory kernel's tile staging (bulk copies) reads the
  // caller's page-locked path over PCIe itself, overlapped with the tiles,
  // instead of one copy in ahead of the proposal; arrays padded to T % 8 == 0
  // only (the staging reads whole 8-site groups)
  const void *h_map = nullptr;
  if (h_in && g.ok && c->T >= ZC_MIN_T && c->T % 8 == 0 && ((uintptr_t)h_in & 15) == 0 && c->timing == 0 &&
      !getenv("RSV_NO_ZERO_COPY")) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, h_in) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      h_map = pa.devicePointer;
    cudaGetLastError();
  }
  // a pageable path (T large enough for the in-place route): copied into a
  // page-locked staging buffer by host threads, then read like a page-locked
  // one -- the driver's own pageable copy is a single staged stream
  if (!h_map && h_in && g.ok && c->T >= ZC_MIN_T && c->T % 8 == 0 && c->timing == 0 && !getenv("RSV_NO_ZERO_COPY") &&
      !getenv("RSV_NO_HOST_STAGE")) {
    cudaPointerAttributes pa;
    const bool pageable = cudaPointerGetAttributes(&pa, h_in) == cudaSuccess && pa.type == cudaMemoryTypeUnregistered;
    cudaGetLastError();
    if (pageable) {
      if (!c->h_stage) {
        CK(cudaHostAlloc((void **)&c->h_stage, sizeof(double) * (size_t)c->T, cudaHostAllocMapped));
      }
      const int64_t T = c->T, nchunk = 64;
#pragma omp parallel for num_threads(HOST_STAGE_THREADS) schedule(static)
      for (int64_t k = 0; k < nchunk; k++) {
        const int64_t lo = T * k / nchunk / 8 * 8, hi = k + 1 == nchunk ? T : T * (k + 1) / nchunk / 8 * 8;
        memcpy(c->h_stage + lo, h_in + lo, sizeof(double) * (size_t)(hi - lo));
      }
      h_in = c->h_stage;
      void *dp = nullptr;
      CK(cudaHostGetDevicePointer(&dp, (void *)c->h_stage, 0));
      h_map = dp;
    }
  }
  c->zc_last = h_map ? 1 : 0;
  if (h_map) {
    rsv_ctx::Cached *cg = nullptr;
    int kpl = 0;
    if ((r = get_graph(c, dt, n_steps, fuse, 0, &cg, &kpl, 2, h_in))) return r;
    if (cg->head_node && cg->head_src != (const void *)h_in) {
      CK(cudaGraphExecMemcpyNodeSetParams1D(cg->exec, cg->head_node, c->hbuf[0], h_in, cg->head_bytes,
                                            cudaMemcpyHostToDevice));
      cg->head_src = h_in;
    }
    if (cg->args.h_src != (const double *)h_map) {  // re-point the kernel node (the cached args follow)
      cg->args.h_src = (const double *)h_map;
      void *kp[] = {&cg->args};
      cudaKernelNodeParams np = cg->traj_params;
      np.kernelParams = kp;
      CK(cudaGraphExecKernelNodeSetParams(cg->exec, cg->traj_node, &np));
    }
    CK(cudaGraphLaunch(cg->exec, c->stream));
    c->launches += kpl;
    if ((r = pull_ctrl(c))) return r;
    c->has_latent = c->h_ctrl->res.accept != 0;  // on a reject the device holds no copy of h_in
  } else {
    if (h_in) CK(cudaMemcpyAsync(c->hbuf[0], h_in, sizeof(double) * c->T, cudaMemcpyHostToDevice, c->stream));
    rsv_ctx::Cached *cg = nullptr;
    int kpl = 0;
    if ((r = get_graph(c, dt, n_steps, fuse, 0, &cg, &kpl))) return r;
    CK(cudaGraphLaunch(cg->exec, c->stream));
    c->launches += kpl;
    if ((r = pull_ctrl(c))) return r;
  }
  if ((r = check_err_bits(c))) return r;
  to_result(c->h_ctrl->res, out);
  st->pos = c->h_ctrl->stream.pos;
  for (int i = 0; i < 4; i++) st->s[i] = c->h_ctrl->stream.s[i];
  if (out->accept) {
    CK(cudaMemcpyAsync(h_out, c->hbuf[c->h_ctrl->cur & 1], sizeof(double) * c->T, cudaMemcpyDeviceToHost,
                       c->stream));
    return sync(c);
  }
  return 0;  // rejected or divergent: the kept path is h_in, h_out is not written
}

int rsv_last_update_zero_copy(const rsv_ctx *c) { return c ? c->zc_last : 0; }

int rsv_last_stats(rsv_ctx *c, double out[7]) {
  if (!c || !out) return fail(c, RSV_E_INVALID, "null argument");
  for (int i = 0; i < 7; i++) out[i] = c->h_ctrl->stats[i];
  return 0;
}

// integrate_trajectory from explicit (h, p)
int rsv_integrate(rsv_ctx *c, const double *h_in, const double *p_in, double dt, int n_steps, int fuse,
                  double *h_out, double *p_out, int32_t *diverged, int on_device) {
  if (!c || !h_in || !p_in) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_md(c, dt, n_steps))) return r;
  if (!c->has_data) return fail(c, RSV_E_STATE, "data not set (rsv_set_data)");
  if (!c->has_params) return fail(c, RSV_E_STATE, "params not set (rsv_set_params)");
  CK(cudaSetDevice(c->device));
  if ((r = copy_in(c, c->sh, h_in, c->T, on_device)) || (r = copy_in(c, c->sp, p_in, c->T, on_device))) return r;
  const TrajGeom g = traj_geometry(c->T, n_steps, c->sm_count, c->variant);
  int l = 0;
  int32_t div = 0;
  if (g.ok) {
    TrajArgs a = traj_args(c, dt, n_steps, fuse, g);
    a.h_src = c->sh;
    a.h_dst = c->sh2;
    a.p_in = c->sp;
    a.p_out = c->sp2;
    a.integrate_only = 1;
    a.stats = 1;
    LK(launch_trajectory(a, c->stream, &l));
    c->launches += l;
    if ((r = pull_ctrl(c))) return r;
    div = c->h_ctrl->res.diverged;
    if ((r = copy_out(c, h_out, c->sh2, c->T, on_device)) || (r = copy_out(c, p_out, c->sp2, c->T, on_device)))
      return r;
  } else {
    // very long trajectories: one streamed elementary step per launch (unfused grouping)
    CK(cudaMemsetAsync(c->dflag, 0, sizeof(int32_t), c->stream));
    double *h0 = c->sh, *p0 = c->sp, *h1 = c->sh2, *p1 = c->sp2;
    for (int k = 0; k < n_steps; k++) {
      LK(launch_elementary_step(h0, p0, h1, p1, c->a, c->lrv, c->prm, dt, c->T, c->dflag, c->stream, &l));
      std::swap(h0, h1);
      std::swap(p0, p1);
    }
    c->launches += l;
    CK(cudaMemcpyAsync(c->h_flag, c->dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    if ((r = copy_out(c, h_out, h0, c->T, on_device)) || (r = copy_out(c, p_out, p0, c->T, on_device))) return r;
    if ((r = sync(c))) return r;
    div = *c->h_flag;
  }
  if ((r = sync(c))) return r;
  if (diverged) *diverged = div;
  return 0;
}

int rsv_elementary_step(rsv_ctx *c, double *h, double *p, double dt, int32_t *diverged, int on_device) {
  if (!c || !h || !p) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_md(c, dt, 1))) return r;
  if (!c->has_data || !c->has_params) return fail(c, RSV_E_STATE, "data/params not set");
  CK(cudaSetDevice(c->device));
  if ((r = copy_in(c, c->sh, h, c->T, on_device)) || (r = copy_in(c, c->sp, p, c->T, on_device))) return r;
  CK(cudaMemsetAsync(c->dflag, 0, sizeof(int32_t), c->stream));
  int l = 0;
  LK(launch_elementary_step(c->sh, c->sp, c->sh2, c->sp2, c->a, c->lrv, c->prm, dt, c->T, c->dflag, c->stream, &l));
  c->launches += l;
  CK(cudaMemcpyAsync(c->h_flag, c->dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  if ((r = copy_out(c, h, c->sh2, c->T, on_device)) || (r = copy_out(c, p, c->sp2, c->T, on_device))) return r;
  if ((r = sync(c))) return r;
  if (diverged) *diverged = *c->h_flag;
  return 0;
}

// Repeated elementary steps on device-resident (h, p) for the paper protocol
// (bench.py:121-190 time_elementary_step).  The state lives in (sh2, sp2):
// set by rsv_bench_state or left by rsv_elementary_step; the steps ping-pong
// with (sh, sp) and the result is moved back to (sh2, sp2) outside the timed
// events.
int rsv_bench_state(rsv_ctx *c, const double *h, const double *p) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  CK(cudaSetDevice(c->device));
  int r;
  if (h && (r = copy_in(c, c->sh2, h, c->T, 0))) return r;
  if (p && (r = copy_in(c, c->sp2, p, c->T, 0))) return r;
  return sync(c);
}

int rsv_bench_elementary(rsv_ctx *c, double dt, int n_steps, float *ms, int32_t *diverged) {
  if (!c || !ms) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_md(c, dt, n_steps))) return r;
  if (!c->has_data || !c->has_params) return fail(c, RSV_E_STATE, "data/params not set");
  CK(cudaSetDevice(c->device));
  // the n steps are one CUDA graph (cached per (n, dt)): kernel nodes run
  // back to back without per-launch host submission
  GraphKey k{-2, n_steps, 0, 0, 0, dt};
  auto it = c->graphs.find(k);
  if (it == c->graphs.end()) {
    auto *cg = new rsv_ctx::Cached();
    memset(&cg->args, 0, sizeof(cg->args));
    cg->dt = dt;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    double *h0 = c->sh2, *p0 = c->sp2, *h1 = c->sh, *p1 = c->sp;
    int l = 0;
    bool ok = true;
    const int pdl_steps = getenv("RSV_NO_PDL") ? 0 : 1;  // step k+1 launched while step k runs
    for (int i = 0; i < n_steps; i++) {
      ok &= launch_elementary_step(h0, p0, h1, p1, c->a, c->lrv, c->prm, dt, c->T, c->dflag, c->stream, &l,
                                   pdl_steps) == 0;
      std::swap(h0, h1);
      std::swap(p0, p1);
    }
    if (h0 != c->sh2) {  // result back into the state buffers
      cudaMemcpyAsync(c->sh2, h0, sizeof(double) * c->T, cudaMemcpyDeviceToDevice, c->stream);
      cudaMemcpyAsync(c->sp2, p0, sizeof(double) * c->T, cudaMemcpyDeviceToDevice, c->stream);
    }
    cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
    if (!ok || e != cudaSuccess) {
      delete cg;
      return fail(c, RSV_E_CUDA, "protocol graph capture failed: %s", cudaGetErrorString(e));
    }
    cg->graph = graph;
    cg->traj_node = nullptr;
    CK(cudaGraphInstantiate(&cg->exec, graph, 0));
    it = c->graphs.emplace(k, cg).first;
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaMemsetAsync(c->dflag, 0, sizeof(int32_t), c->stream));
  CK(cudaEventRecord(e0, c->stream));
  CK(cudaGraphLaunch(it->second->exec, c->stream));
  CK(cudaEventRecord(e1, c->stream));
  c->launches += n_steps;
  CK(cudaMemcpyAsync(c->h_flag, c->dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(ms, e0, e1));
  CK(cudaStreamSynchronize(c->stream));
  if (diverged) *diverged = *c->h_flag;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 0;
}

// The same protocol with the n steps fused into one launch of the persistent
// trajectory kernel (the halo tiles make a segment of n steps exact without
// per-step synchronisation; energies are evaluated but not used).
int rsv_bench_fused(rsv_ctx *c, double dt, int n_steps, float *ms, int32_t *diverged) {
  if (!c || !ms) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_md(c, dt, n_steps))) return r;
  if (!c->has_data || !c->has_params) return fail(c, RSV_E_STATE, "data/params not set");
  if (c->shard || c->ens_C) return fail(c, RSV_E_STATE, "rsv_bench_fused needs a single-chain context");
  CK(cudaSetDevice(c->device));
  const TrajGeom g = traj_geometry(c->T, n_steps, c->sm_count, c->variant);
  if (!g.ok) return fail(c, RSV_E_INVALID, "n_steps=%d too large for one fused segment", n_steps);
  if (g.n_tiles > c->max_tiles) return fail(c, RSV_E_CUDA, "tile count %d exceeds buffer", g.n_tiles);
  TrajArgs a = traj_args(c, dt, n_steps, 0, g);
  a.h_src = c->sh2;
  a.h_dst = c->sh;
  a.p_in = c->sp2;
  a.p_out = c->sp;
  a.integrate_only = 1;
  a.stats = 0;
  if ((r = ensure_events(c, 2))) return r;
  int l = 0;
  CK(cudaEventRecord(c->evpool[0], c->stream));
  LK(launch_trajectory(a, c->stream, &l));
  CK(cudaEventRecord(c->evpool[1], c->stream));
  c->launches += l;
  CK(cudaMemcpyAsync(c->sh2, c->sh, sizeof(double) * c->T, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(c->sp2, c->sp, sizeof(double) * c->T, cudaMemcpyDeviceToDevice, c->stream));
  if ((r = pull_ctrl(c))) return r;
  CK(cudaEventElapsedTime(ms, c->evpool[0], c->evpool[1]));
  if (diverged) *diverged = c->h_ctrl->res.diverged;
  return 0;
}

// The trajectory kernel alone, n launches back to back on the context's
// stream bracketed by one CUDA event pair (the roofline's launch duration,
// bench.py): the proposal's own kernel configuration on the current path and
// the last momenta, integrate-only (no Metropolis bookkeeping, no state
// change; the proposal goes to scratch).  L2 as inside a proposal (warm).
int rsv_bench_trajectory(rsv_ctx *c, double dt, int n_steps, int n, float *ms_per_launch) {
  if (!c || !ms_per_launch || n < 1) return fail(c, RSV_E_INVALID, "bad argument");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  if (c->shard || c->ens_C) return fail(c, RSV_E_STATE, "rsv_bench_trajectory needs a single-chain context");
  CK(cudaSetDevice(c->device));
  const TrajGeom g = traj_geometry(c->T, n_steps, c->sm_count, c->variant);
  if (!g.ok) return fail(c, RSV_E_INVALID, "n_steps=%d too large for one fused trajectory", n_steps);
  TrajArgs a = traj_args(c, dt, n_steps, 0, g);
  CK(cudaMemcpy(c->h_ctrl, c->ctrl, sizeof(DevControl), cudaMemcpyDeviceToHost));
  a.h_src = c->hbuf[c->h_ctrl->cur];
  a.h_dst = c->sh;
  a.integrate_only = 1;
  a.stats = 0;
  if ((r = ensure_events(c, 2))) return r;
  int l = 0;
  LK(launch_trajectory(a, c->stream, &l));  // warm
  CK(cudaEventRecord(c->evpool[0], c->stream));
  for (int i = 0; i < n; i++) LK(launch_trajectory(a, c->stream, &l));
  CK(cudaEventRecord(c->evpool[1], c->stream));
  c->launches += l;
  CK(cudaEventSynchronize(c->evpool[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->evpool[0], c->evpool[1]));
  *ms_per_launch = ms / n;
  return sync(c);
}

static int ensure_plugin(rsv_ctx *c, int64_t n) {
  if (n <= c->pl_n) return 0;
  for (int i = 0; i < 4; i++) {
    if (c->pl[i]) cudaFree(c->pl[i]);
    CK(cudaMalloc(&c->pl[i], sizeof(double) * n));
  }
  c->pl_n = n;
  return 0;
}

static int check_range(rsv_ctx *c, int64_t n, int64_t lo, int64_t hi) {
  if (n < 0 || lo < 0 || hi > n || lo > hi) return fail(c, RSV_E_INVALID, "bad range [%lld, %lld) of %lld",
                                                       (long long)lo, (long long)hi, (long long)n);
  return 0;
}

int rsv_position_update(rsv_ctx *c, double *h, const double *p, double cc, int64_t n, int64_t lo, int64_t hi,
                        int on_device) {
  if (!c || !h || !p) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_range(c, n, lo, hi))) return r;
  CK(cudaSetDevice(c->device));
  int l = 0;
  if (on_device) {
    LK(launch_position_update(h, p, cc, lo, hi, c->stream, &l));
  } else {
    if ((r = ensure_plugin(c, n))) return r;
    CK(cudaMemcpyAsync(c->pl[0] + lo, h + lo, sizeof(double) * (hi - lo), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->pl[1] + lo, p + lo, sizeof(double) * (hi - lo), cudaMemcpyHostToDevice, c->stream));
    LK(launch_position_update(c->pl[0], c->pl[1], cc, lo, hi, c->stream, &l));
    CK(cudaMemcpyAsync(h + lo, c->pl[0] + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToHost, c->stream));
  }
  c->launches += l;
  return sync(c);
}

static int plugin_grad(rsv_ctx *c, const double *h, double *p, const double *y, const double *lrv, double dt,
                       const double *scal, int64_t n, int64_t lo, int64_t hi, int32_t *flag, int on_device,
                       int fill) {
  int r;
  if ((r = check_range(c, n, lo, hi))) return r;
  if (!scal) return fail(c, RSV_E_INVALID, "null scalars");
  CK(cudaSetDevice(c->device));
  CK(cudaMemsetAsync(c->dflag, 0, sizeof(int32_t), c->stream));
  int l = 0;
  PackedScal P;
  for (int i = 0; i < 7; i++) P.v[i] = scal[i];
  if (on_device) {
    if (fill) LK(launch_gradient(h, y, lrv, P, p, n, lo, hi, c->dflag, c->stream, &l));
    else LK(launch_momentum_update(h, p, y, lrv, dt, P, n, lo, hi, c->dflag, c->stream, &l));
  } else {
    if ((r = ensure_plugin(c, n))) return r;
    const int64_t a = lo > 0 ? lo - 1 : 0, b = hi < n ? hi + 1 : n;
    CK(cudaMemcpyAsync(c->pl[0] + a, h + a, sizeof(double) * (b - a), cudaMemcpyHostToDevice, c->stream));
    if (!fill)
      CK(cudaMemcpyAsync(c->pl[1] + lo, p + lo, sizeof(double) * (hi - lo), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->pl[2] + lo, y + lo, sizeof(double) * (hi - lo), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->pl[3] + lo, lrv + lo, sizeof(double) * (hi - lo), cudaMemcpyHostToDevice, c->stream));
    if (fill) LK(launch_gradient(c->pl[0], c->pl[2], c->pl[3], P, c->pl[1], n, lo, hi, c->dflag, c->stream, &l));
    else LK(launch_momentum_update(c->pl[0], c->pl[1], c->pl[2], c->pl[3], dt, P, n, lo, hi, c->dflag, c->stream, &l));
    CK(cudaMemcpyAsync(p + lo, c->pl[1] + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToHost, c->stream));
  }
  c->launches += l;
  CK(cudaMemcpyAsync(c->h_flag, c->dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  if ((r = sync(c))) return r;
  if (flag) *flag = *c->h_flag;
  return 0;
}

int rsv_momentum_update(rsv_ctx *c, const double *h, double *p, const double *y, const double *lrv, double dt,
                        const double *scal, int64_t n, int64_t lo, int64_t hi, int32_t *flag, int on_device) {
  if (!c || !h || !p || !y || !lrv) return fail(c, RSV_E_INVALID, "null argument");
  return plugin_grad(c, h, p, y, lrv, dt, scal, n, lo, hi, flag, on_device, 0);
}

int rsv_gradient(rsv_ctx *c, const double *h, const double *y, const double *lrv, const double *scal,
                 double *out, int64_t n, int64_t lo, int64_t hi, int32_t *flag, int on_device) {
  if (!c || !h || !out || !y || !lrv) return fail(c, RSV_E_INVALID, "null argument");
  return plugin_grad(c, h, out, y, lrv, 0.0, scal, n, lo, hi, flag, on_device, 1);
}

static int energy(rsv_ctx *c, const double *h, const double *p, int on_device, double *kin, double *logf) {
  if (!c->has_data || !c->has_params) return fail(c, RSV_E_STATE, "data/params not set");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = copy_in(c, c->sh, h, c->T, on_device))) return r;
  if (p) {
    if ((r = copy_in(c, c->sp, p, c->T, on_device))) return r;
  } else {
    CK(cudaMemsetAsync(c->sp, 0, sizeof(double) * c->T, c->stream));
  }
  int l = 0;
  LK(launch_energy(c->sh, c->sp, c->y, c->lrv, c->prm, c->T, c->rpart, c->rout, c->stream, &l));
  c->launches += l;
  CK(cudaMemcpyAsync(c->h_out, c->rout, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
  if ((r = sync(c))) return r;
  *kin = c->h_out[0];
  *logf = c->h_out[1];
  return 0;
}

int rsv_hamiltonian(rsv_ctx *c, const double *h, const double *p, double *out, int on_device) {
  if (!c || !h || !p || !out) return fail(c, RSV_E_INVALID, "null argument");
  double k, lf;
  int r = energy(c, h, p, on_device, &k, &lf);
  if (r) return r;
  *out = k - lf;
  return 0;
}

int rsv_log_posterior(rsv_ctx *c, const double *h, double *out, int on_device) {
  if (!c || !h || !out) return fail(c, RSV_E_INVALID, "null argument");
  double k, lf;
  int r = energy(c, h, nullptr, on_device, &k, &lf);
  if (r) return r;
  *out = lf;
  return 0;
}

int rsv_suff_stats(rsv_ctx *c, double c_mu, double c_xi, double out[7]) {
  if (!c || !out) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->has_data || !c->has_latent) return fail(c, RSV_E_STATE, "data/latent not set");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = pull_ctrl(c))) return r;
  int l = 0;
  LK(launch_suff_stats(c->hbuf[c->h_ctrl->cur & 1], c->lrv, c->T, c_mu, c_xi, c->rpart, c->rout, c->stream, &l));
  c->launches += l;
  CK(cudaMemcpyAsync(c->h_out, c->rout, sizeof(double) * 7, cudaMemcpyDeviceToHost, c->stream));
  if ((r = sync(c))) return r;
  for (int i = 0; i < 7; i++) out[i] = c->h_out[i];
  return 0;
}

int rsv_set_l2_flush(rsv_ctx *c, int64_t bytes) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  CK(cudaSetDevice(c->device));
  if (c->flush_buf) {
    CK(cudaFree(c->flush_buf));
    c->flush_buf = nullptr;
  }
  c->flush_bytes = bytes > 0 ? bytes : 0;
  if (c->flush_bytes) CK(cudaMalloc(&c->flush_buf, (size_t)c->flush_bytes));
  return 0;
}

int rsv_measure_fp64_peak(rsv_ctx *c, double *tflops) {
  if (!c || !tflops) return fail(c, RSV_E_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  const int blocks = c->sm_count * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  double best = 0;
  for (int rep = 0; rep < 5; rep++) {
    CK(cudaEventRecord(e0, c->stream));
    dfma_peak_kernel<<<blocks, threads, 0, c->stream>>>(c->rout, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double fl = 2.0 * 8.0 * iters * (double)blocks * threads;
    if (rep > 0 && fl / (ms * 1e-3) / 1e12 > best) best = fl / (ms * 1e-3) / 1e12;
  }
  c->launches += 5;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *tflops = best;
  return 0;
}

// development aid: copy the per-tile timestamps of the last trajectory
int rsv_debug_stamps(rsv_ctx *c, unsigned long long *out, int max_tiles) {
  if (!c || !c->dbg) return fail(c, RSV_E_STATE, "stamps not enabled (RSV_TRAJ_STAMPS=1)");
  CK(cudaStreamSynchronize(c->stream));
  const int n = max_tiles < c->max_tiles ? max_tiles : c->max_tiles;
  CK(cudaMemcpy(out, c->dbg, sizeof(unsigned long long) * 8 * n, cudaMemcpyDeviceToHost));
  return 0;
}

// ---- time sharding (one chain split over several contexts / GPUs) ----------
// Advance the context's stream past a proposal (momenta + the uniform if
// drawn), as the single-chain Metropolis step does.
__device__ void shard_advance(DevControl *C, int drew, const uint64_t *snaps) {
  const uint64_t consumed = C->zig_used + (drew ? 1 : 0);
  if (C->stream.kind == PRNG_SFC64) {
    const uint64_t *q = snaps + 4 * (consumed / SFC_SNAP);
    uint64_t st[4] = {q[0], q[1], q[2], q[3]};
    for (uint64_t i = 0; i < consumed % SFC_SNAP; i++) sfc64_next(st);
    for (int i = 0; i < 4; i++) C->stream.s[i] = st[i];
  } else if (C->stream.kind == PRNG_PCG32) {
    uint64_t q = C->seq_next;
    if (drew) { q = q * PCG_MULT + C->stream.s[1]; q = q * PCG_MULT + C->stream.s[1]; }
    C->seq_state = q;
  } else if (C->stream.kind == PRNG_MINSTD) {
    uint64_t q = C->seq_next;
    if (drew) q = mod31(mod31(mod31(q * MINSTD_A) * MINSTD_A) * MINSTD_A);
    C->seq_state = q;
  }
  C->stream.pos += consumed;
}

__global__ void shard_apply_kernel(DevControl *C, int accept, int drew, const uint64_t *snaps) {
  if (threadIdx.x || blockIdx.x) return;
  shard_advance(C, drew, snaps);
  if (accept) C->cur ^= 1;
}

// ---- device-side orchestration of a sharded chain (no host sync per proposal)
// pack: this shard's record (ShardRec = rsv_shard_totals layout)
__global__ void shard_pack_kernel(const DevControl *C, int own_first, int own_last, ShardRec *out) {
  if (threadIdx.x || blockIdx.x) return;
  ShardRec r;
  r.part = *reinterpret_cast<const TilePart *>(C->shard_parts);
  r.ends[0] = own_first ? C->ends_old[0] : 0.0;
  r.ends[1] = own_last ? C->ends_old[1] : 0.0;
  r.ends[2] = own_first ? C->ends_new[0] : 0.0;
  r.ends[3] = own_last ? C->ends_new[1] : 0.0;
  r.u_word = C->u_word;
  r.words_used = C->zig_used;
  *out = r;
}

__device__ __forceinline__ __int128 rec128(const long long (&w)[2]) {
  return (__int128)(((unsigned __int128)(unsigned long long)w[1] << 64) | (unsigned long long)w[0]);
}
__device__ __forceinline__ double rec_unfix(__int128 q) {  // as unfix128 in leapfrog.cu
  const bool neg = q < 0;
  const unsigned __int128 a = neg ? (unsigned __int128)(-q) : (unsigned __int128)q;
  const double r = __ull2double_rn((unsigned long long)(a >> 64)) + __ull2double_rn((unsigned long long)a) * 0x1p-64;
  return neg ? -r : r;
}

// Metropolis on the all-gathered records (world ShardRecs, rank order):
// dH, H_old and H_new are exact integer sums of the fixed-point parts (the
// same bits as a single context over the whole series, for any world size);
// the moments use fixed-order compensated sums.  Every rank runs this on the
// same data, so every rank takes the same decision (sampler.py:155-167);
// then the stream advances and the kept path's statistics and the result
// are recorded.
__global__ void shard_decide_kernel(DevControl *C, const ShardRec *g, int world, const DevParams *prm,
                                    const uint64_t *snaps, DevResult *ring, int cap, int32_t *count, int windowed) {
  if (threadIdx.x >= 32 || blockIdx.x) return;
  const int lane = threadIdx.x;
  // every control word of the step is loaded up front: a value written and
  // read back through device memory would cost an L2 round trip each time
  const int halt = C->halt;
  const StreamState st = C->stream;
  const uint64_t seq = C->seq_state;
  const int cur = C->cur;
  const double hconst = prm->hconst;
  const int i_ring = ring ? *count : 0;
  if (halt) return;  // sharded run_chain stopped at an earlier sweep
  // lane k < 14: moment / end sum k over the ranks in rank order (TwoSum):
  // old moments 0..4, new 5..9, ends 10..13
  double Sk = 0.0;
  if (lane < 14) {
    double sum = 0.0, comp = 0.0;
    for (int r = 0; r < world; r++) {
      const double x = lane < 5 ? g[r].part.so[lane] : lane < 10 ? g[r].part.sn[lane - 5] : g[r].ends[lane - 10];
      const double t = sum + x;
      const double bp = t - sum;
      comp += (sum - (t - bp)) + (x - bp);
      sum = t;
    }
    Sk = sum + comp;
  }
  // every lane: the exact fixed-point totals and the decision (same values)
  __int128 q0 = 0, q1 = 0, q2 = 0;
  double fl = 0.0;
  for (int r = 0; r < world; r++) {
    q0 += rec128(g[r].part.dh);
    q1 += rec128(g[r].part.hold);
    q2 += rec128(g[r].part.hnew);
    fl = fmax(fl, g[r].part.flag);
  }
  // the momenta's end in the stream: every shard drew the whole series
  // (replicated) -- then all records must agree -- or the last shard's
  // window holds the draw's end (windowed); either way the last record
  const uint64_t u_word = g[world - 1].u_word;
  const uint64_t used = g[world - 1].words_used;
  if (!windowed && lane == 0) {
    bool consistent = true;
    for (int r = 0; r < world - 1; r++) consistent &= g[r].u_word == u_word && g[r].words_used == used;
    if (!consistent) atomicOr(&C->err, 8);
  }
  DevResult res;
  res.h_old = rec_unfix(q1) + hconst;
  res.h_new = rec_unfix(q2) + hconst;
  res.accept = 0;
  res.u = __longlong_as_double(0x7ff8000000000000LL);
  const double dh = rec_unfix(q0);
  bool drew = false;
  if (fl > 0.0 || !isfinite(dh) || fabs(dh) > 1000.0) {
    res.diverged = 1;
    res.delta_h = __longlong_as_double(0x7ff0000000000000LL);
  } else {
    res.diverged = 0;
    res.delta_h = dh;
    res.u = u01(u_word);
    drew = true;
    res.accept = (dh <= 0.0) || (res.u < exp(-dh));
  }
  res.words_used = used + (drew ? 1 : 0);
  // statistics of the kept path (lane k holds sum k)
  if (res.accept) {
    if (lane == 12 || lane == 13) C->stats[lane - 12] = Sk;
    if (lane >= 5 && lane < 10) C->stats[2 + lane - 5] = Sk;
  } else {
    if (lane == 10 || lane == 11) C->stats[lane - 10] = Sk;
    if (lane < 5) C->stats[2 + lane] = Sk;
  }
  if (lane) return;
  // the stream after the momenta (and the uniform, if drawn): from the state
  // at the proposal's stream position, advanced by the words used
  C->zig_used = used;
  if (st.kind == PRNG_SFC64) {
    shard_advance(C, drew, snaps);
  } else {
    uint64_t q = seq;
    if (st.kind == PRNG_PCG32) {
      q = pcg_advance(seq, 2 * used, st.s[1]);
      C->seq_next = q;
      if (drew) { q = q * PCG_MULT + st.s[1]; q = q * PCG_MULT + st.s[1]; }
    } else if (st.kind == PRNG_MINSTD) {
      q = mod31(minstd_pow(3 * used) * seq);
      C->seq_next = q;
      if (drew) q = mod31(mod31(mod31(q * MINSTD_A) * MINSTD_A) * MINSTD_A);
    }
    C->seq_state = q;
    C->stream.pos = st.pos + used + (drew ? 1 : 0);
  }
  if (res.accept) C->cur = cur ^ 1;
  C->res = res;
  if (ring) {
    if (i_ring < cap) ring[i_ring] = res;
    *count = i_ring + 1;
  }
}

// halo: owned boundary sites of the current path out / margins in
__global__ void shard_halo_kernel(DevControl *C, double *h0, double *h1, int64_t own_lo, int64_t own_hi,
                                  int64_t T, double *left, int64_t nl, double *right, int64_t nr, int unpack) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double *h = C->cur ? h1 : h0;
  if (!unpack) {
    if (i < nl) left[i] = h[own_lo + i];
    if (i < nr) right[i] = h[own_hi - nr + i];
  } else {  // left = what the left neighbour sent (my sites [0, nl)), right = [own_hi, own_hi + nr)
    if (i < nl) h[i] = left[i];
    if (i < nr && own_hi + i < T) h[own_hi + i] = right[i];
  }
}

int rsv_create_shard(rsv_ctx **out, int device, int64_t Tg, int64_t lo, int64_t hi, int64_t margin,
                     int64_t *local_start, int64_t *local_len) {
  if (!out) return fail(nullptr, RSV_E_INVALID, "out is null");
  *out = nullptr;
  if (Tg < 2 || lo < 0 || hi > Tg || lo >= hi || margin < 0)
    return fail(nullptr, RSV_E_INVALID, "bad shard [%lld, %lld) of %lld", (long long)lo, (long long)hi, (long long)Tg);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, RSV_E_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, RSV_E_INVALID, "device %d out of range", device);
  // local range: the owned sites plus `margin` on each side, starting on a
  // multiple of 8 sites so tiles stay 64 B aligned in the global momenta
  int64_t ls = lo - margin;
  ls = ls < 0 ? 0 : ls / 8 * 8;
  int64_t le = hi + margin;
  le = le > Tg ? Tg : le;
  rsv_ctx *c = new rsv_ctx();
  c->shard = true;
  c->goff = ls;
  c->own_lo = lo - ls;
  c->own_hi = hi - ls;
  const int r = create_impl(c, device, le - ls, Tg);
  if (r) {
    g_err = c->err;
    rsv_destroy(c);
    return r;
  }
  if (c->variant >= 0 && c->variant < 9) c->variant = -1;  // the persistent kernel carries the shard indexing
  if (local_start) *local_start = ls;
  if (local_len) *local_len = le - ls;
  *out = c;
  return 0;
}

int rsv_shard_propose(rsv_ctx *c, double dt, int n_steps, int fuse, int stats, rsv_shard_totals *out) {
  if (!c || !out) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  CK(cudaSetDevice(c->device));
  rsv_ctx::Cached *cg = nullptr;
  int kpl = 0;
  if ((r = get_graph(c, dt, n_steps, fuse, stats, &cg, &kpl))) return r;
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  CK(cudaGraphLaunch(cg->exec, c->stream));
  c->launches += kpl;
  if ((r = pull_ctrl(c))) return r;
  if ((r = check_err_bits(c))) return r;
  const DevControl &C = *c->h_ctrl;
  static_assert(sizeof(rsv_shard_totals) == sizeof(ShardRec), "rsv_shard_totals mirrors ShardRec");
  ShardRec rec;
  rec.part = *reinterpret_cast<const TilePart *>(C.shard_parts);
  const bool own_first = c->goff + c->own_lo == 0, own_last = c->goff + c->own_hi == c->Tg;
  rec.ends[0] = own_first ? C.ends_old[0] : 0.0;
  rec.ends[1] = own_last ? C.ends_old[1] : 0.0;
  rec.ends[2] = own_first ? C.ends_new[0] : 0.0;
  rec.ends[3] = own_last ? C.ends_new[1] : 0.0;
  rec.u_word = C.u_word;
  rec.words_used = C.zig_used;
  memcpy(out, &rec, sizeof(rec));
  return 0;
}

int rsv_shard_apply(rsv_ctx *c, int accept, int drew) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  CK(cudaSetDevice(c->device));
  shard_apply_kernel<<<1, 1, 0, c->stream>>>(c->ctrl, accept, drew, c->sfc_snaps);
  c->launches++;
  CK(cudaGetLastError());
  return sync(c);
}

int rsv_set_stream(rsv_ctx *c, void *stream) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  if (!c->own_stream) c->own_stream = c->stream;
  c->stream = stream ? (cudaStream_t)stream : c->own_stream;
  return 0;
}

int rsv_shard_propose_async(rsv_ctx *c, double dt, int n_steps, int fuse, int stats, double *totals_dev) {
  if (!c || !totals_dev) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  CK(cudaSetDevice(c->device));
  rsv_ctx::Cached *cg = nullptr;
  int kpl = 0;
  if ((r = get_graph(c, dt, n_steps, fuse, stats, &cg, &kpl))) return r;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(c->stream, &cs));
  if (cs == cudaStreamCaptureStatusActive) {
    // inside the caller's stream capture (the sharded driver records whole
    // halo periods as one CUDA graph): the cached graph's kernels directly
    int l = 0;
    bool ok = true;
    if (!(c->win_mode && !c->blocks)) ok &= launch_momenta(mbufs(c), c->kind, c->Tg, c->stream, &l) == 0;
    if (cg->args.g.ok) ok &= launch_trajectory(cg->args, c->stream, &l) == 0;
    else return fail(c, RSV_E_STATE, "n_steps=%d too large for a sharded trajectory", n_steps);
    if (!ok) return fail(c, RSV_E_CUDA, "captured proposal launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  } else {
    CK(cudaGraphLaunch(cg->exec, c->stream));
  }
  const int own_first = c->goff + c->own_lo == 0, own_last = c->goff + c->own_hi == c->Tg;
  shard_pack_kernel<<<1, 1, 0, c->stream>>>(c->ctrl, own_first, own_last, reinterpret_cast<ShardRec *>(totals_dev));
  c->launches += kpl + 1;
  CK(cudaGetLastError());
  return 0;
}

// Build (and cache) the proposal graph of rsv_shard_propose_async ahead of
// time, e.g. before the caller records its own stream capture.
int rsv_shard_prepare(rsv_ctx *c, double dt, int n_steps, int fuse, int stats) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  CK(cudaSetDevice(c->device));
  rsv_ctx::Cached *cg = nullptr;
  int kpl = 0;
  if ((r = get_graph(c, dt, n_steps, fuse, stats, &cg, &kpl))) return r;
  if (!c->ring || c->ring_cap < 1024) {  // the decision ring (rsv_shard_decide_async), outside any capture
    if (c->ring) cudaFree(c->ring);
    if (c->h_ring) cudaFreeHost(c->h_ring);
    c->ring_cap = 1024;
    CK(cudaMalloc(&c->ring, sizeof(DevResult) * c->ring_cap));
    CK(cudaMallocHost(&c->h_ring, sizeof(DevResult) * c->ring_cap));
    CK(cudaMemsetAsync(c->ring_count, 0, sizeof(int32_t), c->stream));
  }
  return sync(c);
}

int rsv_shard_decide_async(rsv_ctx *c, const double *gathered_dev, int world) {
  if (!c || !gathered_dev || world < 1) return fail(c, RSV_E_INVALID, "bad argument");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  CK(cudaSetDevice(c->device));
  if (!c->ring || c->ring_cap < 1024) {
    if (c->ring) cudaFree(c->ring);
    if (c->h_ring) cudaFreeHost(c->h_ring);
    c->ring_cap = 1024;
    CK(cudaMalloc(&c->ring, sizeof(DevResult) * c->ring_cap));
    CK(cudaMallocHost(&c->h_ring, sizeof(DevResult) * c->ring_cap));
    CK(cudaMemsetAsync(c->ring_count, 0, sizeof(int32_t), c->stream));
  }
  shard_decide_kernel<<<1, 32, 0, c->stream>>>(c->ctrl, reinterpret_cast<const ShardRec *>(gathered_dev), world,
                                              c->prm, c->sfc_snaps, c->ring, c->ring_cap, c->ring_count,
                                              c->win_mode && !c->blocks ? 1 : 0);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

int rsv_shard_halo_async(rsv_ctx *c, double *left, int64_t nl, double *right, int64_t nr, int unpack) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  if (nl < 0 || nr < 0 || (nl && !left) || (nr && !right)) return fail(c, RSV_E_INVALID, "bad halo buffers");
  CK(cudaSetDevice(c->device));
  const int64_t n = nl > nr ? nl : nr;
  if (n == 0) return 0;
  shard_halo_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(c->ctrl, c->hbuf[0], c->hbuf[1], c->own_lo,
                                                                      c->own_hi, c->T, left, nl, right, nr, unpack);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// ---- windowed momenta of a time-sharded chain ----------------------------
// Placement: the all-gathered windows give every shard the global index of
// its window's normals (exclusive prefix of the counts between anchors);
// the neighbours' views of each anchor must agree, and the window must
// cover the shard's sites.  The shard's normals are copied to where the
// trajectory reads them; the last shard also finds the draw's end (the word
// after normal Tg - 1) and the Metropolis uniform right after it.
__global__ void shard_place_kernel(DevControl *C, const WinInfo *g, int world, int rank, const double *win,
                                   const uint32_t *nend, double *dst, int64_t n_local, int64_t ls, int64_t Tg) {
  __shared__ int64_t s_k0;
  if (C->halt) return;
  if (threadIdx.x == 0) {
    int64_t off = 0;
    bool ok = true;
    for (int q = 0; q < world; q++) {
      if (g[q].cnt_lo < 0 || g[q].cnt_hi < g[q].cnt_lo || g[q].n_win < g[q].cnt_hi) ok = false;
      if (q < rank) off += g[q].cnt_hi - g[q].cnt_lo;
      if (q + 1 < world && g[q].s_hi != g[q + 1].s_lo) ok = false;
    }
    const WinInfo &m = g[rank];
    const int64_t k0 = ls - off + m.cnt_lo;  // window index of global normal ls
    int err = ok ? 0 : 16;
    if (k0 < 0 || k0 + n_local > m.n_win) err |= 32;
    if (blockIdx.x == 0 && rank == world - 1 && !err) {
      const int64_t kT = Tg - 1 - off + m.cnt_lo;
      if (kT < 0 || kT >= m.n_win) {
        err |= 32;
      } else {
        const uint64_t used = (uint64_t)(m.w0 + nend[kT]);
        const StreamState &st = C->stream;
        C->zig_used = used;
        C->u_word = word_at(st, st.pos + used);
        if (st.kind == PRNG_PCG32) C->seq_next = pcg_advance(st.s[0], 2 * (st.pos + used), st.s[1]);
        else if (st.kind == PRNG_MINSTD) C->seq_next = mod31(minstd_pow(3 * (st.pos + used)) * st.s[0]);
      }
    }
    if (err && blockIdx.x == 0) atomicOr(&C->err, err);
    s_k0 = err ? -1 : k0;
  }
  __syncthreads();
  const int64_t k0 = s_k0;
  if (k0 < 0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = win[k0 + i];
}

int rsv_shard_set_momenta(rsv_ctx *c, int windowed) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  if (!windowed) {
    c->win_mode = 0;
    return 0;
  }
  if (c->kind == PRNG_SFC64)
    return fail(c, RSV_E_INVALID, "sfc64 has no jump-ahead: its single stream cannot be drawn in windows "
                                "(use the blocked layout, rsv_set_blocked_streams)");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  // the shard's sites [goff, goff + T) are normals [goff, goff + T) of the
  // draw; its window covers their expected words with the slack on both sides
  const int64_t slack = shard_slack(c->Tg);
  int64_t w_lo = shard_anchor(c->goff) - slack;
  w_lo = w_lo < 0 ? 0 : w_lo;
  if (c->goff == 0) w_lo = 0;
  const int64_t w_hi = shard_anchor(c->goff + c->T) + slack;
  c->win_wb0 = w_lo / ZB;
  c->win_nb = (w_hi + ZB - 1) / ZB - c->win_wb0;
  if (c->win_wb0 + c->win_nb > momenta_blocks(c->jump_T))
    return fail(c, RSV_E_STATE, "momenta window beyond the jump tables");
  // anchors: the expected first word of the owned range; the first shard's is
  // word 0 (exact), the last shard has none above
  const int64_t lo_g = c->goff + c->own_lo, hi_g = c->goff + c->own_hi;
  c->win_a_lo = lo_g == 0 ? 0 : shard_anchor(lo_g);
  c->win_a_hi = hi_g == c->Tg ? -1 : shard_anchor(hi_g);
  const int64_t w0 = c->win_wb0 * ZB;
  if (c->win_a_lo < w0 + 64 && lo_g != 0)
    return fail(c, RSV_E_STATE, "momenta window starts too close to its anchor (margin too small)");
  const int64_t cap = c->win_nb * ZB;
  if (cap > c->win_cap) {
    if (c->win_out) cudaFree(c->win_out);
    if (c->win_nend) cudaFree(c->win_nend);
    c->win_out = nullptr;
    c->win_nend = nullptr;
    CK(cudaMalloc(&c->win_out, sizeof(double) * (size_t)cap));
    CK(cudaMalloc(&c->win_nend, sizeof(uint32_t) * (size_t)cap));
    c->win_cap = cap;
  }
  c->win_mode = 1;
  return 0;
}

__global__ void winfo_reset_kernel(WinInfo *w) {
  if (threadIdx.x || blockIdx.x) return;
  w->cnt_lo = w->cnt_hi = w->s_lo = w->s_hi = w->n_win = -1;
  w->w0 = 0;
  w->err = 0;
  w->pad = 0;
}

int rsv_shard_momenta_async(rsv_ctx *c, double *winfo_dev) {
  if (!c || !winfo_dev) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->shard || !c->win_mode) return fail(c, RSV_E_STATE, "windowed momenta not enabled (rsv_shard_set_momenta)");
  int r;
  if ((r = ready(c))) return r;
  CK(cudaSetDevice(c->device));
  WinInfo *wi = reinterpret_cast<WinInfo *>(winfo_dev);
  winfo_reset_kernel<<<1, 1, 0, c->stream>>>(wi);
  ZigWin w;
  w.wb0 = c->win_wb0;
  w.w0 = c->win_wb0 * ZB;
  w.cap = c->win_cap;
  w.a_lo = c->win_a_lo;
  w.a_hi = c->win_a_hi;
  w.out = c->win_out;
  w.nend = c->win_a_hi < 0 ? c->win_nend : nullptr;  // only the last shard finds the draw's end
  w.info = wi;
  int l = 1;
  if (launch_momenta_window(mbufs(c), c->kind, w, (int)c->win_nb, c->stream, &l))
    return fail(c, RSV_E_CUDA, "windowed momenta launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  c->launches += l;
  return 0;
}

int rsv_shard_place_async(rsv_ctx *c, const double *winfo_all, int world, int rank) {
  if (!c || !winfo_all || world < 1 || rank < 0 || rank >= world) return fail(c, RSV_E_INVALID, "bad argument");
  if (!c->shard || !c->win_mode) return fail(c, RSV_E_STATE, "windowed momenta not enabled (rsv_shard_set_momenta)");
  if ((rank == world - 1) != (c->win_a_hi < 0) || (rank == 0) != (c->goff + c->own_lo == 0))
    return fail(c, RSV_E_INVALID, "rank %d of %d does not match this shard's position", rank, world);
  CK(cudaSetDevice(c->device));
  const int nb = (int)((c->T + 255) / 256 < 2 * c->sm_count ? (c->T + 255) / 256 : 2 * c->sm_count);
  shard_place_kernel<<<nb, 256, 0, c->stream>>>(c->ctrl, reinterpret_cast<const WinInfo *>(winfo_all), world, rank,
                                                c->win_out, c->win_nend, c->normals + c->goff, c->T, c->goff, c->Tg);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// ---- peer-memory exchange of the per-proposal records (instead of an NCCL
// all-gather): push = this shard's record into every shard's box over
// NVLink, collect = wait for every flag of my box, copy the records out.
// One thread per destination / source rank; the records are 8-23 words.
__global__ void p2p_push_kernel(DevControl *C, P2PBox *const *peers, int world, int rank, const double *src, int kind,
                                int words) {
  __shared__ unsigned long long s_e;
  if (threadIdx.x == 0) {
    const unsigned long long e = C->p2p_seq[kind] + 1;
    C->p2p_seq[kind] = e;
    s_e = e;
  }
  __syncthreads();
  const unsigned long long e = s_e;
  const int q = threadIdx.x;
  if (q >= world) return;
  P2PBox *box = peers[q];
  double *dst = box->rec[kind][e & 1][rank];
  for (int k = 0; k < words; k++) dst[k] = src[k];
  // the record before its flag, for any observer in the system
  asm volatile("fence.sc.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&box->flag[kind][e & 1][rank]), "l"(e) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long p2p_ld_acquire(const unsigned long long *f) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
  return v;
}

__global__ void p2p_collect_kernel(DevControl *C, const P2PBox *box, int world, int kind, int words, double *out,
                                   unsigned long long timeout_ns) {
  const int q = threadIdx.x;
  const unsigned long long e = C->p2p_seq[kind];  // my own push of this exchange came first on the stream
  if (q < world) {
    const unsigned long long *f = &box->flag[kind][e & 1][q];
    const unsigned long long t0 = gtimer_ns();
    bool ok = true;
    while (p2p_ld_acquire(f) != e) {
      if (gtimer_ns() - t0 > timeout_ns) {  // (5 s) a peer is gone: flagged, never a hang
        ok = false;
        break;
      }
      __nanosleep(100);
    }
    if (!ok) atomicOr(&C->err, 64);
    const double *r = box->rec[kind][e & 1][q];
    for (int k = 0; k < words; k++) out[(size_t)q * words + k] = __ldcv(r + k);  // not from a stale L1 line
  }
}

int rsv_shard_p2p_init(rsv_ctx *c, int world, int rank, unsigned char *handle, uint64_t *box_dev) {
  if (!c || !handle) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  if (world < 1 || world > P2P_MAXW || rank < 0 || rank >= world)
    return fail(c, RSV_E_INVALID, "peer exchange supports 1..%d shards (rank %d of %d)", P2P_MAXW, rank, world);
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  if (!c->p2p_box) CK(cudaMalloc(&c->p2p_box, sizeof(P2PBox)));
  CK(cudaMemset(c->p2p_box, 0, sizeof(P2PBox)));
  CK(cudaMemset(c->ctrl->p2p_seq, 0, sizeof(c->ctrl->p2p_seq)));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->p2p_box));
  memcpy(handle, &h, sizeof(h));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "rsv_shard_p2p_init: 64-byte handles");
  if (box_dev) *box_dev = (uint64_t)(uintptr_t)c->p2p_box;
  c->p2p_world = world;
  c->p2p_rank = rank;
  const char *to = getenv("RSV_P2P_TIMEOUT_MS");
  c->p2p_timeout_ns = (to && atoll(to) > 0 ? (unsigned long long)atoll(to) : 5000ull) * 1000000ull;
  return 0;
}

int rsv_shard_p2p_connect(rsv_ctx *c, const unsigned char *handles, const uint64_t *boxes) {
  if (!c || (!handles && !boxes)) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->p2p_box) return fail(c, RSV_E_STATE, "rsv_shard_p2p_init first");
  CK(cudaSetDevice(c->device));
  const int w = c->p2p_world;
  std::vector<P2PBox *> ptr(w, nullptr);
  for (int q = 0; q < w; q++) {
    if (q == c->p2p_rank) {
      ptr[q] = c->p2p_box;
    } else if (boxes && boxes[q]) {  // a shard of this process (same device)
      ptr[q] = reinterpret_cast<P2PBox *>((uintptr_t)boxes[q]);
    } else {  // another process's box: mapped over NVLink
      cudaIpcMemHandle_t h;
      memcpy(&h, handles + 64 * (size_t)q, sizeof(h));
      void *d = nullptr;
      CK(cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess));
      c->p2p_opened.push_back(d);
      ptr[q] = reinterpret_cast<P2PBox *>(d);
    }
  }
  if (!c->p2p_peers) CK(cudaMalloc(&c->p2p_peers, sizeof(P2PBox *) * P2P_MAXW));
  CK(cudaMemcpy(c->p2p_peers, ptr.data(), sizeof(P2PBox *) * w, cudaMemcpyHostToDevice));
  return 0;
}

int rsv_shard_p2p_push_async(rsv_ctx *c, const double *mine_dev, int words) {
  if (!c || !mine_dev) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->p2p_peers) return fail(c, RSV_E_STATE, "peer exchange not connected (rsv_shard_p2p_connect)");
  if (words != SHARD_W && words != (int)(sizeof(WinInfo) / 8)) return fail(c, RSV_E_INVALID, "bad record size");
  CK(cudaSetDevice(c->device));
  p2p_push_kernel<<<1, 32, 0, c->stream>>>(c->ctrl, c->p2p_peers, c->p2p_world, c->p2p_rank, mine_dev,
                                          words == SHARD_W ? 0 : 1, words);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

int rsv_shard_p2p_collect_async(rsv_ctx *c, double *out_dev, int words) {
  if (!c || !out_dev) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->p2p_peers) return fail(c, RSV_E_STATE, "peer exchange not connected (rsv_shard_p2p_connect)");
  if (words != SHARD_W && words != (int)(sizeof(WinInfo) / 8)) return fail(c, RSV_E_INVALID, "bad record size");
  CK(cudaSetDevice(c->device));
  p2p_collect_kernel<<<1, 32, 0, c->stream>>>(c->ctrl, c->p2p_box, c->p2p_world, words == SHARD_W ? 0 : 1, words,
                                             out_dev, c->p2p_timeout_ns);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// ---- run_chain of a time-sharded chain (sampler.py:291-358): every shard
// runs the same theta kernel on the all-gathered statistics, so the
// parameters stay identical across shards -----------------------------------
int rsv_shard_run_begin(rsv_ctx *c, double dt, const rsv_prior *prior, int64_t n_burnin, int64_t n_samples,
                        int64_t thin) {
  if (!c || !prior) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  int r;
  if ((r = ready(c))) return r;
  if (n_burnin < 0 || n_samples < 1 || thin < 1) return fail(c, RSV_E_INVALID, "bad burn-in / samples / thin");
  const double pv[] = {prior->mu_var, prior->xi_var, prior->var_shape, prior->var_scale, prior->phi_a, prior->phi_b};
  for (double v : pv)
    if (!(v > 0.0)) return fail(c, RSV_E_INVALID, "prior variances, shapes and scales must be positive");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  if (!c->kdev) CK(cudaMalloc(&c->kdev, sizeof(TrajConsts)));
  if (!c->run) CK(cudaMalloc(&c->run, sizeof(DevRun)));
  if (n_samples > c->run_cap) {
    if (c->run_store) cudaFree(c->run_store);
    CK(cudaMalloc(&c->run_store, (size_t)n_samples * (5 * sizeof(double) + sizeof(double) + sizeof(int64_t) +
                                                      sizeof(int32_t))));
    c->run_cap = n_samples;
  }
  DevRun hr;
  memset(&hr, 0, sizeof(hr));
  hr.n_burnin = n_burnin;
  hr.thin = thin;
  hr.n_store = n_samples;
  char *base = (char *)c->run_store;
  hr.params = (double *)base;
  hr.delta_h = hr.params + 5 * n_samples;
  hr.iters = (int64_t *)(hr.delta_h + n_samples);
  hr.accept = (int32_t *)(hr.iters + n_samples);
  hr.storm_sweep = -1;
  CK(cudaMemcpyAsync(c->run, &hr, sizeof(DevRun), cudaMemcpyHostToDevice, c->stream));
  const TrajConsts k0 = traj_consts(*c->h_prm, dt);
  CK(cudaMemcpyAsync(c->kdev, &k0, sizeof(TrajConsts), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  CK(cudaMemsetAsync(&c->ctrl->halt, 0, sizeof(int32_t), c->stream));
  c->run_prior = DevPrior{prior->mu_mean, prior->mu_var, prior->xi_mean, prior->xi_var,
                          prior->var_shape, prior->var_scale, prior->phi_a, prior->phi_b};
  c->run_dt = dt;
  c->run_active = 1;
  return sync(c);
}

// the theta draws of one sweep, after rsv_shard_decide_async (statistics of
// the kept path over the whole series, combined from every shard)
int rsv_shard_theta_async(rsv_ctx *c) {
  if (!c || !c->shard || !c->run_active) return fail(c, RSV_E_STATE, "no sharded run (rsv_shard_run_begin)");
  CK(cudaSetDevice(c->device));
  int l = 0;
  if (launch_theta_sweep(c->ctrl, c->prm, c->kdev, c->run, c->run_prior, c->run_dt, c->Tg, c->sfc_snaps, c->stream, &l,
                         0))
    return fail(c, RSV_E_CUDA, "theta kernel launch failed");
  c->launches += l;
  return 0;
}

int rsv_shard_run_end(rsv_ctx *c, int64_t *iters, double *params, int32_t *accept, double *delta_h,
                      int64_t *n_stored, int64_t *storm_sweep) {
  if (!c || !c->shard || !c->run_active) return fail(c, RSV_E_STATE, "no sharded run (rsv_shard_run_begin)");
  CK(cudaSetDevice(c->device));
  c->run_active = 0;
  DevRun hr;
  CK(cudaMemcpyAsync(&hr, c->run, sizeof(DevRun), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_prm, c->prm, sizeof(DevParams), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemsetAsync(&c->ctrl->halt, 0, sizeof(int32_t), c->stream));
  int r;
  if ((r = pull_ctrl(c)) || (r = check_err_bits(c))) return r;
  if ((r = refresh_graph_params(c))) return r;
  if (storm_sweep) *storm_sweep = hr.storm_sweep;
  if (n_stored) *n_stored = hr.stored;
  if (hr.storm_sweep >= 0)
    return fail(c, RSV_E_STORM, "more than %d of the last %d HMC proposals diverged at sweep %lld", RUN_STORM_LIMIT,
                RUN_STORM_WINDOW, (long long)hr.storm_sweep);
  if (hr.degenerate) return fail(c, RSV_E_INVALID, "degenerate full-conditional precision");
  const int64_t n = hr.stored;
  if (params) CK(cudaMemcpyAsync(params, hr.params, sizeof(double) * 5 * n, cudaMemcpyDeviceToHost, c->stream));
  if (delta_h) CK(cudaMemcpyAsync(delta_h, hr.delta_h, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  if (iters) CK(cudaMemcpyAsync(iters, hr.iters, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  if (accept) CK(cudaMemcpyAsync(accept, hr.accept, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

// results recorded by rsv_shard_decide_async since the last call (syncs)
int rsv_shard_results(rsv_ctx *c, rsv_result *out, int max_n, int *n_out) {
  if (!c || !n_out) return fail(c, RSV_E_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  int32_t n = 0;
  CK(cudaMemcpyAsync(&n, c->ring_count, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int r;
  if ((r = pull_ctrl(c))) return r;
  if (c->h_ctrl->err & 8) return fail(c, RSV_E_CUDA, "shards drew different momenta streams");
  if ((r = check_err_bits(c))) return r;
  const int m = n < c->ring_cap ? n : c->ring_cap;
  if (m > 0 && c->ring) {
    CK(cudaMemcpy(c->h_ring, c->ring, sizeof(DevResult) * m, cudaMemcpyDeviceToHost));
    for (int i = 0; i < m && i < max_n; i++) to_result(c->h_ring[i], out + i);
  }
  *n_out = n;
  CK(cudaMemset(c->ring_count, 0, sizeof(int32_t)));
  return 0;
}

int rsv_latent_slice(rsv_ctx *c, int64_t offset, int64_t n, double *buf, int to_ctx, int on_device) {
  if (!c || (!buf && n > 0)) return fail(c, RSV_E_INVALID, "null argument");
  if (offset < 0 || n < 0 || offset + n > c->T) return fail(c, RSV_E_INVALID, "slice out of range");
  if (!c->has_latent) return fail(c, RSV_E_STATE, "latent path not set");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = pull_ctrl(c))) return r;
  double *h = c->hbuf[c->h_ctrl->cur & 1] + offset;
  if (n == 0) return 0;
  if (to_ctx) {
    CK(cudaMemcpyAsync(h, buf, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       c->stream));
  } else {
    CK(cudaMemcpyAsync(buf, h, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       c->stream));
  }
  return sync(c);
}

// ---- simulate_rsv on the device (data.py:72-95) ----------------------------
int rsv_simulate(int device, const rsv_params *p, int64_t T, rsv_prng_state *st, double *h, double *y,
                 double *log_rv, int on_device) {
  if (!p || !st || !h || !y || !log_rv) return fail(nullptr, RSV_E_INVALID, "null argument");
  if (T < 2) return fail(nullptr, RSV_E_INVALID, "need t_len >= 2, got %lld", (long long)T);
  if (st->kind < 0 || st->kind > 3) return fail(nullptr, RSV_E_INVALID, "invalid bit generator state");
  if (!(p->phi > -1.0 && p->phi < 1.0) || !(p->sigma_eta_sq > 0.0) || !(p->sigma_u_sq > 0.0))
    return fail(nullptr, RSV_E_INVALID, "params outside the model's domain");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(nullptr, RSV_E_CUDA, "no CUDA device %d", device);
  // a lean context: only what the momenta draw of 3T normals needs
  rsv_ctx *c = new rsv_ctx();
  c->device = device;
  c->T = c->Tg = 3 * T;
  int r = 0;
  double *work = nullptr, *out = nullptr;
  auto body = [&]() -> int {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    const int64_t Tn = 3 * T;
    CK(cudaMalloc(&c->normals, sizeof(double) * (size_t)((Tn + 7) / 8 * 8)));
    CK(cudaMalloc(&c->zscratch, momenta_scratch_bytes(Tn)));
    CK(cudaMemset(c->zscratch, 0, momenta_scratch_bytes(Tn)));
    const int64_t nw = momenta_words(Tn) + 64;
    CK(cudaMalloc(&c->sfc_words, sizeof(uint64_t) * nw));
    CK(cudaMalloc(&c->sfc_snaps, sizeof(uint64_t) * 4 * (nw / SFC_SNAP + 2)));
    CK(cudaMalloc(&c->bjump, momenta_jump_bytes(Tn)));
    CK(cudaMalloc(&c->ctrl, sizeof(DevControl)));
    CK(cudaMallocHost(&c->h_ctrl, sizeof(DevControl)));
    memset(c->h_ctrl, 0, sizeof(DevControl));
    StreamState ss;
    ss.kind = st->kind;
    ss.reserved = 0;
    for (int i = 0; i < 4; i++) ss.s[i] = st->s[i];
    ss.pos = st->pos;
    c->h_ctrl->stream = ss;
    c->h_ctrl->seq_state = ss.kind == PRNG_PCG32    ? pcg_advance(ss.s[0], 2 * ss.pos, ss.s[1])
                           : ss.kind == PRNG_MINSTD ? mod31(minstd_pow(3 * ss.pos) * ss.s[0])
                                                    : 0;
    c->kind = ss.kind;
    CK(cudaMemcpy(c->ctrl, c->h_ctrl, sizeof(DevControl), cudaMemcpyHostToDevice));
    if (momenta_init(c->stream, c->bjump, Tn)) return fail(c, RSV_E_CUDA, "momenta table init failed");
    int l = 0;
    if (launch_momenta(mbufs(c), c->kind, Tn, c->stream, &l) || launch_momenta_advance(mbufs(c), c->stream, &l))
      return fail(c, RSV_E_CUDA, "momenta launch failed");
    const int64_t n_chunks = (T - 1 + 255) / 256;
    CK(cudaMalloc(&work, sizeof(double) * (size_t)(T + 2 * n_chunks + 8)));
    double *dh = h, *dy = y, *dl = log_rv;
    if (!on_device) {
      CK(cudaMalloc(&out, sizeof(double) * 3 * (size_t)T));
      dh = out;
      dy = out + T;
      dl = out + 2 * T;
    }
    if (launch_simulate(c->normals, T, p->phi, p->mu, p->xi, p->sigma_eta_sq, p->sigma_u_sq, dh, dy, dl, work,
                        c->stream, &l))
      return fail(c, RSV_E_CUDA, "simulate launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (!on_device) {
      CK(cudaMemcpyAsync(h, dh, sizeof(double) * T, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(y, dy, sizeof(double) * T, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(log_rv, dl, sizeof(double) * T, cudaMemcpyDeviceToHost, c->stream));
    }
    int q;
    if ((q = pull_ctrl(c)) || (q = check_err_bits(c))) return q;
    st->pos = c->h_ctrl->stream.pos;
    for (int i = 0; i < 4; i++) st->s[i] = c->h_ctrl->stream.s[i];
    return 0;
  };
  r = body();
  if (work) cudaFree(work);
  if (out) cudaFree(out);
  if (r) g_err = c->err;
  rsv_destroy(c);
  return r;
}

// ---- blocked momenta streams (config 5) -----------------------------------
static int set_blocks(rsv_ctx *c, int64_t block_len, int64_t first_block, int64_t n_blocks, const uint64_t *states);

int rsv_set_blocked_streams(rsv_ctx *c, int64_t block_len, int64_t n_blocks, const uint64_t *states) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (c->shard || c->ens_C) return fail(c, RSV_E_STATE, "blocked momenta need a single-chain context");
  return set_blocks(c, block_len, 0, n_blocks, states);
}

// a time-sharded chain: the shard holds the streams of the blocks its local
// range (owned sites and margins) touches, [first_block, first_block +
// n_blocks) of the series' Tg / block_len blocks; a block in two shards'
// ranges is drawn by both, from identical states
int rsv_shard_set_blocked_streams(rsv_ctx *c, int64_t block_len, int64_t first_block, int64_t n_blocks,
                                  const uint64_t *states) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!c->shard) return fail(c, RSV_E_STATE, "not a shard context (rsv_create_shard)");
  if (states && n_blocks) {
    if (block_len < 64 || block_len % 8 || c->Tg % block_len)
      return fail(c, RSV_E_INVALID, "blocks must tile the series (block length a multiple of 8, >= 64)");
    const int64_t j0 = c->goff / block_len, j1 = (c->goff + c->T + block_len - 1) / block_len;
    if (first_block != j0 || n_blocks != j1 - j0)
      return fail(c, RSV_E_INVALID, "shard [%lld, %lld) needs blocks [%lld, %lld)", (long long)c->goff,
                  (long long)(c->goff + c->T), (long long)j0, (long long)j1);
  }
  return set_blocks(c, block_len, first_block, n_blocks, states);
}

static int set_blocks(rsv_ctx *c, int64_t block_len, int64_t first_block, int64_t n_blocks, const uint64_t *states) {
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  if (!states || n_blocks == 0) {  // back to the single-stream layout
    if (c->blocks) cudaFree(c->blocks);
    if (c->h_blocks) cudaFreeHost(c->h_blocks);
    c->blocks = c->h_blocks = nullptr;
    c->block_len = 0;
    c->n_blocks = 0;
    c->block_first = 0;
    drop_graphs(c);
    return 0;
  }
  if (!c->shard && (block_len < 64 || block_len % 8 || block_len * n_blocks != c->T || n_blocks > (1 << 24)))
    return fail(c, RSV_E_INVALID, "blocks must tile the series: %lld x %lld != %lld (block length a multiple of 8, >= 64)",
                (long long)n_blocks, (long long)block_len, (long long)c->T);
  if (n_blocks != c->n_blocks) {
    if (c->blocks) cudaFree(c->blocks);
    if (c->h_blocks) cudaFreeHost(c->h_blocks);
    c->blocks = c->h_blocks = nullptr;
    CK(cudaMalloc(&c->blocks, sizeof(EnsChain) * (size_t)n_blocks));
    CK(cudaMallocHost(&c->h_blocks, sizeof(EnsChain) * (size_t)n_blocks));
  }
  memset(c->h_blocks, 0, sizeof(EnsChain) * (size_t)n_blocks);
  for (int64_t i = 0; i < n_blocks; i++)
    for (int k = 0; k < 4; k++) c->h_blocks[i].st[k] = states[4 * i + k];
  CK(cudaMemcpy(c->blocks, c->h_blocks, sizeof(EnsChain) * (size_t)n_blocks, cudaMemcpyHostToDevice));
  const bool changed = c->block_len != block_len || c->n_blocks != (int)n_blocks || c->block_first != first_block;
  c->block_len = block_len;
  c->n_blocks = (int)n_blocks;
  c->block_first = first_block;
  if (changed) drop_graphs(c);
  return 0;
}

int rsv_get_blocked_streams(rsv_ctx *c, uint64_t *states) {
  if (!c || !states) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->blocks) return fail(c, RSV_E_STATE, "no blocked streams set");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(c->h_blocks, c->blocks, sizeof(EnsChain) * (size_t)c->n_blocks, cudaMemcpyDeviceToHost));
  for (int i = 0; i < c->n_blocks; i++)
    for (int k = 0; k < 4; k++) states[4 * (size_t)i + k] = c->h_blocks[i].st[k];
  return 0;
}

// ---- run_chain on the device ---------------------------------------------
int rsv_get_params(rsv_ctx *c, rsv_params *out) {
  if (!c || !out) return fail(c, RSV_E_INVALID, "null argument");
  if (!c->has_params) return fail(c, RSV_E_STATE, "params not set (rsv_set_params)");
  const DevParams &q = *c->h_prm;
  out->phi = q.phi;
  out->mu = q.mu;
  out->xi = q.xi;
  out->sigma_eta_sq = q.se2;
  out->sigma_u_sq = q.su2;
  return 0;
}

int rsv_run_chain(rsv_ctx *c, double dt, int n_steps, int fuse, const rsv_prior *prior, int64_t n_burnin,
                  int64_t n_samples, int64_t thin, int64_t *iters, double *params, int32_t *accept,
                  double *delta_h, int64_t *storm_sweep) {
  if (!c || !prior) return fail(c, RSV_E_INVALID, "null argument");
  int r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  if (c->shard || c->ens_C) return fail(c, RSV_E_STATE, "rsv_run_chain needs a single-chain context");
  if (n_burnin < 0 || n_samples < 1 || thin < 1) return fail(c, RSV_E_INVALID, "bad burn-in / samples / thin");
  const double pv[] = {prior->mu_var, prior->xi_var, prior->var_shape, prior->var_scale, prior->phi_a, prior->phi_b};
  for (double v : pv)
    if (!(v > 0.0)) return fail(c, RSV_E_INVALID, "prior variances, shapes and scales must be positive");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  if (!c->kdev) CK(cudaMalloc(&c->kdev, sizeof(TrajConsts)));
  if (!c->run) CK(cudaMalloc(&c->run, sizeof(DevRun)));
  if (n_samples > c->run_cap) {
    if (c->run_store) cudaFree(c->run_store);
    CK(cudaMalloc(&c->run_store, (size_t)n_samples * (5 * sizeof(double) + sizeof(double) + sizeof(int64_t) +
                                                      sizeof(int32_t))));
    c->run_cap = n_samples;
  }
  DevRun hr;
  memset(&hr, 0, sizeof(hr));
  hr.n_burnin = n_burnin;
  hr.thin = thin;
  hr.n_store = n_samples;
  char *base = (char *)c->run_store;
  hr.params = (double *)base;
  hr.delta_h = hr.params + 5 * n_samples;
  hr.iters = (int64_t *)(hr.delta_h + n_samples);
  hr.accept = (int32_t *)(hr.iters + n_samples);
  hr.storm_sweep = -1;
  CK(cudaMemcpyAsync(c->run, &hr, sizeof(DevRun), cudaMemcpyHostToDevice, c->stream));
  const TrajConsts k0 = traj_consts(*c->h_prm, dt);
  CK(cudaMemcpyAsync(c->kdev, &k0, sizeof(TrajConsts), cudaMemcpyHostToDevice, c->stream));
  DevPrior pr{prior->mu_mean, prior->mu_var, prior->xi_mean, prior->xi_var,
              prior->var_shape, prior->var_scale, prior->phi_a, prior->phi_b};
  // one sweep = one graph: momenta, trajectory (+ statistics, device theta
  // constants), theta draws.  Not cached (the prior is baked in).
  const TrajGeom g = traj_geometry(c->T, n_steps, c->sm_count, c->variant < 0 ? -1 : c->variant);
  // longer trajectories than a tile holds run as streamed elementary steps
  if (g.ok && (g.variant < 11 || g.variant > 14))
    return fail(c, RSV_E_STATE, "device run_chain needs a persistent shape");
  TrajArgs ta = g.ok ? traj_args(c, dt, n_steps, fuse, g) : TrajArgs{};
  ta.stats = 1;
  ta.kdev = c->kdev;
  ta.pdl = 1;
  // graphs of KS sweeps (fewer graph launches: the gap between two graphs
  // is ~4 us, between two kernels of one graph ~1 us) and of one sweep
  constexpr int KS = 8;
  cudaGraph_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  int l = 0;
  for (int gi = 0; gi < 2; gi++) {
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    l = 0;
    for (int k = 0; k < (gi == 0 ? KS : 1); k++) {
      // programmatic dependent launches: momenta after the previous sweep's
      // theta kernel, trajectory after the momenta, theta after the trajectory
      MomentaBufs mb = mbufs(c);
      mb.pdl = (k > 0 && !getenv("RSV_NO_PDL") && !getenv("RSV_NO_PDL_SWEEP")) ? 1 : 0;
      ok &= launch_momenta(mb, c->kind, c->Tg, c->stream, &l) == 0;
      if (g.ok) ok &= launch_trajectory(ta, c->stream, &l) == 0;
      else ok &= enqueue_fallback(c, dt, n_steps, 1, &l);
      ok &= launch_theta_sweep(c->ctrl, c->prm, c->kdev, c->run, pr, dt, c->T, c->sfc_snaps, c->stream, &l,
                               g.ok && !getenv("RSV_NO_PDL") && !getenv("RSV_NO_PDL_SWEEP") ? 1 : 0) == 0;
    }
    cudaError_t e = cudaStreamEndCapture(c->stream, &graph[gi]);
    if (!ok || e != cudaSuccess) {
      for (int q = 0; q < 2; q++) {
        if (exec[q]) cudaGraphExecDestroy(exec[q]);
        if (graph[q]) cudaGraphDestroy(graph[q]);
      }
      return fail(c, RSV_E_CUDA, "run_chain graph capture failed: %s", cudaGetErrorString(e));
    }
    CK(cudaGraphInstantiate(&exec[gi], graph[gi], 0));
  }
  const int lps = l;  // kernel launches per sweep
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  CK(cudaMemsetAsync(&c->ctrl->halt, 0, sizeof(int32_t), c->stream));
  const int64_t n_sweeps = n_burnin + n_samples * thin;
  int64_t storm = -1;
  cudaError_t le = cudaSuccess;
  for (int64_t i = 0; i < n_sweeps && le == cudaSuccess;) {
    const int k = n_sweeps - i >= KS ? KS : 1;
    le = cudaGraphLaunch(exec[k == KS ? 0 : 1], c->stream);
    c->launches += (int64_t)lps * k;
    const int64_t before = i;
    i += k;
    if ((before >> 8) != (i >> 8) || i == n_sweeps) {  // every 256 sweeps: early exit on a storm
      if ((le = cudaMemcpyAsync(&hr, c->run, sizeof(DevRun), cudaMemcpyDeviceToHost, c->stream)) == cudaSuccess &&
          (le = cudaStreamSynchronize(c->stream)) == cudaSuccess && hr.storm_sweep >= 0) {
        storm = hr.storm_sweep;
        break;
      }
    }
  }
  // a stop (storm / degenerate) left every later kernel of the run a no-op;
  // re-arm the context for ordinary calls
  if (le == cudaSuccess) le = cudaMemsetAsync(&c->ctrl->halt, 0, sizeof(int32_t), c->stream);
  CK(cudaStreamSynchronize(c->stream));
  for (int q = 0; q < 2; q++) {
    cudaGraphExecDestroy(exec[q]);
    cudaGraphDestroy(graph[q]);
  }
  if (le != cudaSuccess) return fail(c, RSV_E_CUDA, "run_chain: %s", cudaGetErrorString(le));
  CK(cudaMemcpyAsync(&hr, c->run, sizeof(DevRun), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_prm, c->prm, sizeof(DevParams), cudaMemcpyDeviceToHost, c->stream));
  if ((r = pull_ctrl(c)) || (r = check_err_bits(c))) return r;
  if ((r = refresh_graph_params(c))) return r;
  if (storm_sweep) *storm_sweep = storm;
  if (storm >= 0) return fail(c, RSV_E_STORM, "more than %d of the last %d HMC proposals diverged at sweep %lld",
                              RUN_STORM_LIMIT, RUN_STORM_WINDOW, (long long)storm);
  if (hr.degenerate) return fail(c, RSV_E_INVALID, "degenerate full-conditional precision");
  const int64_t n = hr.stored;
  if (params) CK(cudaMemcpyAsync(params, hr.params, sizeof(double) * 5 * n, cudaMemcpyDeviceToHost, c->stream));
  if (delta_h) CK(cudaMemcpyAsync(delta_h, hr.delta_h, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  if (iters) CK(cudaMemcpyAsync(iters, hr.iters, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  if (accept) CK(cudaMemcpyAsync(accept, hr.accept, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

// ---- ensemble of independent chains (config 4) -----------------------------
int rsv_ens_create(rsv_ctx **out, int device, int n_chains, int64_t T_chain) {
  if (!out) return fail(nullptr, RSV_E_INVALID, "out is null");
  *out = nullptr;
  if (n_chains < 1) return fail(nullptr, RSV_E_INVALID, "need at least one chain, got %d", n_chains);
  if (T_chain < 64 || T_chain % 8)
    return fail(nullptr, RSV_E_INVALID, "chain length must be a multiple of 8 and >= 64, got %lld",
                (long long)T_chain);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, RSV_E_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, RSV_E_INVALID, "device %d out of range", device);
  rsv_ctx *c = new rsv_ctx();
  const int64_t T = (int64_t)n_chains * T_chain;
  c->own_lo = 0;
  c->own_hi = T;
  c->ens_C = n_chains;
  c->ens_Tc = T_chain;
  c->kind = PRNG_SFC64;
  int r = create_impl(c, device, T, T);
  if (!r) {
    const int64_t tiles = (T + T_chain - 1) / T_chain + (T + 63) / 64 + 16;  // >= tiles of any ensemble geometry
    if (cudaMalloc(&c->ens_cur, (size_t)n_chains) != cudaSuccess ||
        cudaMemset(c->ens_cur, 0, (size_t)n_chains) != cudaSuccess ||
        cudaMalloc(&c->ens_parts, sizeof(EnsPart) * 2 * 8 * (size_t)tiles) != cudaSuccess ||
        cudaMalloc(&c->ens, sizeof(EnsChain) * (size_t)n_chains) != cudaSuccess ||
        cudaMemset(c->ens, 0, sizeof(EnsChain) * (size_t)n_chains) != cudaSuccess ||
        cudaMallocHost(&c->h_ens, sizeof(EnsChain) * (size_t)n_chains) != cudaSuccess)
      r = fail(c, RSV_E_CUDA, "ensemble buffers: %s", cudaGetErrorString(cudaGetLastError()));
  }
  if (r) {
    g_err = c->err;
    rsv_destroy(c);
    return r;
  }
  *out = c;
  return 0;
}

static int ens_check(rsv_ctx *c) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  if (!c->ens_C) return fail(c, RSV_E_STATE, "not an ensemble context (rsv_ens_create)");
  return 0;
}

int rsv_ens_set_streams(rsv_ctx *c, const uint64_t *states) {
  int r;
  if ((r = ens_check(c))) return r;
  if (!states) return fail(c, RSV_E_INVALID, "null states");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  memset(c->h_ens, 0, sizeof(EnsChain) * (size_t)c->ens_C);
  for (int i = 0; i < c->ens_C; i++)
    for (int k = 0; k < 4; k++) c->h_ens[i].st[k] = states[4 * (size_t)i + k];
  CK(cudaMemcpyAsync(c->ens, c->h_ens, sizeof(EnsChain) * (size_t)c->ens_C, cudaMemcpyHostToDevice, c->stream));
  c->ens_streams = true;
  return sync(c);
}

static int ens_pull(rsv_ctx *c) {
  CK(cudaMemcpyAsync(c->h_ens, c->ens, sizeof(EnsChain) * (size_t)c->ens_C, cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

int rsv_ens_get_streams(rsv_ctx *c, uint64_t *states) {
  int r;
  if ((r = ens_check(c))) return r;
  if (!states) return fail(c, RSV_E_INVALID, "null states");
  CK(cudaSetDevice(c->device));
  if ((r = ens_pull(c))) return r;
  for (int i = 0; i < c->ens_C; i++)
    for (int k = 0; k < 4; k++) states[4 * (size_t)i + k] = c->h_ens[i].st[k];
  return 0;
}

int rsv_ens_refresh_momenta(rsv_ctx *c, double *normals) {
  int r;
  if ((r = ens_check(c))) return r;
  if (!c->ens_streams) return fail(c, RSV_E_STATE, "streams not set (rsv_ens_set_streams)");
  CK(cudaSetDevice(c->device));
  int l = 0;
  if (launch_momenta_ens(c->ens, c->normals, c->ens_Tc, c->ens_C, c->stream, &l,
                         getenv("RSV_ENS_STAMPS") ? c->dbg : nullptr))
    return fail(c, RSV_E_CUDA, "ensemble momenta launch failed");
  ens_advance_kernel<<<(c->ens_C + 127) / 128, 128, 0, c->stream>>>(c->ens, c->ens_C);
  c->launches += l + 1;
  CK(cudaGetLastError());
  if (normals && (r = copy_out(c, normals, c->normals, c->T, 0))) return r;
  return sync(c);
}

static int ens_graph(rsv_ctx *c, double dt, int n_steps, int fuse, rsv_ctx::Cached **out) {
  GraphKey k{-1, n_steps, fuse ? 1 : 0, 0, 0, dt};
  auto it = c->ens_graphs.find(k);
  if (it != c->ens_graphs.end()) {
    *out = it->second;
    return 0;
  }
  const TrajGeom g = traj_geometry_ens(c->T, c->ens_Tc, n_steps, c->sm_count);
  if (!g.ok) return fail(c, RSV_E_INVALID, "n_steps=%d too large for one trajectory tile", n_steps);
  auto *cg = new rsv_ctx::Cached();
  cg->dt = dt;
  cg->args = traj_args(c, dt, n_steps, fuse, g);
  cg->args.Tc = c->ens_Tc;
  cg->args.n_chains = c->ens_C;
  cg->args.ens_cur = c->ens_cur;
  cg->args.ens_parts = c->ens_parts;
  cg->args.ens = c->ens;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int l = 0;
  bool ok = launch_momenta_ens(c->ens, c->normals, c->ens_Tc, c->ens_C, c->stream, &l) == 0;
  ok &= launch_trajectory(cg->args, c->stream, &l) == 0;
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (!ok || e != cudaSuccess) {
    delete cg;
    return fail(c, RSV_E_CUDA, "ensemble graph capture failed: %s", cudaGetErrorString(e));
  }
  cg->graph = graph;
  size_t n = 0;
  CK(cudaGraphGetNodes(graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CK(cudaGraphGetNodes(graph, nodes.data(), &n));
  const void *fn = traj_kernel_fn_ens(fuse);
  cg->traj_node = nullptr;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) {
      cudaKernelNodeParams kp;
      CK(cudaGraphKernelNodeGetParams(nd, &kp));
      if (fn && kp.func == fn) {
        cg->traj_node = nd;
        cg->traj_params = kp;
      }
    }
  }
  if (!cg->traj_node) return fail(c, RSV_E_CUDA, "ensemble trajectory node not found");
  CK(cudaGraphInstantiate(&cg->exec, graph, 0));
  c->ens_graphs.emplace(k, cg);
  *out = cg;
  return 0;
}

int rsv_ens_hmc_update(rsv_ctx *c, double dt, int n_steps, int fuse, int n_rounds, int32_t *accept,
                       double *delta_h) {
  int r;
  if ((r = ens_check(c))) return r;
  if ((r = check_md(c, dt, n_steps)) || (r = ready(c))) return r;
  if (!c->ens_streams) return fail(c, RSV_E_STATE, "streams not set (rsv_ens_set_streams)");
  if (n_rounds < 1) return fail(c, RSV_E_INVALID, "n_rounds must be >= 1");
  CK(cudaSetDevice(c->device));
  rsv_ctx::Cached *cg = nullptr;
  if ((r = ens_graph(c, dt, n_steps, fuse, &cg))) return r;
  if (c->timing && (r = ensure_events(c, 4 * (size_t)n_rounds + 4))) return r;
  CK(cudaMemsetAsync(&c->ctrl->err, 0, sizeof(int32_t), c->stream));
  for (int i = 0; i < n_rounds; i++) {
    if (c->flush_bytes > 0) CK(cudaMemsetAsync(c->flush_buf, i & 0xff, (size_t)c->flush_bytes, c->stream));
    if (c->timing) CK(cudaEventRecord(c->evpool[4 + 4 * i], c->stream));
    CK(cudaGraphLaunch(cg->exec, c->stream));
    if (c->timing) CK(cudaEventRecord(c->evpool[4 + 4 * i + 3], c->stream));
    c->launches += 3;
  }
  if ((r = ens_pull(c))) return r;
  if ((r = pull_ctrl(c)) || (r = check_err_bits(c))) return r;
  for (int i = 0; i < c->ens_C; i++) {
    if (accept) accept[i] = c->h_ens[i].last_accept;
    if (delta_h) delta_h[i] = c->h_ens[i].last_dh;
  }
  if (c->timing) {
    c->last_traj_ms.assign(n_rounds, 0.0);
    c->last_mom_ms.assign(n_rounds, 0.0);
    c->last_total_ms.assign(n_rounds, 0.0);
    for (int i = 0; i < n_rounds; i++) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, c->evpool[4 + 4 * i], c->evpool[4 + 4 * i + 3]));
      c->last_total_ms[i] = t;
    }
  }
  return 0;
}

int rsv_ens_counts(rsv_ctx *c, int32_t *n_accept, int32_t *n_diverged) {
  int r;
  if ((r = ens_check(c))) return r;
  CK(cudaSetDevice(c->device));
  if ((r = ens_pull(c))) return r;
  for (int i = 0; i < c->ens_C; i++) {
    if (n_accept) n_accept[i] = c->h_ens[i].n_accept;
    if (n_diverged) n_diverged[i] = c->h_ens[i].n_diverged;
  }
  return 0;
}

int rsv_kernel_stamps(rsv_ctx *c, uint64_t out[5]) {
  if (!c || !out) return fail(c, RSV_E_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  int r;
  if ((r = pull_ctrl(c))) return r;
  for (int i = 0; i < 5; i++) out[i] = c->h_ctrl->t_stamp[i];
  return 0;
}

int rsv_set_timing(rsv_ctx *c, int enable) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  c->timing = enable < 0 ? 0 : enable > 2 ? 2 : enable;
  return 0;
}

int rsv_get_timing(rsv_ctx *c, double *traj_ms, double *momenta_ms, double *total_ms) {
  if (!c) return fail(c, RSV_E_INVALID, "null context");
  auto avg = [](const std::vector<double> &v) {
    double s = 0;
    for (double x : v) s += x;
    return v.empty() ? 0.0 : s / v.size();
  };
  if (traj_ms) *traj_ms = avg(c->last_traj_ms);
  if (momenta_ms) *momenta_ms = avg(c->last_mom_ms);
  if (total_ms) *total_ms = avg(c->last_total_ms);
  return 0;
}

}  // extern "C"
