// Latency of one leapfrog step of the trajectory kernel's loop body (the
// scaled-state kick of traj_dev.cuh) for one warp alone on an SM, and the
// throughput with W warps: what bounds the step loop (development aid).
// Variants (bit mask F): 1 = no exp-table LDS (constant scale), 2 = no
// neighbour shuffles, 4 = uniform table index (no bank conflicts).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1603_08114_b200/csrc/traj_dev.cuh"

using namespace rsv;

template <int F>
__global__ void steps_kernel(double *out, long long *cyc, int n, TrajConsts s) {
  __shared__ __align__(16) unsigned long long tab[RSV_EXP_TAB_N];
  for (int i = threadIdx.x; i < RSV_EXP_TAB_N; i += blockDim.x) tab[i] = g_exp_tab2[i];
  __syncthreads();
  constexpr int R = 4;
  double d[R], p[R], Ad[R], Cd[R];
  for (int r = 0; r < R; r++) {
    d[r] = (0.01 * ((threadIdx.x * 7 + r) % 23) - 0.1) * s.kx;
    p[r] = 0.05 * ((threadIdx.x + 3 * r) % 11) - 0.25;
    Ad[r] = 1e-3 * (1 + r);
    Cd[r] = 1e-4 * r;
  }
  unsigned nmax = 0;
  const long long t0 = clock64();
  for (int step = 0; step < n; step++) {
    for (int r = 0; r < R; r++) d[r] = fma(s.xc_half, p[r], d[r]);
    double dl = d[R - 1], dr = d[0];
    if (!(F & 2)) {
      dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
      dr = __shfl_down_sync(0xffffffffu, d[0], 1);
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const double dm = r ? d[r - 1] : dl;
      const double dp = r < R - 1 ? d[r + 1] : dr;
      double t = MAGIC - d[r];
      const double nd = t - MAGIC;
      const double f = -d[r] - nd;
      double q = fma(f, s.ex3, s.ex2);
      q = fma(q, f, s.ex1);
      q = q * f;
      const int nn = __double2loint(t);
      double S;
      if (F & 1) {
        S = 1.0 + 1e-3 * (nn & 7);
      } else {
        const unsigned long long tb = tab[(F & 4) ? (step & 7) : (nn & (RSV_EXP_TAB_N - 1))];
        S = __hiloint2double((int)(tb >> 32) + (nn << EXP_HI_SHIFT), (int)(unsigned)tb);
      }
      const double E = fma(S, q, S);
      nmax = max(nmax, (unsigned)nn - (unsigned)s.n_lo);
      double pp = p[r] - Cd[r];
      pp = fma(-s.xg_int, d[r], pp);
      pp = fma(s.xbphi, dm + dp, pp);
      pp = fma(Ad[r], E, pp);
      p[r] = pp;
    }
    for (int r = 0; r < R; r++) d[r] = fma(s.xc_half, p[r], d[r]);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double acc = nmax;
  for (int r = 0; r < R; r++) acc += d[r] + p[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  DevParams P{};
  P.phi = 0.97; P.mu = -9.0; P.xi = -0.3; P.se2 = 0.05; P.su2 = 0.1;
  P.inv_su2 = 10.0; P.inv_se2 = 20.0; P.emu = 8103.08; P.one_m_phi2 = 1 - 0.97 * 0.97;
  P.n_lo = -200000; P.n_span = 400000;
  const TrajConsts s = traj_consts(P, 0.02);
  double *out; long long *cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
  const int n = 2000;
  auto run = [&](auto kern, const char *name, int warps, int blocks) {
    kern<<<blocks, 32 * warps>>>(out, cyc, n, s);
    cudaDeviceSynchronize();
    kern<<<blocks, 32 * warps>>>(out, cyc, n, s);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // per-SM FP64 throughput: 14 FP64 instr per site-step, R = 4 sites per thread
    const double site_steps = 4.0 * 32 * warps * n;  // on this SM (blocks <= SMs: one CTA per SM)
    printf("%-34s warps/SM %2d: %7.1f cycles/step, %.2f FP64 warp-instr/cycle (pipe max 2)\n", name, warps,
           (double)c / n, site_steps * 14 / 32 / (double)c);
  };
  for (int w : {1, 4, 8, 16, 32}) run(steps_kernel<0>, "full step", w, 1);
  for (int w : {1, 16}) run(steps_kernel<1>, "no table LDS", w, 1);
  for (int w : {1, 16}) run(steps_kernel<4>, "uniform table index", w, 1);
  for (int w : {1, 16}) run(steps_kernel<2>, "no shuffles", w, 1);
  for (int w : {1, 16}) run(steps_kernel<3>, "no LDS, no shuffles", w, 1);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
