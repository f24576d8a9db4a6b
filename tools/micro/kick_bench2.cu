// Which features of the trajectory kernel cost throughput? (development aid)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1603_08114_b200/csrc/exp_table.h"

__device__ const unsigned long long g_tab[64] = RSV_EXP_TAB2_INIT;
constexpr double MAGIC = 6755399441055744.0;

__device__ __forceinline__ double expn(double d, const unsigned long long *tab, int &n) {
  const double t = fma(-d, RSV_INV_LN2_N, MAGIC);
  const double nd = t - MAGIC;
  double r = fma(nd, -RSV_LN2_N_HI, -d);
  r = fma(nd, -RSV_LN2_N_LO, r);
  double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  n = __double2loint(t);
  const unsigned long long tb = tab[n & 63];
  const double S = __hiloint2double((int)(tb >> 32) + (n << 14), (int)(unsigned)tb);
  return fma(S, q, S);
}

// F bits: 1 = per-site Ad/Cd from memory, 2 = masked range check, 4 = flag exchange, 8 = branchy edge dispatch,
//         16 = unmasked range check
template <int F, int R>
__global__ void __launch_bounds__(256, 2) kick_kernel(double *out, const double *ad, const double *cd, int steps,
                                                      int nlo) {
  constexpr int NW = 8;
  __shared__ unsigned long long tab[64];
  __shared__ double s_first[2][NW], s_last[2][NW];
  __shared__ int s_flag[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 64) tab[threadIdx.x] = g_tab[threadIdx.x];
  if (threadIdx.x < NW) s_flag[threadIdx.x] = 0;
  __syncthreads();
  double d[R], p[R], A[R], C[R];
  unsigned cm[R];
  const int base = (blockIdx.x * blockDim.x + threadIdx.x) * R;
  for (int r = 0; r < R; r++) {
    d[r] = 0.01 * ((threadIdx.x + r) % 17) - 0.08;
    p[r] = 0.1 * ((threadIdx.x * 7 + r) % 13) - 0.6;
    if (F & 1) { A[r] = ad[base + r]; C[r] = cd[base + r]; }
    else { A[r] = 1e-3 * (r + 1); C[r] = 1e-4 * r; }
    cm[r] = ((threadIdx.x + r) % 5) ? ~0u : 0u;
  }
  const bool edge = (F & 8) && threadIdx.x == 3;
  const double G = 0.6, bphi = 0.28, c = 0.02;
  unsigned nmax = 0;
  volatile int *vflag = s_flag;
  for (int s = 0; s < steps; s++) {
    for (int r = 0; r < R; r++) d[r] = fma(c, p[r], d[r]);
    double dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
    double dr = __shfl_down_sync(0xffffffffu, d[0], 1);
    if (F & 4) {
      const int slot = s & 1;
      if (lane == 0) s_first[slot][warp] = d[0];
      if (lane == 31) s_last[slot][warp] = d[R - 1];
      __syncwarp();
      if (lane == 0) { __threadfence_block(); vflag[warp] = s + 1; }
      if (lane == 0 && warp > 0) { while (vflag[warp - 1] <= s) {} __threadfence_block(); dl = s_last[slot][warp - 1]; }
      if (lane == 31 && warp < NW - 1) { while (vflag[warp + 1] <= s) {} __threadfence_block(); dr = s_first[slot][warp + 1]; }
    }
    if (edge) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        const double dm = r ? d[r - 1] : dl;
        const double dp = r < R - 1 ? d[r + 1] : dr;
        int n;
        const double E = expn(d[r], tab, n);
        nmax = max(nmax, ((unsigned)n - (unsigned)nlo) & cm[r]);
        const double GG = (r == 2) ? 0.3 : G;
        double pp = p[r] - C[r];
        pp = fma(-GG, d[r], pp);
        pp = fma(bphi, dm + dp, pp);
        pp = fma(A[r], E, pp);
        p[r] = r == 5 ? 0.0 : pp;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; r++) {
        const double dm = r ? d[r - 1] : dl;
        const double dp = r < R - 1 ? d[r + 1] : dr;
        int n;
        const double E = expn(d[r], tab, n);
        if (F & 2) nmax = max(nmax, ((unsigned)n - (unsigned)nlo) & cm[r]);
        if (F & 16) nmax = max(nmax, (unsigned)n - (unsigned)nlo);
        double pp = p[r] - C[r];
        pp = fma(-G, d[r], pp);
        pp = fma(bphi, dm + dp, pp);
        p[r] = fma(A[r], E, pp);
      }
    }
  }
  double acc = nmax;
  for (int r = 0; r < R; r++) acc += d[r] + p[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int F, int R>
void run(const char *name, double *out, const double *ad, const double *cd, int sms) {
  const int steps = 2000, blocks = sms * 2, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kick_kernel<F, R><<<blocks, threads>>>(out, ad, cd, 10, -600);
  cudaEventRecord(a);
  kick_kernel<F, R><<<blocks, threads>>>(out, ad, cd, steps, -600);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double su = (double)blocks * threads * R * steps / (ms * 1e-3);
  printf("%-44s F=%2d R=%d  %.3e site-steps/s  (%.2f /clk/SM)\n", name, F, R, su, su / sms / 1.965e9);
}

int main() {
  const int n = 148 * 2 * 256 * 16;
  double *out, *ad, *cd;
  cudaMalloc(&out, n * 8); cudaMalloc(&ad, n * 8); cudaMalloc(&cd, n * 8);
  cudaMemset(ad, 0, n * 8); cudaMemset(cd, 0, n * 8);
  int sms = 148;
  run<0, 8>("baseline (const Ad/Cd)", out, ad, cd, sms);
  run<1, 8>("Ad/Cd in registers from memory", out, ad, cd, sms);
  run<1 | 16, 8>("+ unmasked range check", out, ad, cd, sms);
  run<1 | 2, 8>("+ masked range check", out, ad, cd, sms);
  run<1 | 2 | 4, 8>("+ flag exchange", out, ad, cd, sms);
  run<1 | 2 | 4 | 8, 8>("+ edge dispatch (1 thread/CTA edge)", out, ad, cd, sms);
  run<1 | 2 | 4, 4>("R=4 masked + flags", out, ad, cd, sms);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
