// Throughput of the leapfrog kick arithmetic in isolation (development aid).
// Mode 0: kick + table exp, no exchange; 1: + warp shuffles; 2: + CTA barrier
// per step; 3: like 0 with no table (polynomial-only exp, no LDS).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1603_08114_b200/csrc/exp_table.h"

__device__ const unsigned long long g_tab[64] = RSV_EXP_TAB2_INIT;
constexpr double MAGIC = 6755399441055744.0;

template <int MODE>
__device__ __forceinline__ double expn(double d, const unsigned long long *tab) {
  const double t = fma(-d, RSV_INV_LN2_N, MAGIC);
  const double nd = t - MAGIC;
  double r = fma(nd, -RSV_LN2_N_HI, -d);
  r = fma(nd, -RSV_LN2_N_LO, r);
  double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const int n = __double2loint(t);
  unsigned long long tb;
  if (MODE == 3) tb = 0x3ff0000000000000ULL + ((unsigned long long)(n & 63) << 40);
  else tb = tab[n & 63];
  const double S = __hiloint2double((int)(tb >> 32) + (n << 14), (int)(unsigned)tb);
  return fma(S, q, S);
}

template <int MODE, int R>
__global__ void __launch_bounds__(256, 2) kick_kernel(double *out, int steps) {
  __shared__ unsigned long long tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = g_tab[threadIdx.x];
  __syncthreads();
  double d[R], p[R], A[R], C[R];
  for (int r = 0; r < R; r++) {
    d[r] = 0.01 * ((threadIdx.x + r) % 17) - 0.08;
    p[r] = 0.1 * ((threadIdx.x * 7 + r) % 13) - 0.6;
    A[r] = 1e-3 * (r + 1);
    C[r] = 1e-4 * r;
  }
  const double G = 0.6, bphi = 0.28, c = 0.02;
  for (int s = 0; s < steps; s++) {
    for (int r = 0; r < R; r++) d[r] = fma(c, p[r], d[r]);
    double dl = d[0], dr = d[R - 1];
    if (MODE == 1 || MODE == 2) {
      dl = __shfl_up_sync(0xffffffffu, d[R - 1], 1);
      dr = __shfl_down_sync(0xffffffffu, d[0], 1);
    }
    if (MODE == 2) __syncthreads();
#pragma unroll
    for (int r = 0; r < R; r++) {
      const double dm = r ? d[r - 1] : dl;
      const double dp = r < R - 1 ? d[r + 1] : dr;
      const double E = expn<MODE>(d[r], tab);
      double pp = p[r] - C[r];
      pp = fma(-G, d[r], pp);
      pp = fma(bphi, dm + dp, pp);
      p[r] = fma(A[r], E, pp);
    }
  }
  double acc = 0;
  for (int r = 0; r < R; r++) acc += d[r] + p[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int R>
void run(const char *name, double *out, int sms) {
  const int steps = 2000, blocks = sms * 2, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kick_kernel<MODE, R><<<blocks, threads>>>(out, 10);
  cudaEventRecord(a);
  kick_kernel<MODE, R><<<blocks, threads>>>(out, steps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double su = (double)blocks * threads * R * steps / (ms * 1e-3);
  printf("%-40s R=%d  %.3e site-steps/s  (%.2f per clk per SM @1.965GHz)\n", name, R, su, su / sms / 1.965e9);
}

int main() {
  double *out; cudaMalloc(&out, 148 * 2 * 256 * 8);
  int sms = 148;
  run<0, 8>("kick + table exp, no exchange", out, sms);
  run<1, 8>("+ warp shuffles", out, sms);
  run<2, 8>("+ shuffles + CTA barrier", out, sms);
  run<3, 8>("no table (constant-built scale)", out, sms);
  run<0, 4>("kick + table exp, no exchange", out, sms);
  run<2, 4>("+ shuffles + CTA barrier", out, sms);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
