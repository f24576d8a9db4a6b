// Latency microbenchmarks on the B200 (development aid): dependent-chain
// cycles of DFMA / DADD / FFMA / SHFL / LDS and a CTA barrier.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, long long *cyc, int n) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = fma(x, 0.9999999, 1e-9);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void k_dadd(double *out, long long *cyc, int n) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = x + 1e-9;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void k_ffma(float *out, long long *cyc, int n) {
  float x = threadIdx.x * 1e-9f + 1.0f;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = fmaf(x, 0.9999f, 1e-7f);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void k_shfl(double *out, long long *cyc, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void k_bar(double *out, long long *cyc, int n) {
  __shared__ double s[1024];
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    s[threadIdx.x] = x;
    __syncthreads();
    x = s[(threadIdx.x + 1) % blockDim.x] + 1.0;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}
// 8 independent chains per thread, 1 warp: throughput-per-warp for DFMA
__global__ void k_dfma8(double *out, long long *cyc, int n) {
  double x[8];
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-9 + k;
  long long t0 = clock64();
  for (int i = 0; i < n; i++)
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = fma(x[k], 0.9999999, 1e-9);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
  for (int k = 0; k < 8; k++) s += x[k];
  out[threadIdx.x] = s;
}

int main() {
  double *d; float *f; long long *c, h;
  cudaMalloc(&d, 1024 * 8); cudaMalloc(&f, 1024 * 4); cudaMalloc(&c, 8);
  const int n = 4096;
  auto run = [&](const char *name, auto kern, int threads, auto *buf, double per) {
    kern<<<1, threads>>>(buf, c, n);
    kern<<<1, threads>>>(buf, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s threads=%4d  %.2f cycles/iter\n", name, threads, (double)h / n / per);
  };
  run("DFMA dependent", k_dfma, 32, d, 1);
  run("DADD dependent", k_dadd, 32, d, 1);
  run("FFMA dependent", k_ffma, 32, f, 1);
  run("SHFL(f64)+DADD dependent", k_shfl, 32, d, 1);
  run("DFMA 8 indep chains /FMA", k_dfma8, 32, d, 8);
  run("DFMA 8 indep x 4 warps", k_dfma8, 128, d, 8);
  run("DFMA 8 indep x 16 warps", k_dfma8, 512, d, 8);
  run("STS+BAR+LDS 256 thr", k_bar, 256, d, 1);
  run("STS+BAR+LDS 1024 thr", k_bar, 1024, d, 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
