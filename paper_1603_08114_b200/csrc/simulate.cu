// simulate.cu -- data.py:72-95 simulate_rsv on the device.
//
// Draw order of the reference: one normal (initial deviation), T-1 normals
// (latent innovations), T normals (return shocks), T normals (measurement
// noise) -- i.e. 3T consecutive numpy normals from the stream, drawn here by
// the momenta kernel bit for bit.  The AR(1) path out[t+1] = phi*out[t] +
// eta[t] (_kernels.py:70-76) is a linear recurrence with a constant
// coefficient, evaluated as a parallel affine scan: per chunk of SIM_C sites
// from zero, the chunk carries by a one-CTA scan of (phi^C, b) pairs, then
// every site adds phi^j times its chunk's carry.  The grouping differs from
// the sequential recursion, so the path agrees to rounding (~1e-15 relative),
// not bit for bit; returns = exp(h/2) eps and log_rv = xi + h + u as in the
// reference (CUDA exp within an ulp of numpy's).
#include <math.h>

#include "rsv_internal.h"
#include "rsv_launch.h"

namespace rsv {

constexpr int SIM_C = 256;    // sites per chunk (one thread)
constexpr int SIM_NT = 1024;  // threads of the carry scan

// local recurrence per chunk: dev[i] for i in (k*C, (k+1)*C] from a zero start
__global__ void sim_local_kernel(const double *n, int64_t T, double se, double phi, double *dev, double *ends,
                                 int64_t n_chunks) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_chunks) return;
  double x = 0.0;
  const int64_t i0 = k * SIM_C + 1, i1 = min((k + 1) * SIM_C, T - 1);
  for (int64_t i = i0; i <= i1; i++) {
    x = fma(phi, x, __dmul_rn(se, n[i]));  // eta_{i-1} = se * normal[1 + (i - 1)]
    dev[i] = x;
  }
  ends[k] = x;
}

// carries c_k = dev[k*C]: c_0 = dev0, c_{k+1} = phi^C c_k + e_k.  One CTA:
// each thread folds a contiguous run of chunks into one affine map, a block
// scan composes the maps, then each thread re-walks its run.
__global__ void __launch_bounds__(SIM_NT) sim_carry_kernel(const double *ends, double *carry, int64_t n_chunks,
                                                           double phiC, double dev0) {
  __shared__ double sA[SIM_NT], sB[SIM_NT];
  const int t = threadIdx.x;
  const int64_t per = (n_chunks + SIM_NT - 1) / SIM_NT;
  const int64_t k0 = t * per, k1 = min(k0 + per, n_chunks);
  double A = 1.0, B = 0.0;  // x -> A x + B over my chunks
  for (int64_t k = k0; k < k1; k++) {
    A *= phiC;
    B = fma(phiC, B, ends[k]);
  }
  sA[t] = A;
  sB[t] = B;
  __syncthreads();
  for (int off = 1; off < SIM_NT; off <<= 1) {  // inclusive scan of the maps (earlier applied first)
    double a = 1.0, b = 0.0;
    if (t >= off) { a = sA[t - off]; b = sB[t - off]; }
    __syncthreads();
    if (t >= off) {
      const double A2 = sA[t] * a, B2 = fma(sA[t], b, sB[t]);
      sA[t] = A2;
      sB[t] = B2;
    }
    __syncthreads();
  }
  double c = t == 0 ? dev0 : fma(sA[t - 1], dev0, sB[t - 1]);  // carry into my first chunk
  for (int64_t k = k0; k < k1; k++) {
    carry[k] = c;
    c = fma(phiC, c, ends[k]);
  }
}

// dev[i] = local[i] + phi^j c_k (j = i - k*C), then h, returns, log_rv
__global__ void sim_finish_kernel(const double *n, int64_t T, const double *carry, const double *dev, double mu,
                                  double xi, double phi, double su, double dev0, double *h, double *y,
                                  double *lrv) {
  __shared__ double pw[SIM_C + 1];
  if (threadIdx.x == 0) {
    double q = 1.0;
    for (int j = 0; j <= SIM_C; j++) {
      pw[j] = q;
      q *= phi;
    }
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  double d;
  if (i == 0) {
    d = dev0;
  } else {
    const int64_t k = (i - 1) / SIM_C;
    const int j = (int)(i - k * SIM_C);
    d = fma(pw[j], carry[k], dev[i]);
  }
  const double hv = __dadd_rn(mu, d);
  h[i] = hv;
  y[i] = __dmul_rn(exp(__dmul_rn(0.5, hv)), n[T + i]);
  lrv[i] = __dadd_rn(__dadd_rn(xi, hv), __dmul_rn(su, n[2 * T + i]));
}

int launch_simulate(const double *normals, int64_t T, double phi, double mu, double xi, double se2, double su2,
                    double *h, double *y, double *lrv, double *work, cudaStream_t s, int *launches) {
  const double se = sqrt(se2), su = sqrt(su2);
  const int64_t n_chunks = (T - 1 + SIM_C - 1) / SIM_C;
  double *dev = work, *ends = work + T, *carry = ends + n_chunks;
  // dev0 = sqrt(se2 / (1 - phi^2)) * normal[0], rounded on the host exactly as the reference does
  double n0 = 0.0;
  if (cudaMemcpyAsync(&n0, normals, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  const double dev0 = sqrt(se2 / (1.0 - phi * phi)) * n0;
  double phiC = 1.0;
  for (int j = 0; j < SIM_C; j++) phiC *= phi;
  if (n_chunks > 0) {
    sim_local_kernel<<<(unsigned)((n_chunks + 127) / 128), 128, 0, s>>>(normals, T, se, phi, dev, ends, n_chunks);
    sim_carry_kernel<<<1, SIM_NT, 0, s>>>(ends, carry, n_chunks, phiC, dev0);
    *launches += 2;
  }
  sim_finish_kernel<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(normals, T, carry, dev, mu, xi, phi, su, dev0, h, y,
                                                               lrv);
  (*launches)++;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace rsv
