// misc.cu — K6 (δ reduction) and K7 (payoff initial state).
#include "launch.h"
#include <cuda_runtime.h>
#include <stdint.h>

namespace pr {

// K7: U_0 = max(S_j − K_b, 0), S_j = j L_b/(M+1)  (Eq. 2; reading Q4)
__global__ void k_payoff(float *U0, int M, int Mp, int B, const double *Lb, const double *Kb) {
  const int b = blockIdx.y;
  const double dS = Lb[b] / (M + 1), K = Kb[b];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < Mp; j += gridDim.x * blockDim.x) {
    const double S = (j + 1) * dS;
    U0[(size_t)b * Mp + j] = (j < M) ? (float)(S > K ? S - K : 0.0) : 0.f;
  }
}

// K6: δ^k = max over (slice, instance) of ‖U^k_n − U^{k−1}_n‖₂ / ‖U^k_n‖₂ (reading Q13).
// Partials hold (Σ d², Σ u²) per (local slice, instance, chunk); chunks are summed in a
// fixed order, the max is order-free, so δ is bitwise reproducible and independent of
// how slices are sharded across ranks.
// One row's chunks summed by one warp in a fixed order: lane l adds chunks l, l+32, … in index
// order, then a fixed xor-shuffle tree; lane 0's result is the one used (deterministic).
__device__ __forceinline__ double row_rel(const double *p, int nch, int lane) {
  double num = 0.0, den = 0.0;
  for (int c = lane; c < nch; c += 32) { num += p[2 * c]; den += p[2 * c + 1]; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  return (den > 0.0) ? sqrt(num) / sqrt(den) : sqrt(num);
}

// one warp per (slice, instance) row; rows ln_lo..ln_hi
__global__ void k_delta(const double *partials, int B, int nch, int ln_lo, int ln_hi,
                        unsigned long long *dmax) {
  const int row = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int total = (ln_hi - ln_lo + 1) * B;
  if (row >= total) return;
  const int ln = ln_lo + row / B, b = row % B;
  const double rel = row_rel(partials + (((size_t)ln * B + b) * nch) * 2, nch, lane);
  // non-negative doubles order like their bit patterns
  if (lane == 0) atomicMax(dmax, (unsigned long long)__double_as_longlong(rel));
}

cudaError_t launch_payoff(float *U0, int M, int Mp, int B, const double *Lb, const double *Kb, cudaStream_t s) {
  dim3 grid((Mp + 255) / 256, B);
  k_payoff<<<grid, 256, 0, s>>>(U0, M, Mp, B, Lb, Kb);
  return cudaGetLastError();
}

// K6 for many chunks per (slice, instance): one 128-thread CTA per pair; thread t sums chunks
// t, t+128, … in order, then a fixed shuffle/shared-memory tree -- still a fixed order.
__global__ void k_delta_wide(const double *partials, int B, int nch, int ln_lo, unsigned long long *dmax) {
  __shared__ double red[8];
  const int ln = ln_lo + blockIdx.x / B, b = blockIdx.x % B;
  const double *p = partials + (((size_t)ln * B + b) * nch) * 2;
  double num = 0.0, den = 0.0;
  for (int c = threadIdx.x; c < nch; c += blockDim.x) { num += p[2 * c]; den += p[2 * c + 1]; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[2 * w] = num; red[2 * w + 1] = den; }
  __syncthreads();
  if (threadIdx.x == 0) {
    num = 0.0; den = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { num += red[2 * q]; den += red[2 * q + 1]; }
    const double rel = (den > 0.0) ? sqrt(num) / sqrt(den) : sqrt(num);
    atomicMax(dmax, (unsigned long long)__double_as_longlong(rel));
  }
}

// Up to kDeltaWarpMax chunks a warp sums a row (k_delta, and the pipelined kernel's tail: the same
// order in the blocking and pipelined schedules; unused chunks are zero), beyond that a CTA per row does
// (k_delta_wide).
constexpr int kDeltaWarpMax = 1024;
cudaError_t launch_delta(const double *partials, int B, int nch, int ln_lo, int ln_hi, unsigned long long *dmax,
                         cudaStream_t s) {
  const int total = (ln_hi - ln_lo + 1) * B;
  if (nch > kDeltaWarpMax)
    k_delta_wide<<<total, 128, 0, s>>>(partials, B, nch, ln_lo, dmax);
  else
    k_delta<<<(total * 32 + 255) / 256, 256, 0, s>>>(partials, B, nch, ln_lo, ln_hi, dmax);
  return cudaGetLastError();
}

}  // namespace pr
