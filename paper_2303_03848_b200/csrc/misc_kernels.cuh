// misc_kernels.cuh — K6 (δ reduction) and K7 (payoff initial state).
#pragma once
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
__global__ void k_delta(const double *partials, int B, int nch, int ln_lo, int ln_hi,
                        unsigned long long *dmax) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = (ln_hi - ln_lo + 1) * B;
  double rel = 0.0;
  if (idx < total) {
    const int ln = ln_lo + idx / B, b = idx % B;
    const double *p = partials + (((size_t)ln * B + b) * nch) * 2;
    double num = 0.0, den = 0.0;
    for (int c = 0; c < nch; ++c) { num += p[2 * c]; den += p[2 * c + 1]; }
    rel = (den > 0.0) ? sqrt(num) / sqrt(den) : sqrt(num);
  }
  // warp max then one atomic per warp; non-negative doubles order like their bit patterns
  unsigned long long v = (unsigned long long)__double_as_longlong(rel);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(dmax, v);
}

}  // namespace pr
