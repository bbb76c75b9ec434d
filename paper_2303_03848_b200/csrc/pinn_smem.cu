// pinn_smem.cu — K3 with shared-memory weights (any instantiated width, runtime depth).
#include "launch.h"
#include "pinn_chain.cuh"
#include <stdlib.h>

namespace pr {
typedef void (*SmemKernel)(PinnArgs);
template <int IN, int ACT>
static SmemKernel smem_kernel_w(int W) {
  switch (W) {
    case 8: return k_pinn_chain<IN, 8, ACT, 2>;
    case 16: return k_pinn_chain<IN, 16, ACT, 2>;
    case 20: return k_pinn_chain<IN, 20, ACT, 2>;
    case 32: return k_pinn_chain<IN, 32, ACT, 2>;
    case 50: return k_pinn_chain<IN, 50, ACT, 1>;
    case 64: return k_pinn_chain<IN, 64, ACT, 1>;
  }
  return nullptr;
}
static SmemKernel smem_kernel(int IN, int W, int act) {
  if (IN == 4) return act ? smem_kernel_w<4, 1>(W) : smem_kernel_w<4, 0>(W);
  if (IN == 2) return act ? smem_kernel_w<2, 1>(W) : smem_kernel_w<2, 0>(W);
  return nullptr;
}
bool pinn_smem_supported(int IN, int W, int act) { return smem_kernel(IN, W, act) != nullptr; }
int pinn_smem_pts(int W) { return W <= 32 ? 2 : 1; }
cudaError_t pinn_smem_prepare(int IN, int W, int act, int smem_bytes) {
  SmemKernel k = smem_kernel(IN, W, act);
  if (!k) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}
cudaError_t launch_pinn_smem(int IN, int W, int act, const PinnArgs &a, dim3 grid, size_t smem, cudaStream_t s) {
  SmemKernel k = smem_kernel(IN, W, act);
  if (!k) return cudaErrorInvalidValue;
  k<<<grid, 128, smem, s>>>(a);
  return cudaGetLastError();
}
}  // namespace pr

namespace pr {
// Latency mode (few grid points): G threads per point.  G = 4 with 20-wide nets is the shuffle
// kernel (k_pinn_chain_split, shared-memory weights); every other G is a group kernel
// (k_pinn_chain_group: shared-memory activation exchange, group-ordered weights through L1).
typedef void (*SplitKernel)(PinnArgs);
static SplitKernel split_kernel(int IN, int W, int act, int G) {
  if (G == 10 && IN == 4 && W == 50) return act ? k_pinn_chain_group<4, 50, 10, 1> : k_pinn_chain_group<4, 50, 10, 0>;
  if (G == 10 && IN == 4 && W == 20) return act ? k_pinn_chain_group<4, 20, 10, 1> : k_pinn_chain_group<4, 20, 10, 0>;
  if (G == 10 && IN == 2 && W == 20 && act == 0) return k_pinn_chain_group<2, 20, 10, 0>;
  if (G == 16 && IN == 4 && W == 64 && act == 0) return k_pinn_chain_group<4, 64, 16, 0>;
  if (G == 8 && IN == 4 && W == 32 && act == 0) return k_pinn_chain_group<4, 32, 8, 0>;
  if (G != 4 || W != 20) return nullptr;
  if (IN == 4) return act ? k_pinn_chain_split<4, 20, 4, 1> : k_pinn_chain_split<4, 20, 4, 0>;
  if (IN == 2 && act == 0) return k_pinn_chain_split<2, 20, 4, 0>;
  return nullptr;
}
bool pinn_split_supported(int IN, int W, int act, int G) { return split_kernel(IN, W, act, G) != nullptr; }
// Group size of the group kernel for a width (0: none).  (W = 50 with G = 25 -- two neurons per
// thread, one point per warp -- measured slower: every warp re-reads the whole weight matrix.)
int pinn_group_G(int W) { return W == 20 ? 10 : W == 32 ? 8 : W == 50 ? 10 : W == 64 ? 16 : 0; }
bool pinn_split_is_group(int W, int G) { return G > 1 && !(W == 20 && G == 4); }
int pinn_split_ppc(int G) { return G ? 4 * (32 / G) : 0; }
cudaError_t pinn_split_prepare(int IN, int W, int act, int G, int smem_bytes) {
  SplitKernel k = split_kernel(IN, W, act, G);
  if (!k) return cudaErrorInvalidValue;
  if (pinn_split_is_group(W, G)) return cudaSuccess;  // group kernels: no dynamic shared memory
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}
cudaError_t launch_pinn_split(int IN, int W, int act, int G, const PinnArgs &a, dim3 grid, size_t smem,
                              cudaStream_t s) {
  SplitKernel k = split_kernel(IN, W, act, G);
  if (!k) return cudaErrorInvalidValue;
  k<<<grid, 128, pinn_split_is_group(W, G) ? 0 : smem, s>>>(a);
  return cudaGetLastError();
}
}  // namespace pr
