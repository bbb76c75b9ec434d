// pinn_param.cu — K3 with the weights as kernel parameters (constant bank), small networks.
#include <string.h>

#include "launch.h"
#include "pinn_chain.cuh"

namespace pr {
typedef void (*ParamLauncher)(const float *, const PinnArgs &, dim3, cudaStream_t);
template <int IN, int W, int LH, int ACT>
static void launch_param(const float *pk, const PinnArgs &a, dim3 grid, cudaStream_t s) {
  ParamNet<IN, W, LH> P;
  memcpy(P.w, pk, sizeof P.w);
  k_pinn_chain_param<IN, W, LH, ACT><<<grid, 128, 0, s>>>(a, P);
}
struct ParamEntry {
  int IN, W, LH, act;
  ParamLauncher fn;
};
static const ParamEntry kParamKernels[] = {
    {4, 20, 3, 0, launch_param<4, 20, 3, 0>},   // BASELINE configs' network [4,20,20,20,1] tanh
    {4, 20, 3, 1, launch_param<4, 20, 3, 1>},   // same, ReLU
    {2, 20, 3, 0, launch_param<2, 20, 3, 0>},   // 2-input form
};
static ParamLauncher find(int IN, int W, int LH, int act) {
  for (const auto &e : kParamKernels)
    if (e.IN == IN && e.W == W && e.LH == LH && e.act == act) return e.fn;
  return nullptr;
}
bool pinn_param_supported(int IN, int W, int LH, int act) { return find(IN, W, LH, act) != nullptr; }
cudaError_t launch_pinn_param(int IN, int W, int LH, int act, const float *pk, const PinnArgs &a, dim3 grid,
                              cudaStream_t s) {
  ParamLauncher f = find(IN, W, LH, act);
  if (!f) return cudaErrorInvalidValue;
  f(pk, a, grid, s);
  return cudaGetLastError();
}
}  // namespace pr
