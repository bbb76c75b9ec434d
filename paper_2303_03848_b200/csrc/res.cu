// res.cu — translation unit of K1 (fine_resident.cuh): the (P, NT, SPB) instantiations.
#include "launch.h"
#include "fine_resident.cuh"
#include <stdlib.h>

namespace pr {
template <int P, int NT, int SPB>
static void launch_res(bool chain, const ResidentArgs &a, int nsys, cudaStream_t s) {
  const int grid = (nsys + SPB - 1) / SPB;
  const bool cn = a.theta != 1.0;  // θ-step with an explicit part (Crank–Nicolson, NEXT-1)
  const bool zz = !cn && a.use_zz;  // zig-zag LU/UL form (θ = 1; fine_resident.cuh)
  if (chain) {
    if (cn) k_resident_chain<P, NT, SPB, true><<<grid, NT * SPB, 0, s>>>(a);
    else if (zz) k_resident_chain<P, NT, SPB, false, true><<<grid, NT * SPB, 0, s>>>(a);
    else k_resident_chain<P, NT, SPB, false><<<grid, NT * SPB, 0, s>>>(a);
  } else {
    if (cn) k_fine_sweep<P, NT, SPB, true><<<grid, NT * SPB, 0, s>>>(a);
    else if (zz) k_fine_sweep<P, NT, SPB, false, true><<<grid, NT * SPB, 0, s>>>(a);
    else k_fine_sweep<P, NT, SPB, false><<<grid, NT * SPB, 0, s>>>(a);
  }
}

cudaError_t launch_resident(bool chain, int M, const ResidentArgs &a, int nsys, cudaStream_t s) {
  if (M <= 64) launch_res<2, 32, 4>(chain, a, nsys, s);
  else if (M <= 128) launch_res<4, 32, 4>(chain, a, nsys, s);
  else if (M <= 256) launch_res<8, 32, 4>(chain, a, nsys, s);
  else if (M <= 512) launch_res<8, 64, 2>(chain, a, nsys, s);
  else if (M <= 1024) {
    static const bool wide = getenv("PR_K1_WIDE") && atoi(getenv("PR_K1_WIDE")) == 1;  // tuning: 8 warps x 4 points
    if (wide) launch_res<4, 256, 1>(chain, a, nsys, s);
    else launch_res<8, 128, 1>(chain, a, nsys, s);
  }
  else launch_res<8, 256, 1>(chain, a, nsys, s);
  return cudaGetLastError();
}
}  // namespace pr
