// peaks_microbench.cu — measured per-GPU peaks of the pipes the non-tensor kernels use (BASELINE.md
// §2: "FP32, FP64 and MUFU peaks have not been measured yet"): fp64 FMA, fp32 FMA, MUFU ex2,
// and the f32<->f64 conversions (F2F) that K1/K2 issue per point; plus the dependent-issue
// latency of DFMA and F2F (one warp, one chain).  Prints one JSON object.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peaks scripts/peaks_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIlp = 8, kIter = 4096;

__global__ void k_dfma(double *out, double a, double b) {
  double x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIter; ++it)
#pragma unroll
    for (int i = 0; i < kIlp; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_ffma(float *out, float a, float b) {
  float x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIter; ++it)
#pragma unroll
    for (int i = 0; i < kIlp; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_ex2(float *out) {
  float x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = 1e-3f * (threadIdx.x + i);
  for (int it = 0; it < kIter; ++it)
#pragma unroll
    for (int i = 0; i < kIlp; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  float s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
// one f32->f64 and one f64->f32 conversion per step and chain
__global__ void k_f2f(float *out) {
  float x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = 1.0f + threadIdx.x + i;
  for (int it = 0; it < kIter; ++it)
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
      double d;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(x[i]));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(x[i]) : "d"(d));
    }
  float s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
// latency: one dependent chain in one warp, clock64 around it
__global__ void k_lat_dfma(double *out, long long *cyc, double a, double b) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < kIter; ++it) x = fma(x, a, b);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lat_f2f(float *out, long long *cyc) {
  float x = 1.0f + threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < kIter; ++it) {
    double d;
    asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(x));
    asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(x) : "d"(d));
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename F>
static double time_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, nsm = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  void *buf;
  cudaMalloc(&buf, 1 << 20);
  long long *cyc;
  cudaMalloc(&cyc, 64);
  const int blocks = nsm * 8, threads = 256;
  const double ops = (double)blocks * threads * kIlp * kIter;  // per kernel: operations (lanes)
  const double t_dfma = time_ms([&] { k_dfma<<<blocks, threads>>>((double *)buf, 0.999, 1e-3); });
  const double t_ffma = time_ms([&] { k_ffma<<<blocks, threads>>>((float *)buf, 0.999f, 1e-3f); });
  const double t_ex2 = time_ms([&] { k_ex2<<<blocks, threads>>>((float *)buf); });
  const double t_f2f = time_ms([&] { k_f2f<<<blocks, threads>>>((float *)buf); });
  long long c_dfma = 0, c_f2f = 0;
  k_lat_dfma<<<1, 32>>>((double *)buf, cyc, 0.999, 1e-3);
  cudaMemcpy(&c_dfma, cyc, 8, cudaMemcpyDeviceToHost);
  k_lat_f2f<<<1, 32>>>((float *)buf, cyc);
  cudaMemcpy(&c_f2f, cyc, 8, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaDeviceSynchronize();
  const double sec = 1e-3;
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f,\n", nsm, clk_khz / 1e3);
  printf(" \"fp64_fma_tflops\": %.2f, \"fp64_fma_per_clk_per_sm_at_attr_clock\": %.1f,\n",
         2 * ops / (t_dfma * sec) / 1e12, ops / (t_dfma * sec) / nsm / (clk_khz * 1e3));
  printf(" \"fp32_fma_tflops\": %.2f, \"fp32_fma_per_clk_per_sm_at_attr_clock\": %.1f,\n",
         2 * ops / (t_ffma * sec) / 1e12, ops / (t_ffma * sec) / nsm / (clk_khz * 1e3));
  printf(" \"mufu_ex2_gops\": %.1f, \"mufu_ex2_per_clk_per_sm_at_attr_clock\": %.1f,\n",
         ops / (t_ex2 * sec) / 1e9, ops / (t_ex2 * sec) / nsm / (clk_khz * 1e3));
  printf(" \"f2f_f32_f64_pair_gops\": %.1f, \"f2f_conversions_per_clk_per_sm_at_attr_clock\": %.1f,\n",
         ops / (t_f2f * sec) / 1e9, 2 * ops / (t_f2f * sec) / nsm / (clk_khz * 1e3));
  printf(" \"dfma_dependent_latency_clk\": %.2f, \"f2f_pair_dependent_latency_clk\": %.2f,\n",
         (double)c_dfma / kIter, (double)c_f2f / kIter);
  printf(" \"ms\": {\"dfma\": %.4f, \"ffma\": %.4f, \"ex2\": %.4f, \"f2f\": %.4f}, \"status\": \"%s\"}\n", t_dfma,
         t_ffma, t_ex2, t_f2f, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
