// probes.cu -- microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry (MUFU ex2, DFMA).
#include "../../include/uot_b200_bench.h"
#include "common.cuh"

namespace uot {

__global__ void __launch_bounds__(256) probe_ex2(int iters, float seed, float* out) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed * (threadIdx.x + k) * 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[k]));
      v[k] = y * -0.5f;  // keep the argument bounded; FMUL rides the FMA pipe
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 12345.f) out[0] = s;
}

__global__ void __launch_bounds__(256) probe_dfma(int iters, double seed, double* out) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed + threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fma(v[k], 0.999999, 1e-9);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 12345.0) out[0] = s;
}

template <class K>
static int time_kernel(cudaStream_t st, K launch, double work, double* rate) {
  cudaEvent_t e0, e1;
  UOT_CUDA_TRY(cudaEventCreate(&e0));
  UOT_CUDA_TRY(cudaEventCreate(&e1));
  launch();  // warm-up
  UOT_CUDA_TRY(cudaEventRecord(e0, st));
  for (int r = 0; r < 5; ++r) launch();
  UOT_CUDA_TRY(cudaEventRecord(e1, st));
  UOT_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  UOT_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  UOT_CHECK_LAUNCH();
  *rate = work * 5.0 / (ms * 1e-3);
  return UOT_OK;
}

}  // namespace uot

extern "C" int uot_probe_mufu_ex2(void* stream, double* ex2_per_s) {
  using namespace uot;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  UOT_CUDA_TRY(cudaMalloc(&out, 64));
  const int blocks = sms * 8, iters = 4096;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = time_kernel(
      st, [&] { probe_ex2<<<blocks, 256, 0, st>>>(iters, 0.37f, out); },
      (double)blocks * 256 * iters * 8, ex2_per_s);
  cudaFree(out);
  return rc;
}

extern "C" int uot_probe_dfma(void* stream, double* dfma_per_s) {
  using namespace uot;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  UOT_CUDA_TRY(cudaMalloc(&out, 64));
  const int blocks = sms * 8, iters = 4096;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = time_kernel(
      st, [&] { probe_dfma<<<blocks, 256, 0, st>>>(iters, 0.5, out); },
      (double)blocks * 256 * iters * 8, dfma_per_s);
  cudaFree(out);
  return rc;
}
