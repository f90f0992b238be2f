// tc_selftest.cu -- one-tile check of the tcgen05 path used by the d >= 32
// Sinkhorn kernel: D[128x128] = A[128xK] * B[128xK]^T with A written to TMEM
// (tcgen05.st), B staged in shared memory in the canonical K-major layout,
// kind::tf32 MMAs issued by one thread, D read back with tcgen05.ld.
// Exported as uot_tc_selftest (include/uot_b200_bench.h); tests compare it
// with an fp64 host product.
#include "../../include/uot_b200_bench.h"
#include "common.cuh"
#include "tcgen05.cuh"

namespace uot {

__global__ void __launch_bounds__(128) tc_selftest_kernel(const float* A, const float* B, int K,
                                                          float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  constexpr int N = 128, M = 128;
  const int t = threadIdx.x, warp = t >> 5;
  float* sB = reinterpret_cast<float*>(smem);
  const uint32_t LBO = (N / 8) * 128, SBO = 128;
  // B -> shared memory, canonical K-major no-swizzle layout
  for (int idx = t; idx < N * K; idx += blockDim.x) {
    const int n = idx / K, k = idx % K;
    const uint32_t off = (k / 4) * LBO + (n / 8) * SBO + (n % 8) * 16 + (k % 4) * 4;
    sB[off / 4] = B[idx];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tc::tmem_alloc(&tbase_s, 512);
  if (t == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tbase_s;
  // A -> TMEM: lane = row, column = K element
  const int row = t;
  for (int c = 0; c < K; c += 8) {
    uint32_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float_as_uint(A[row * K + c + e]);
    tc::tmem_st8(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
  }
  tc::wait_st();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t d_col = 256;
  if (t == 0) {
    const uint32_t idesc = tc::idesc_tf32(M, N);
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t bd = tc::sdesc(sB + (2 * s * LBO) / 4, LBO, SBO);
      tc::mma_tf32_ts(tbase + d_col, tbase + 8 * s, bd, idesc, s > 0 ? 1u : 0u);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + d_col + c, v);
    tc::wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) D[row * N + c + e] = __uint_as_float(v[e]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tbase, 512);
}

// Issue-rate probe: `reps` back-to-back 128 x N x 8 tf32 MMAs, timed with
// clock64 by the issuing thread; cycles summed over CTAs.  MODE 0: one
// accumulator, A from TMEM; 1: A from shared memory; 2: two interleaved
// accumulators; 3: four interleaved accumulators (N <= 64).
template <int MODE>
__global__ void __launch_bounds__(128) tc_rate_kernel(int reps, int N, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int t = threadIdx.x, warp = t >> 5;
  float* s = reinterpret_cast<float*>(smem);
  for (int i = t; i < 2 * 256 * 8; i += blockDim.x) s[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tc::tmem_alloc(&tbase_s, 512);
  if (t == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tbase_s;
  if (t == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, N);
    const uint64_t bd = tc::sdesc(s, (N / 8) * 128, 128);
    const uint64_t ad = tc::sdesc(s + 256 * 8, 16 * 128, 128);
    const long long c0 = clock64();
    if (MODE == 0) {
      tc::mma_tf32_ts(tbase + 256, tbase, bd, idesc, 0u);
      for (int r = 1; r < reps; ++r) tc::mma_tf32_ts(tbase + 256, tbase, bd, idesc, 1u);
    } else if (MODE == 1) {
      tc::mma_tf32_ss(tbase + 256, ad, bd, idesc, 0u);
      for (int r = 1; r < reps; ++r) tc::mma_tf32_ss(tbase + 256, ad, bd, idesc, 1u);
    } else if (MODE == 2) {
      for (int r = 0; r < reps; r += 2) {
        tc::mma_tf32_ts(tbase + 256, tbase, bd, idesc, 1u);
        tc::mma_tf32_ts(tbase + 384, tbase, bd, idesc, 1u);
      }
    } else {
      for (int r = 0; r < reps; r += 4) {
        tc::mma_tf32_ts(tbase + 256, tbase, bd, idesc, 1u);
        tc::mma_tf32_ts(tbase + 320, tbase, bd, idesc, 1u);
        tc::mma_tf32_ts(tbase + 384, tbase, bd, idesc, 1u);
        tc::mma_tf32_ts(tbase + 448, tbase, bd, idesc, 1u);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    atomicAdd(out, (unsigned long long)(clock64() - c0));
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tbase, 512);
}

// Pair check: D[256x128] = A[256xK] * B[128xK]^T on a cluster of two CTAs
// with tcgen05.mma.cta_group::2 -- CTA r holds A rows [128r, 128r+128) in
// its TMEM and B rows [64r, 64r+64) in its shared memory; the leader issues.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    tc_selftest2_kernel(const float* A, const float* B, int K, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  constexpr int N = 128, NH = 64;
  const int t = threadIdx.x, warp = t >> 5;
  const uint32_t rank = tc::cluster_rank();
  float* sB = reinterpret_cast<float*>(smem);
  const uint32_t LBO = (NH / 8) * 128, SBO = 128;
  for (int idx = t; idx < NH * K; idx += blockDim.x) {
    const int n = idx / K, k = idx % K;
    const uint32_t off = (k / 4) * LBO + (n / 8) * SBO + (n % 8) * 16 + (k % 4) * 4;
    sB[off / 4] = B[(rank * NH + n) * K + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tc::tmem_alloc2(&tbase_s, 512);
  if (t == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tbase_s;
  const int row = t;
  for (int c = 0; c < K; c += 8) {
    uint32_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float_as_uint(A[(rank * 128 + row) * K + c + e]);
    tc::tmem_st8(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
  }
  tc::wait_st();
  tc::fence_before();
  tc::cluster_sync_all();
  tc::fence_after();
  const uint32_t d_col = 256;
  if (rank == 0 && t == 0) {
    const uint32_t idesc = tc::idesc_tf32(256, N);
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t bd = tc::sdesc(sB + (2 * s * LBO) / 4, LBO, SBO);
      tc::mma2_tf32_ts(tbase + d_col, tbase + 8 * s, bd, idesc, s > 0 ? 1u : 0u);
    }
    tc::mma2_commit_mc(&bar, 3);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + d_col + c, v);
    tc::wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) D[(rank * 128 + row) * N + c + e] = __uint_as_float(v[e]);
  }
  tc::fence_before();
  tc::cluster_sync_all();
  if (warp == 0) tc::tmem_free2(tbase, 512);
}

}  // namespace uot

extern "C" int uot_tc_selftest2(const float* A, const float* B, int K, float* D, void* stream) {
  using namespace uot;
  if (K < 8 || K % 8 != 0 || K > 256) {
    set_error("uot_tc_selftest2: K must be a multiple of 8 in [8, 256]");
    return UOT_INVALID;
  }
  const size_t smem = (size_t)64 * K * 4;
  UOT_CUDA_TRY(cudaFuncSetAttribute(tc_selftest2_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tc_selftest2_kernel<<<2, 128, smem, (cudaStream_t)stream>>>(A, B, K, D);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_probe_tc_rate(int ctas, int reps, int n, int ss, unsigned long long* out_dev,
                                 void* stream) {
  using namespace uot;
  if (n < 8 || n > 256 || n % 8 != 0) {
    set_error("uot_probe_tc_rate: N in [8, 256], multiple of 8");
    return UOT_INVALID;
  }
  const size_t smem = 2 * 256 * 8 * 4;
  cudaStream_t st = (cudaStream_t)stream;
  switch (ss) {
    case 0: tc_rate_kernel<0><<<ctas, 128, smem, st>>>(reps, n, out_dev); break;
    case 1: tc_rate_kernel<1><<<ctas, 128, smem, st>>>(reps, n, out_dev); break;
    case 2: tc_rate_kernel<2><<<ctas, 128, smem, st>>>(reps, n, out_dev); break;
    default: tc_rate_kernel<3><<<ctas, 128, smem, st>>>(reps, n, out_dev); break;
  }
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_tc_selftest(const float* A, const float* B, int K, float* D, void* stream) {
  using namespace uot;
  if (K < 8 || K % 8 != 0 || K > 256) {
    set_error("uot_tc_selftest: K must be a multiple of 8 in [8, 256]");
    return UOT_INVALID;
  }
  const size_t smem = (size_t)128 * K * 4;
  UOT_CUDA_TRY(cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  tc_selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(A, B, K, D);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
