// common.cuh -- shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "../../include/uot_b200.h"

namespace uot {

// Status codes of the C-ABI (include/uot_b200.h); the Python shim maps them onto
// the reference's exception classes (src/exceptions.py:4-25).
// (UOT_OK itself is the global enumerator from uot_b200.h.)
enum Status : int {
  UOT_MASS_BALANCE = 1,        // MassBalanceError
  UOT_UNSUPPORTED_ENTROPY = 2, // UnsupportedEntropyError
  UOT_INVALID = 3,             // ValueError (shape / finiteness / arguments)
  UOT_CUDA = 4,                // CUDA runtime failure
  UOT_NCCL = 5,                // NCCL failure
  UOT_INFEASIBLE = 6,          // InfeasibleDualError
};

void set_error(const char* fmt, ...);
const char* get_error();

#define UOT_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::uot::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                       __FILE__, __LINE__);                                         \
      return ::uot::UOT_CUDA;                                                       \
    }                                                                               \
  } while (0)

#define UOT_CHECK_LAUNCH()                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      ::uot::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                       __FILE__, __LINE__);                                         \
      return ::uot::UOT_CUDA;                                                       \
    }                                                                               \
  } while (0)

#define UOT_TRY(expr)              \
  do {                             \
    int _s = (expr);               \
    if (_s != UOT_OK) return _s; \
  } while (0)

constexpr double LN2 = 0.69314718055994530942;
constexpr double LOG2E = 1.44269504088896340736;

// ---------------------------------------------------------------------------
// Plan-support hash (trace mode, parity tests only).  A plan entry with index
// tuple (i_0 .. i_{K-1}) hashes to mix64(sum_q mix64(((q+1) << 40) | i_q));
// the plan hashes to the wrapping sum over its positive-mass entries, so the
// value is independent of the order in which threads find the entries and
// equal plans give equal hashes (tests/golden/make_golden.py: plan_hash).
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned long long coord_key(int q, int i) {
  return mix64(((unsigned long long)(q + 1) << 40) | (unsigned long long)(unsigned)i);
}
__host__ __device__ __forceinline__ unsigned long long pair_hash(int i, int j) {
  return mix64(coord_key(0, i) + coord_key(1, j));
}

// ---------------------------------------------------------------------------
// Warp / block reductions.

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Combine two (max, sum) log-sum-exp partials in the natural domain.  A pair
// with sum == 0 is empty (max is ignored).
struct LsePair {
  double m, s;
};

__device__ __forceinline__ LsePair lse_merge(LsePair a, LsePair b) {
  if (!(a.s > 0.0)) return b;
  if (!(b.s > 0.0)) return a;
  if (a.m >= b.m) return {a.m, a.s + b.s * exp(b.m - a.m)};
  return {b.m, b.s + a.s * exp(a.m - b.m)};
}

__device__ __forceinline__ LsePair warp_lse(LsePair p) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    LsePair q{__shfl_xor_sync(0xffffffffu, p.m, o), __shfl_xor_sync(0xffffffffu, p.s, o)};
    p = lse_merge(p, q);
  }
  return p;
}

// Block-wide reductions (blockDim.x multiple of 32, <= 1024).  `scratch`
// needs 32 entries.  All threads get the result.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* scratch, Op op, T ident) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = (threadIdx.x < nw) ? scratch[threadIdx.x] : ident;
  if (warp == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) scratch[0] = v;
  }
  __syncthreads();
  v = scratch[0];
  __syncthreads();
  return v;
}

__device__ __forceinline__ LsePair block_lse(LsePair p, double* sm, double* ss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  p = warp_lse(p);
  __syncthreads();
  if (lane == 0) {
    sm[warp] = p.m;
    ss[warp] = p.s;
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (warp == 0) {
    LsePair q = (lane < nw) ? LsePair{sm[lane], ss[lane]} : LsePair{-CUDART_INF, 0.0};
    q = warp_lse(q);
    if (lane == 0) {
      sm[0] = q.m;
      ss[0] = q.s;
    }
  }
  __syncthreads();
  LsePair r{sm[0], ss[0]};
  __syncthreads();
  return r;
}

struct MaxOp {
  template <typename T>
  __device__ T operator()(T a, T b) const { return fmax(a, b); }
};
struct MinOp {
  template <typename T>
  __device__ T operator()(T a, T b) const { return fmin(a, b); }
};
struct SumOp {
  template <typename T>
  __device__ T operator()(T a, T b) const { return a + b; }
};

// Block log-sum-exp of (m, s) pairs as max then rescaled sum: one exp per
// thread and two plain reductions (block_lse merges pairwise, one exp per
// butterfly step).  Pairs with s <= 0 are empty; an empty block gives
// (-inf, 0).  `sx` needs 32 doubles.
__device__ __forceinline__ LsePair block_lse_ms(LsePair p, double* sx) {
  const bool live = p.s > 0.0;
  const double m = block_reduce(live ? p.m : -CUDART_INF, sx, MaxOp(), -CUDART_INF);
  const double s = block_reduce(live ? p.s * exp(p.m - m) : 0.0, sx, SumOp(), 0.0);
  return LsePair{m, s};
}

// "Last block done" pattern: every block publishes its partial then calls
// this; exactly one block (the last to arrive) gets true and must reset the
// counter.  Requires a __threadfence() by the publishing thread first.
__device__ __forceinline__ bool last_block_arrive(unsigned int* counter, unsigned int nblocks,
                                                  int* flag_smem) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    *flag_smem = (prev == nblocks - 1) ? 1 : 0;
  }
  __syncthreads();
  bool last = *flag_smem != 0;
  if (last) __threadfence();
  return last;
}

inline unsigned int ceil_div(long a, long b) { return (unsigned int)((a + b - 1) / b); }

}  // namespace uot
