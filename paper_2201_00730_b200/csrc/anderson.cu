// anderson.cu -- Anderson extrapolation of the Sinkhorn fixed-point map on
// the device (reference src/sinkhorn.py:197-243 and
// the Anderson branch of run(), :281-292).
//
// State per problem (workspace, fp64): a ring of `depth` slots holding the
// window's map values T(z) and residuals T(z) - z (length len = n + m, the
// concatenated (f, g)), the Gram matrix of the residuals indexed by slot,
// and the window metadata (count, oldest slot, last residual sup norm).
// One push + extrapolate is two kernels:
//   and_push  -- writes the new slot, its sup norm, <r, r> and <r, r_s> for
//                every surviving slot (block partials, fixed-order final
//                reduction by the last block); the last block then applies
//                the reference's restart / eviction rule (:225-233), updates
//                the Gram row, solves (U'U + reg I) c = 1 by Gaussian
//                elimination with partial pivoting in chronological order
//                and normalises c (anderson_weights, :197-212);
//   and_mix   -- z' = sum_k c_k T(z)_k (or T(z) itself for a one-entry
//                window, :240-241) and delta_f = max |z'_f - z_f| (:294).
// A singular system sets status 1 (the reference raises LinAlgError).
#include <algorithm>
#include <cstdio>

#include "common.cuh"

namespace uot {
namespace {

constexpr int AND_THREADS = 256;
constexpr int AND_MAX_DEPTH = 32;

struct AndMeta {
  int count, head;
  double last_size;
};

struct AndWs {
  double* maps;    // [B][depth][len]
  double* res;     // [B][depth][len]
  double* gram;    // [B][depth][depth], slot-indexed
  double* coef;    // [B][depth], slot-indexed
  double* part;    // [B][nblk][depth + 2]: max |r|, <r, r>, <r, r_s>
  double* part2;   // [B][nblk]: max |z'_f - z_f|
  AndMeta* meta;   // [B]
  unsigned int* counter;  // [B][2]
  int nblk;
};

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

int and_nblk(int batch, long len) {
  long nb = (len + AND_THREADS * 8 - 1) / (AND_THREADS * 8);
  const long target = std::max(1L, 4L * 148 / std::max(batch, 1));
  nb = std::max(1L, std::min(nb, target));
  return (int)std::min(nb, 1024L);
}

size_t and_layout(int batch, long len, int depth, AndWs* w, char* base) {
  const int nblk = and_nblk(batch, len);
  size_t sz[8];
  sz[0] = sizeof(double) * (size_t)batch * depth * len;
  sz[1] = sz[0];
  sz[2] = sizeof(double) * (size_t)batch * depth * depth;
  sz[3] = sizeof(double) * (size_t)batch * depth;
  sz[4] = sizeof(double) * (size_t)batch * nblk * (depth + 2);
  sz[5] = sizeof(double) * (size_t)batch * nblk;
  sz[6] = sizeof(AndMeta) * (size_t)batch;
  sz[7] = sizeof(unsigned int) * 2 * (size_t)batch;
  size_t off[8], o = 0;
  for (int k = 0; k < 8; ++k) {
    off[k] = o;
    o += align256(sz[k]);
  }
  if (w != nullptr) {
    w->maps = (double*)(base + off[0]);
    w->res = (double*)(base + off[1]);
    w->gram = (double*)(base + off[2]);
    w->coef = (double*)(base + off[3]);
    w->part = (double*)(base + off[4]);
    w->part2 = (double*)(base + off[5]);
    w->meta = (AndMeta*)(base + off[6]);
    w->counter = (unsigned int*)(base + off[7]);
    w->nblk = nblk;
  }
  return o;
}

__global__ void and_reset(int batch, AndMeta* meta, unsigned int* counter) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) {
    meta[b] = AndMeta{0, 0, 0.0};
    counter[2 * b] = 0u;
    counter[2 * b + 1] = 0u;
  }
}

// Solve A x = 1 (k x k, row-major in `a`, overwritten) by Gaussian
// elimination with partial pivoting; false on an exactly zero pivot.
__device__ bool solve_ones(double* a, double* x, int k) {
  for (int i = 0; i < k; ++i) x[i] = 1.0;
  for (int c = 0; c < k; ++c) {
    int piv = c;
    double best = fabs(a[c * k + c]);
    for (int r = c + 1; r < k; ++r) {
      const double v = fabs(a[r * k + c]);
      if (v > best) {
        best = v;
        piv = r;
      }
    }
    if (a[piv * k + c] == 0.0) return false;
    if (piv != c) {
      for (int j = 0; j < k; ++j) {
        const double t = a[c * k + j];
        a[c * k + j] = a[piv * k + j];
        a[piv * k + j] = t;
      }
      const double t = x[c];
      x[c] = x[piv];
      x[piv] = t;
    }
    const double inv = a[c * k + c];
    for (int r = c + 1; r < k; ++r) {
      const double fac = a[r * k + c] / inv;
      for (int j = c; j < k; ++j) a[r * k + j] -= fac * a[c * k + j];
      x[r] -= fac * x[c];
    }
  }
  for (int r = k - 1; r >= 0; --r) {
    double s = 0.0;
    for (int j = r + 1; j < k; ++j) s += a[r * k + j] * x[j];
    x[r] = (x[r] - s) / a[r * k + r];
  }
  return true;
}

// Chronological window -> normalised weights (anderson_weights :197-212) from
// the slot-indexed Gram; single thread.  Returns 0 or 1 (LinAlgError).
__device__ int window_weights(const double* gram, int depth, int head, int count, double reg,
                              double* coef_slot) {
  double a[AND_MAX_DEPTH * AND_MAX_DEPTH];
  double x[AND_MAX_DEPTH];
  for (int i = 0; i < count; ++i) {
    const int si = (head + i) % depth;
    for (int j = 0; j < count; ++j) {
      const int sj = (head + j) % depth;
      a[i * count + j] = gram[si * depth + sj] + (i == j ? reg : 0.0);
    }
  }
  if (!solve_ones(a, x, count)) return 1;
  double den = 0.0;
  for (int i = 0; i < count; ++i) den += x[i];
  if (!isfinite(den) || den == 0.0) return 1;
  for (int i = 0; i < count; ++i) coef_slot[(head + i) % depth] = x[i] / den;
  return 0;
}

__global__ void __launch_bounds__(AND_THREADS)
and_push(long len, int depth, double reg, const double* __restrict__ z,
         const double* __restrict__ tz, AndWs w, int* __restrict__ status) {
  __shared__ double scratch[32];
  __shared__ int flag;
  const int b = blockIdx.y;
  const AndMeta mt = w.meta[b];
  const int slot_new = mt.count < depth ? (mt.head + mt.count) % depth : mt.head;
  const double* zb = z + (size_t)b * len;
  const double* tzb = tz + (size_t)b * len;
  double* resb = w.res + (size_t)b * depth * len;
  double* mapb = w.maps + (size_t)b * depth * len;
  const long per = (len + gridDim.x - 1) / gridDim.x;
  const long lo = (long)blockIdx.x * per;
  const long hi = std::min(len, lo + per);
  double mx = 0.0, rr = 0.0;
  for (long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double t = tzb[i];
    const double r = t - zb[i];
    resb[(size_t)slot_new * len + i] = r;
    mapb[(size_t)slot_new * len + i] = t;
    mx = fmax(mx, fabs(r));
    rr = fma(r, r, rr);
  }
  double* pb = w.part + ((size_t)b * w.nblk + blockIdx.x) * (depth + 2);
  mx = block_reduce(mx, scratch, MaxOp(), 0.0);
  rr = block_reduce(rr, scratch, SumOp(), 0.0);
  if (threadIdx.x == 0) {
    pb[0] = mx;
    pb[1] = rr;
  }
  // <r, r_s> for the surviving slots (the oldest is evicted when full)
  const int first = mt.count < depth ? 0 : 1;
  for (int j = first; j < mt.count; ++j) {
    const int s = (mt.head + j) % depth;
    const double* rs = resb + (size_t)s * len;
    double dot = 0.0;
    for (long i = lo + threadIdx.x; i < hi; i += blockDim.x) dot = fma(tzb[i] - zb[i], rs[i], dot);
    dot = block_reduce(dot, scratch, SumOp(), 0.0);
    if (threadIdx.x == 0) pb[2 + s] = dot;
  }
  if (!last_block_arrive(&w.counter[2 * b], gridDim.x, &flag)) return;
  // fixed-order reduction of the block partials
  __shared__ double tot[AND_MAX_DEPTH + 2];
  const double* p0 = w.part + (size_t)b * w.nblk * (depth + 2);
  for (int q = threadIdx.x; q < depth + 2; q += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) {
      const double v = p0[(size_t)k * (depth + 2) + q];
      acc = q == 0 ? fmax(acc, v) : acc + v;
    }
    tot[q] = acc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  w.counter[2 * b] = 0u;
  double* gb = w.gram + (size_t)b * depth * depth;
  const double size = tot[0];
  AndMeta nm = mt;
  if (mt.count > 0 && size > mt.last_size) {  // restart (:227-229)
    nm.head = slot_new;
    nm.count = 1;
  } else {
    for (int j = first; j < mt.count; ++j) {
      const int s = (mt.head + j) % depth;
      gb[slot_new * depth + s] = tot[2 + s];
      gb[s * depth + slot_new] = tot[2 + s];
    }
    if (mt.count < depth) {
      nm.count = mt.count + 1;
    } else {
      nm.head = (mt.head + 1) % depth;  // pop the oldest (:232-233)
    }
  }
  gb[slot_new * depth + slot_new] = tot[1];
  nm.last_size = size;
  w.meta[b] = nm;
  double* cb = w.coef + (size_t)b * depth;
  int st = 0;
  if (nm.count == 1) {
    cb[slot_new] = 1.0;
  } else {
    st = window_weights(gb, depth, nm.head, nm.count, reg, cb);
  }
  status[b] = st;
}

__global__ void __launch_bounds__(AND_THREADS)
and_mix(long len, long nf, int depth, const double* __restrict__ z, const double* __restrict__ tz,
        double* znew, AndWs w, const int* __restrict__ status, double* __restrict__ delta) {
  __shared__ double scratch[32];
  __shared__ int flag;
  const int b = blockIdx.y;
  const AndMeta mt = w.meta[b];
  const double* cb = w.coef + (size_t)b * depth;
  const double* mapb = w.maps + (size_t)b * depth * len;
  const double* zb = z + (size_t)b * len;
  const double* tzb = tz + (size_t)b * len;
  double* ob = znew + (size_t)b * len;
  const bool plain = mt.count == 1 || status[b] != 0;
  const long per = (len + gridDim.x - 1) / gridDim.x;
  const long lo = (long)blockIdx.x * per;
  const long hi = std::min(len, lo + per);
  double dmax = 0.0;
  for (long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double v;
    if (plain) {
      v = tzb[i];
    } else {
      v = 0.0;
      for (int j = 0; j < mt.count; ++j) {
        const int s = (mt.head + j) % depth;
        v = fma(cb[s], mapb[(size_t)s * len + i], v);
      }
    }
    if (i < nf) dmax = fmax(dmax, fabs(v - zb[i]));
    ob[i] = v;
  }
  dmax = block_reduce(dmax, scratch, MaxOp(), 0.0);
  if (threadIdx.x == 0) w.part2[(size_t)b * w.nblk + blockIdx.x] = dmax;
  if (!last_block_arrive(&w.counter[2 * b + 1], gridDim.x, &flag)) return;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) m = fmax(m, w.part2[(size_t)b * w.nblk + k]);
    delta[b] = m;
    w.counter[2 * b + 1] = 0u;
  }
}

// anderson_weights on a given window U [rows][k] (row-major, as numpy):
// one CTA, Gram by block reductions, then the pivoted solve.
__global__ void __launch_bounds__(AND_THREADS)
and_weights(int rows, int k, const double* __restrict__ U, double reg, double* c, int* status) {
  __shared__ double scratch[32];
  __shared__ double gram[AND_MAX_DEPTH * AND_MAX_DEPTH];
  for (int i = 0; i < k; ++i)
    for (int j = i; j < k; ++j) {
      double s = 0.0;
      for (int r = threadIdx.x; r < rows; r += blockDim.x)
        s = fma(U[(size_t)r * k + i], U[(size_t)r * k + j], s);
      s = block_reduce(s, scratch, SumOp(), 0.0);
      if (threadIdx.x == 0) {
        gram[i * k + j] = s;
        gram[j * k + i] = s;
      }
    }
  __syncthreads();
  if (threadIdx.x == 0) *status = window_weights(gram, k, 0, k, reg, c);
}

int check_dims(int batch, long len, int depth) {
  if (batch < 1 || len < 1) {
    set_error("anderson: batch and length must be positive");
    return UOT_INVALID;
  }
  if (depth < 1 || depth > AND_MAX_DEPTH) {
    set_error("anderson: depth must be in [1, %d] on the device", AND_MAX_DEPTH);
    return UOT_INVALID;
  }
  return UOT_OK;
}

}  // namespace
}  // namespace uot

using namespace uot;

extern "C" int uot_anderson_workspace_size(int32_t batch, int64_t len, int32_t depth,
                                           size_t* bytes) {
  UOT_TRY(check_dims(batch, len, depth));
  *bytes = and_layout(batch, len, depth, nullptr, nullptr);
  return UOT_OK;
}

extern "C" int uot_anderson_reset(int32_t batch, int64_t len, int32_t depth, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  UOT_TRY(check_dims(batch, len, depth));
  AndWs w;
  const size_t need = and_layout(batch, len, depth, &w, (char*)workspace);
  if (workspace_bytes < need) {
    set_error("anderson workspace too small: %zu < %zu", workspace_bytes, need);
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  and_reset<<<ceil_div(batch, 128), 128, 0, st>>>(batch, w.meta, w.counter);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_anderson_step(int32_t batch, int64_t len, int64_t nf, int32_t depth,
                                 double reg, const double* z, const double* tz, double* znew,
                                 double* delta_f, int32_t* status, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  UOT_TRY(check_dims(batch, len, depth));
  if (reg < 0 || nf < 0 || nf > len || z == nullptr || tz == nullptr || znew == nullptr ||
      delta_f == nullptr || status == nullptr) {
    set_error("anderson: invalid arguments");
    return UOT_INVALID;
  }
  AndWs w;
  const size_t need = and_layout(batch, len, depth, &w, (char*)workspace);
  if (workspace_bytes < need) {
    set_error("anderson workspace too small: %zu < %zu", workspace_bytes, need);
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid(w.nblk, batch);
  and_push<<<grid, AND_THREADS, 0, st>>>(len, depth, reg, z, tz, w, status);
  UOT_CHECK_LAUNCH();
  and_mix<<<grid, AND_THREADS, 0, st>>>(len, nf, depth, z, tz, znew, w, status, delta_f);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_anderson_weights(int32_t rows, int32_t k, const double* U, double reg,
                                    double* c, int32_t* status, void* stream) {
  if (rows < 1 || k < 1 || k > AND_MAX_DEPTH || reg < 0) {
    set_error("anderson_weights: need rows >= 1, 1 <= k <= %d, reg >= 0", AND_MAX_DEPTH);
    return UOT_INVALID;
  }
  and_weights<<<1, AND_THREADS, 0, (cudaStream_t)stream>>>(rows, k, U, reg, c, status);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
