// dense.cu -- the dense / plan-level helpers of the reference API on the
// device: the cost matrix (src/measures.py:125-145), its quadruple diameter
// (:168-184, for birkhoff_rate_bound, src/sinkhorn.py:338-346), the
// reweighted marginals of the FW oracle (src/duality.py:293-303) and the
// primal objective of a transport plan (src/duality.py:306-344).
#include <cstdint>

#include "common.cuh"

namespace uot {
namespace {

__device__ __forceinline__ double pow_cost(double xi, double yj, double p) {
  const double d = fabs(xi - yj);
  if (p == 1.0) return d;
  if (p == 2.0) return d * d;
  return pow(d, p);
}

__global__ void cost_matrix_kernel(int n, int m, const double* __restrict__ x,
                                   const double* __restrict__ y, double p, double* __restrict__ C) {
  const long total = (long)n * m;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / m), j = (int)(idx - (long)i * m);
    C[idx] = pow_cost(x[i], y[j], p);
  }
}

// Column k per block: for every l, the range over rows of C[:, k] - C[:, l];
// the maximum over (k, l) by an order-preserving integer max (ranges >= 0).
__global__ void __launch_bounds__(256) quad_diam_kernel(int n, int m, const double* __restrict__ C,
                                                        unsigned long long* __restrict__ out) {
  __shared__ double scratch[32];
  const int k = blockIdx.x;
  double best = 0.0;
  for (int l = threadIdx.x; l < m; l += blockDim.x) {
    double mx = -CUDART_INF, mn = CUDART_INF;
    for (int j = 0; j < n; ++j) {
      const double dv = C[(long)j * m + k] - C[(long)j * m + l];
      mx = fmax(mx, dv);
      mn = fmin(mn, dv);
    }
    best = fmax(best, mx - mn);
  }
  best = block_reduce(best, scratch, MaxOp(), 0.0);
  if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

// KL marginals reweighted at the translation lam: a exp((-f - lam)/rho1),
// b exp((-g + lam)/rho2) (conj_grad of KL, src/entropies.py).
__global__ void updated_marginals_kernel(int n, int m, const double* __restrict__ a,
                                         const double* __restrict__ b,
                                         const double* __restrict__ f,
                                         const double* __restrict__ g, double rho1, double rho2,
                                         double lam, double* __restrict__ ta,
                                         double* __restrict__ tb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ta[i] = a[i] * exp((-f[i] - lam) / rho1);
  if (i < m) tb[i] = b[i] * exp((-g[i] + lam) / rho2);
}

// One side's divergence terms for index range [lo, hi) with marginals from
// the plan entries (every entry scanned per index: deterministic, general
// plans).  KL: sum_{w>0} [mu log(mu/w) - mu + w], singular mass -> inf;
// Berg: sum_{w>0} [mu - w - w log(mu/w)] + singular mass, inf at mu = 0 < w
// (src/entropies.py:132-137); Balanced: max |mu - w| (the caller applies the
// 1e-9 tolerance).
struct SideAcc {
  double terms, sing, maxdiff, maxw, inf;
};

__device__ SideAcc side_terms(int count, const double* w, int E, const int64_t* idx,
                              const double* mass, int ent) {
  const bool balanced = ent == UOT_ENT_BALANCED;
  SideAcc s{0.0, 0.0, 0.0, 0.0, 0.0};
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double mu = 0.0;
    for (int e = 0; e < E; ++e)
      if (idx[e] == i) mu += mass[e];
    const double wi = w[i];
    if (balanced) {
      s.maxdiff = fmax(s.maxdiff, fabs(mu - wi));
      s.maxw = fmax(s.maxw, fabs(wi));
    } else if (wi > 0.0 && ent == UOT_ENT_BERG) {
      if (mu == 0.0)
        s.inf = 1.0;
      else
        s.terms += mu - wi - wi * log(mu / wi);
    } else if (wi > 0.0) {
      s.terms += (mu > 0.0 ? mu * log(mu / wi) : 0.0) - mu + wi;
    } else {
      s.sing += mu;
    }
  }
  return s;
}

// out[0] = <plan, C> + eps KL(plan | a x b) + D1(plan_1 | a) + D2(plan_2 | b)
__global__ void __launch_bounds__(1024)
    eval_primal_kernel(int n, int m, const double* x, const double* y, double p, const double* C,
                       const double* a, const double* b, int E, const int64_t* ii,
                       const int64_t* jj, const double* mass, int ent1, int ent2, double rho1,
                       double rho2, double eps, double* out) {
  __shared__ double scratch[32];
  double cost = 0.0, klp = 0.0, qbad = 0.0, ma = 0.0, mb = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const long i = ii[e], j = jj[e];
    const double ms = mass[e];
    cost += ms * (C != nullptr ? C[i * m + j] : pow_cost(x[i], y[j], p));
    if (eps > 0.0 && ms > 0.0) {
      const double q = a[i] * b[j];
      if (q == 0.0)
        qbad = 1.0;
      else
        klp += ms * log(ms / q) - ms;
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) ma += a[i];
  for (int j = threadIdx.x; j < m; j += blockDim.x) mb += b[j];
  const SideAcc s1 = side_terms(n, a, E, ii, mass, ent1);
  const SideAcc s2 = side_terms(m, b, E, jj, mass, ent2);
  cost = block_reduce(cost, scratch, SumOp(), 0.0);
  klp = block_reduce(klp, scratch, SumOp(), 0.0);
  qbad = block_reduce(qbad, scratch, MaxOp(), 0.0);
  ma = block_reduce(ma, scratch, SumOp(), 0.0);
  mb = block_reduce(mb, scratch, SumOp(), 0.0);
  const double t1 = block_reduce(s1.terms, scratch, SumOp(), 0.0);
  const double g1 = block_reduce(s1.sing, scratch, SumOp(), 0.0);
  const double d1 = block_reduce(s1.maxdiff, scratch, MaxOp(), 0.0);
  const double w1 = block_reduce(s1.maxw, scratch, MaxOp(), 0.0);
  const double t2 = block_reduce(s2.terms, scratch, SumOp(), 0.0);
  const double g2 = block_reduce(s2.sing, scratch, SumOp(), 0.0);
  const double d2 = block_reduce(s2.maxdiff, scratch, MaxOp(), 0.0);
  const double w2 = block_reduce(s2.maxw, scratch, MaxOp(), 0.0);
  const double i1 = block_reduce(s1.inf, scratch, MaxOp(), 0.0);
  const double i2 = block_reduce(s2.inf, scratch, MaxOp(), 0.0);
  if (threadIdx.x != 0) return;
  auto div = [](int ent, double rho, double t, double sing, double md, double mw, double inf) {
    if (ent == UOT_ENT_BALANCED) return md <= 1e-9 * (1.0 + mw) ? 0.0 : CUDART_INF;  // :119-121
    if (ent == UOT_ENT_BERG) return inf > 0.0 ? CUDART_INF : rho * (t + sing);
    if (sing > 0.0) return CUDART_INF;
    return rho * t;
  };
  double total = cost + div(ent1, rho1, t1, g1, d1, w1, i1) + div(ent2, rho2, t2, g2, d2, w2, i2);
  if (eps > 0.0) total += qbad > 0.0 ? CUDART_INF : eps * (klp + ma * mb);
  out[0] = total;
}

// Large entry lists (dense plans): eval_primal_kernel scans every entry once
// per index -- O((n + m) E) on one CTA, 1 s for a dense 2048 x 2048 plan.
// Here the entries are walked once by a whole grid: block partials of the cost
// and KL sums at part[4 * block ..], the marginals by fp64 atomics into mu1 /
// mu2 (zeroed by the caller; the summation order, hence the last bits, vary
// from run to run), and eval_primal_fold finishes on one CTA.
__global__ void __launch_bounds__(256)
    eval_primal_entries(int m, const double* x, const double* y, double p, const double* C,
                        const double* a, const double* b, int E, const int64_t* ii,
                        const int64_t* jj, const double* mass, double eps, double* mu1, double* mu2,
                        double* part) {
  __shared__ double scratch[32];
  double cost = 0.0, klp = 0.0, qbad = 0.0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < E; e += (long)gridDim.x * blockDim.x) {
    const long i = ii[e], j = jj[e];
    const double ms = mass[e];
    cost += ms * (C != nullptr ? C[i * m + j] : pow_cost(x[i], y[j], p));
    if (eps > 0.0 && ms > 0.0) {
      const double q = a[i] * b[j];
      if (q == 0.0)
        qbad = 1.0;
      else
        klp += ms * log(ms / q) - ms;
    }
    if (ms != 0.0) {
      atomicAdd(mu1 + i, ms);
      atomicAdd(mu2 + j, ms);
    }
  }
  cost = block_reduce(cost, scratch, SumOp(), 0.0);
  klp = block_reduce(klp, scratch, SumOp(), 0.0);
  qbad = block_reduce(qbad, scratch, MaxOp(), 0.0);
  if (threadIdx.x == 0) {
    part[4 * blockIdx.x + 0] = cost;
    part[4 * blockIdx.x + 1] = klp;
    part[4 * blockIdx.x + 2] = qbad;
  }
}

__device__ SideAcc side_terms_mu(int count, const double* w, const double* mus, int ent) {
  const bool balanced = ent == UOT_ENT_BALANCED;
  SideAcc s{0.0, 0.0, 0.0, 0.0, 0.0};
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const double mu = mus[i], wi = w[i];
    if (balanced) {
      s.maxdiff = fmax(s.maxdiff, fabs(mu - wi));
      s.maxw = fmax(s.maxw, fabs(wi));
    } else if (wi > 0.0 && ent == UOT_ENT_BERG) {
      if (mu == 0.0)
        s.inf = 1.0;
      else
        s.terms += mu - wi - wi * log(mu / wi);
    } else if (wi > 0.0) {
      s.terms += (mu > 0.0 ? mu * log(mu / wi) : 0.0) - mu + wi;
    } else {
      s.sing += mu;
    }
  }
  return s;
}

__global__ void __launch_bounds__(1024)
    eval_primal_fold(int n, int m, const double* a, const double* b, const double* mu1,
                     const double* mu2, int nblk, const double* part, int ent1, int ent2,
                     double rho1, double rho2, double eps, double* out) {
  __shared__ double scratch[32];
  double cost = 0.0, klp = 0.0, qbad = 0.0, ma = 0.0, mb = 0.0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x) {
    cost += part[4 * k + 0];
    klp += part[4 * k + 1];
    qbad = fmax(qbad, part[4 * k + 2]);
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) ma += a[i];
  for (int j = threadIdx.x; j < m; j += blockDim.x) mb += b[j];
  const SideAcc s1 = side_terms_mu(n, a, mu1, ent1);
  const SideAcc s2 = side_terms_mu(m, b, mu2, ent2);
  cost = block_reduce(cost, scratch, SumOp(), 0.0);
  klp = block_reduce(klp, scratch, SumOp(), 0.0);
  qbad = block_reduce(qbad, scratch, MaxOp(), 0.0);
  ma = block_reduce(ma, scratch, SumOp(), 0.0);
  mb = block_reduce(mb, scratch, SumOp(), 0.0);
  const double t1 = block_reduce(s1.terms, scratch, SumOp(), 0.0);
  const double g1 = block_reduce(s1.sing, scratch, SumOp(), 0.0);
  const double d1 = block_reduce(s1.maxdiff, scratch, MaxOp(), 0.0);
  const double w1 = block_reduce(s1.maxw, scratch, MaxOp(), 0.0);
  const double t2 = block_reduce(s2.terms, scratch, SumOp(), 0.0);
  const double g2 = block_reduce(s2.sing, scratch, SumOp(), 0.0);
  const double d2 = block_reduce(s2.maxdiff, scratch, MaxOp(), 0.0);
  const double w2 = block_reduce(s2.maxw, scratch, MaxOp(), 0.0);
  const double i1 = block_reduce(s1.inf, scratch, MaxOp(), 0.0);
  const double i2 = block_reduce(s2.inf, scratch, MaxOp(), 0.0);
  if (threadIdx.x != 0) return;
  auto div = [](int ent, double rho, double t, double sing, double md, double mw, double inf) {
    if (ent == UOT_ENT_BALANCED) return md <= 1e-9 * (1.0 + mw) ? 0.0 : CUDART_INF;  // :119-121
    if (ent == UOT_ENT_BERG) return inf > 0.0 ? CUDART_INF : rho * (t + sing);
    if (sing > 0.0) return CUDART_INF;
    return rho * t;
  };
  double total = cost + div(ent1, rho1, t1, g1, d1, w1, i1) + div(ent2, rho2, t2, g2, d2, w2, i2);
  if (eps > 0.0) total += qbad > 0.0 ? CUDART_INF : eps * (klp + ma * mb);
  out[0] = total;
}

}  // namespace
}  // namespace uot

using namespace uot;

extern "C" int uot_cost_matrix(int32_t n, int32_t m, const double* x, const double* y, double p,
                               double* C, void* stream) {
  if (n < 1 || m < 1 || x == nullptr || y == nullptr || C == nullptr || !(p > 0.0)) {
    set_error("cost_matrix: invalid arguments");
    return UOT_INVALID;
  }
  const unsigned blocks = ceil_div((long)n * m, 256);
  cost_matrix_kernel<<<blocks > 4096u ? 4096u : blocks, 256, 0, (cudaStream_t)stream>>>(n, m, x, y,
                                                                                       p, C);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_cost_quadruple_diameter(int32_t n, int32_t m, const double* C, double* out,
                                           void* stream) {
  if (n < 1 || m < 1 || C == nullptr || out == nullptr) {
    set_error("cost_quadruple_diameter: invalid arguments");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  UOT_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));  // +0.0
  quad_diam_kernel<<<m, 256, 0, st>>>(n, m, C, reinterpret_cast<unsigned long long*>(out));
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_updated_marginals(int32_t n, int32_t m, const double* a, const double* b,
                                     const double* f, const double* g, double rho1, double rho2,
                                     double lam, double* ta, double* tb, void* stream) {
  if (n < 1 || m < 1 || !(rho1 > 0.0) || !(rho2 > 0.0)) {
    set_error("updated_marginals: invalid arguments");
    return UOT_INVALID;
  }
  const int nm = n > m ? n : m;
  updated_marginals_kernel<<<ceil_div(nm, 256), 256, 0, (cudaStream_t)stream>>>(
      n, m, a, b, f, g, rho1, rho2, lam, ta, tb);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_eval_primal(int32_t n, int32_t m, const double* x, const double* y, double p,
                               const double* C, const double* a, const double* b, int32_t E,
                               const int64_t* ii, const int64_t* jj, const double* mass,
                               int32_t ent1, int32_t ent2, double rho1, double rho2, double eps,
                               double* out, void* stream) {
  if (n < 1 || m < 1 || E < 0 || out == nullptr || (C == nullptr && (x == nullptr || y == nullptr))) {
    set_error("eval_primal: invalid arguments");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // small entry lists: the deterministic one-CTA kernel (the parity fixtures);
  // large ones (dense plans): one grid pass over the entries
  if ((long)E * ((long)n + m) <= (1L << 26)) {
    eval_primal_kernel<<<1, 1024, 0, st>>>(n, m, x, y, p, C, a, b, E, ii, jj, mass, ent1, ent2, rho1,
                                           rho2, eps, out);
    UOT_CHECK_LAUNCH();
    return UOT_OK;
  }
  const int nblk = (int)std::min<long>(1184, ((long)E + 255) / 256);
  const size_t bytes = sizeof(double) * ((size_t)n + m + 4 * (size_t)nblk);
  double* scr = nullptr;
  UOT_CUDA_TRY(cudaMallocAsync(&scr, bytes, st));
  UOT_CUDA_TRY(cudaMemsetAsync(scr, 0, bytes, st));
  eval_primal_entries<<<nblk, 256, 0, st>>>(m, x, y, p, C, a, b, E, ii, jj, mass, eps, scr, scr + n,
                                            scr + n + m);
  eval_primal_fold<<<1, 1024, 0, st>>>(n, m, a, b, scr, scr + n, nblk, scr + n + m, ent1, ent2, rho1,
                                       rho2, eps, out);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(scr, st);
  if (le != cudaSuccess) {
    set_error("eval_primal: launch failed: %s", cudaGetErrorString(le));
    return UOT_INVALID;
  }
  return UOT_OK;
}
