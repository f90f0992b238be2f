// fw1d_generic.cu -- the dual functionals and Frank-Wolfe at eps = 0 for
// strictly convex penalties other than KL/KL (Berg, mixed KL/Berg):
//   * the optimal translation by the reference's bracketed Newton on the
//     mass-balance equation (src/duality.py:182-247), with the updated
//     marginals (:293-303) and the invariant dual value _h0
//     (src/fw.py:106-115: <w, -phi*(-pot)> sums, src/duality.py:102-114)
//     -- uot_translation;
//   * Frank-Wolfe (src/fw.py:176-252) as three launches per iteration:
//     fwg_prep (translation, reweighted marginals, dual value, mass check,
//     err_f), the 1-D OT oracle kernel of fw1d_kernel.cuh on the reweighted
//     marginals, fwg_step (linear gap, primal of the oracle plan with the
//     Csiszar divergences of src/entropies.py:104-138, ternary line search
//     :118-148 whose every H0 evaluation solves its own translation, the
//     blend).  uot_fw1d_run routes here when a penalty is not KL.
// One CTA per problem; the per-problem vectors stay in global memory (L1/L2
// resident at these sizes).  KL/KL problems use the fused kernel instead.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "fw1d_kernel.cuh"

namespace uot {
namespace fwk {
int launch_fw_ot(const FwArgs& a, int batch, cudaStream_t st);  // fw1d.cu
size_t ot_scratch_bytes(int batch, int n, int m);               // fw1d.cu
}  // namespace fwk

namespace {
using fwk::FwArgs;

constexpr int GT = 256;
constexpr double NEWTON_TOL = 1e-11;  // duality.py:160
constexpr int NEWTON_ITERS = 100;
constexpr double LMO_MASS_TOL = 1e-9;  // fw.py:49

// conj_grad / conj_hess / -phi*(-pot) (src/entropies.py:141-184,
// src/duality.py:102-114) for KL, Berg and Balanced.
__device__ __forceinline__ double cgrad(int e, double rho, double x) {
  if (e == UOT_ENT_KL) return exp(x / rho);
  if (e == UOT_ENT_BERG) return rho / (rho - x);
  return 1.0;
}
__device__ __forceinline__ double chess(int e, double rho, double x) {
  if (e == UOT_ENT_KL) return exp(x / rho) / rho;
  if (e == UOT_ENT_BERG) return rho / ((rho - x) * (rho - x));
  return 0.0;
}
__device__ __forceinline__ double negconj(int e, double rho, double pot) {
  if (e == UOT_ENT_KL) return rho * (1.0 - exp(-pot / rho));
  if (e == UOT_ENT_BERG) return pot > -rho ? rho * log1p(pot / rho) : -CUDART_INF;
  return pot;
}

// Sum of K doubles over the block with one pair of barriers; scratch holds
// K * 8 doubles + K.  Every thread gets the sums.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[k * 8 + warp] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int w = 0; w < GT / 32; ++w) s += scratch[k * 8 + w];
    v[k] = s;
  }
  __syncthreads();
}

struct Sides {
  int n, m;
  const double* a;
  const double* b;
  int e1, e2;
  double r1, r2;
  double tol = NEWTON_TOL;     // lambda_star(tol, max_iters) (duality.py:160)
  int max_iters = NEWTON_ITERS;
};

// (1 - gamma) u + gamma v without FMA contraction (numpy's rounding, fw.py:140-144)
__device__ __forceinline__ double blend(double u, double v, double gm) {
  return __dadd_rn(__dmul_rn(1.0 - gm, u), __dmul_rn(gm, v));
}

// Optimal translation of (pf(i), pg(j)) by the bracketed Newton of
// src/duality.py:182-247 started at `init`.  err: 1 = empty domain, 2 = no
// bracket, 3 = no convergence (NewtonError).  Block-uniform result.
template <class PF, class PG>
__device__ double newton_lambda(const Sides& S, PF pf, PG pg, double init, double* scr, int* err) {
  double fmn = CUDART_INF, gmn = CUDART_INF;
  for (int i = threadIdx.x; i < S.n; i += GT) fmn = fmin(fmn, pf(i));
  for (int j = threadIdx.x; j < S.m; j += GT) gmn = fmin(gmn, pg(j));
  fmn = block_reduce(fmn, scr, MinOp(), CUDART_INF);
  gmn = block_reduce(gmn, scr, MinOp(), CUDART_INF);
  const double lo_dom = S.e1 == UOT_ENT_BERG ? -S.r1 - fmn : -CUDART_INF;
  const double hi_dom = S.e2 == UOT_ENT_BERG ? S.r2 + gmn : CUDART_INF;
  *err = 0;
  if (!(lo_dom < hi_dom)) {
    *err = 1;
    return CUDART_NAN;
  }
  auto clamp = [&](double x) {
    if (lo_dom > -CUDART_INF) x = fmax(x, lo_dom + 1e-12 * fmax(1.0, fabs(lo_dom)));
    if (hi_dom < CUDART_INF) x = fmin(x, hi_dom - 1e-12 * fmax(1.0, fabs(hi_dom)));
    return x;
  };
  auto eval = [&](double lam, double& res, double& slope) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < S.n; i += GT) {
      const double w = S.a[i];
      if (w > 0.0) {
        const double xv = -pf(i) - lam;
        v[0] += w * cgrad(S.e1, S.r1, xv);
        v[2] += w * chess(S.e1, S.r1, xv);
      }
    }
    for (int j = threadIdx.x; j < S.m; j += GT) {
      const double w = S.b[j];
      if (w > 0.0) {
        const double xv = -pg(j) + lam;
        v[1] += w * cgrad(S.e2, S.r2, xv);
        v[3] += w * chess(S.e2, S.r2, xv);
      }
    }
    block_sum<4>(v, scr);
    res = v[0] - v[1];
    slope = -v[2] - v[3];
  };
  double lam = clamp(init), r, ds;
  eval(lam, r, ds);
  if (fabs(r) < S.tol) return lam;
  double lo = lam, hi = lam, step = 1.0;
  bool ok = false;
  if (r > 0.0) {
    for (int it = 0; it < 200 && !ok; ++it) {
      hi = clamp(lam + step);
      double rh, dh;
      eval(hi, rh, dh);
      ok = rh <= 0.0;
      step *= 2.0;
    }
  } else {
    for (int it = 0; it < 200 && !ok; ++it) {
      lo = clamp(lam - step);
      double rl, dl;
      eval(lo, rl, dl);
      ok = rl >= 0.0;
      step *= 2.0;
    }
  }
  if (!ok) {
    *err = 2;
    return CUDART_NAN;
  }
  double x = 0.5 * (lo + hi);
  for (int it = 0; it < S.max_iters; ++it) {
    eval(x, r, ds);
    if (fabs(r) < S.tol) return x;
    if (r > 0.0)
      lo = x;
    else
      hi = x;
    const double nt = (ds < 0.0 && isfinite(ds)) ? x - r / ds : CUDART_NAN;
    x = (nt > lo && nt < hi) ? nt : 0.5 * (lo + hi);
  }
  *err = 3;
  return CUDART_NAN;
}

// <a, -phi1*(-(f + lam))> + <b, -phi2*(-(g - lam))> (fw.py:113-115)
template <class PF, class PG>
__device__ double h_value(const Sides& S, PF pf, PG pg, double lam, double* scr) {
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < S.n; i += GT)
    if (S.a[i] > 0.0) v[0] += S.a[i] * negconj(S.e1, S.r1, pf(i) + lam);
  for (int j = threadIdx.x; j < S.m; j += GT)
    if (S.b[j] > 0.0) v[0] += S.b[j] * negconj(S.e2, S.r2, pg(j) - lam);
  block_sum<1>(v, scr);
  return v[0];
}

// ---------------------------------------------------------------------------
// uot_translation: lam (solved or given), optional marginals and H value.

__global__ void __launch_bounds__(GT) translation_kernel(Sides S0, const double* f,
                                                         const double* g, int solve, double lam0,
                                                         double* lam_out, double* ta, double* tb,
                                                         double* h, int* status) {
  __shared__ double scr[40];
  const int bi = blockIdx.x;
  Sides S = S0;
  S.a += (long)bi * S.n;
  S.b += (long)bi * S.m;
  const double* fb = f + (long)bi * S.n;
  const double* gb = g + (long)bi * S.m;
  auto pf = [&](int i) { return fb[i]; };
  auto pg = [&](int j) { return gb[j]; };
  int err = 0;
  const double lam = solve ? newton_lambda(S, pf, pg, lam0, scr, &err) : lam0;
  if (threadIdx.x == 0) {
    if (status) status[bi] = err;
    if (lam_out) lam_out[bi] = lam;
  }
  if (err) return;
  if (ta)
    for (int i = threadIdx.x; i < S.n; i += GT)
      ta[(long)bi * S.n + i] = S.a[i] * cgrad(S.e1, S.r1, -fb[i] - lam);
  if (tb)
    for (int j = threadIdx.x; j < S.m; j += GT)
      tb[(long)bi * S.m + j] = S.b[j] * cgrad(S.e2, S.r2, -gb[j] + lam);
  if (h) {
    const double v = h_value(S, pf, pg, lam, scr);
    if (threadIdx.x == 0) h[bi] = v;
  }
}

// ---------------------------------------------------------------------------
// Frank-Wolfe iterations.

struct GenState {
  double* ta;    // [B][n] reweighted marginals (oracle input)
  double* tb;    // [B][m]
  double* af;    // [B][n] oracle atom
  double* ag;    // [B][m]
  int* pi;       // [B][n+m-1] oracle plan (scratch)
  int* pj;
  double* pm;
  int* pcount;   // [B]
  int* pstatus;  // [B]
  double* dual;  // [B] H0 of the current iterate
  int* done;     // [B]
};

struct GenArgs {
  FwArgs A;  // problem, outputs (f, g in/out; traces; last plan; summary; status)
  Sides S;
  GenState G;
};

__global__ void __launch_bounds__(GT) fwg_prep(GenArgs P, int t) {
  __shared__ double scr[40];
  const int bi = blockIdx.x;
  if (P.G.done[bi]) return;
  const FwArgs& A = P.A;
  Sides S = P.S;
  S.a += (long)bi * S.n;
  S.b += (long)bi * S.m;
  const double* f = A.f + (long)bi * S.n;
  const double* g = A.g + (long)bi * S.m;
  auto pf = [&](int i) { return f[i]; };
  auto pg = [&](int j) { return g[j]; };
  int err = 0;
  const double lam = newton_lambda(S, pf, pg, 0.0, scr, &err);  // updated_marginals :301
  if (err) {
    if (threadIdx.x == 0) {
      A.status[bi] = 3;  // NewtonError
      P.G.done[bi] = 1;
    }
    return;
  }
  double ms[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < S.n; i += GT) {
    const double v = S.a[i] * cgrad(S.e1, S.r1, -f[i] - lam);
    P.G.ta[(long)bi * S.n + i] = v;
    ms[0] += v;
  }
  for (int j = threadIdx.x; j < S.m; j += GT) {
    const double v = S.b[j] * cgrad(S.e2, S.r2, -g[j] + lam);
    P.G.tb[(long)bi * S.m + j] = v;
    ms[1] += v;
  }
  block_sum<2>(ms, scr);
  const double dual = h_value(S, pf, pg, lam, scr);  // _h0 (fw.py:111-115)
  double err_f = 0.0;
  if (A.ref_f != nullptr) {  // fw.py:217-219
    for (int i = threadIdx.x; i < S.n; i += GT)
      err_f = fmax(err_f, fabs(f[i] + lam - A.ref_f[(long)bi * S.n + i]));
    err_f = block_reduce(err_f, scr, MaxOp(), 0.0);
  }
  if (threadIdx.x == 0) {
    P.G.dual[bi] = dual;
    A.h0[(long)bi * A.max_iters + t] = dual;
    if (A.err_f != nullptr) A.err_f[(long)bi * A.max_iters + t] = err_f;
    if (fabs(ms[0] - ms[1]) > LMO_MASS_TOL * fmax(ms[0], ms[1])) {  // fw.py:161-166
      A.status[bi] = 1;
      P.G.done[bi] = 1;
    }
  }
}

__device__ __forceinline__ double cost_at(const FwArgs& A, int bi, int i, int j) {
  if (A.C != nullptr) return A.C[((long)bi * A.n + i) * A.m + j];
  const double d = fabs(A.x[(long)bi * A.n + i] - A.y[(long)bi * A.m + j]);
  if (A.p == 1.0) return d;
  if (A.p == 2.0) return d * d;
  return pow(d, A.p);
}

// first entry index with idx[e] >= v on a non-decreasing array
__device__ __forceinline__ int lower_bound(const int* idx, int E, int v) {
  int lo = 0, hi = E;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (idx[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One side's divergence D(mu | w) (src/entropies.py:104-138); the plan is in
// sweep order, so the entries of index i are contiguous in `idx`.
__device__ double side_div(int e, double rho, int cnt, const double* w, const int* idx,
                           const double* mass, int E, double* scr) {
  double v[3] = {0.0, 0.0, 0.0};  // terms, singular mass, "infinite" flag
  for (int i = threadIdx.x; i < cnt; i += GT) {
    double mu = 0.0;
    for (int k = lower_bound(idx, E, i); k < E && idx[k] == i; ++k) mu += mass[k];
    const double nu = w[i];
    if (nu > 0.0) {
      if (e == UOT_ENT_KL) {
        v[0] += (mu > 0.0 ? mu * log(mu / nu) : 0.0) - mu + nu;
      } else {  // Berg: mu - nu - nu log(mu / nu), infinite at mu = 0
        if (mu == 0.0)
          v[2] = 1.0;
        else
          v[0] += mu - nu - nu * log(mu / nu);
      }
    } else {
      v[1] += mu;
    }
  }
  block_sum<3>(v, scr);
  if (v[2] > 0.0) return CUDART_INF;
  if (e == UOT_ENT_KL) return v[1] > 0.0 ? CUDART_INF : rho * v[0];
  return rho * (v[0] + v[1]);
}

__global__ void __launch_bounds__(GT) fwg_step(GenArgs P, int t) {
  __shared__ double scr[40];
  const int bi = blockIdx.x;
  if (P.G.done[bi]) return;
  const FwArgs& A = P.A;
  Sides S = P.S;
  S.a += (long)bi * S.n;
  S.b += (long)bi * S.m;
  const int n = S.n, m = S.m, L = n + m - 1;
  double* f = A.f + (long)bi * n;
  double* g = A.g + (long)bi * m;
  const double* af = P.G.af + (long)bi * n;
  const double* ag = P.G.ag + (long)bi * m;
  if (P.G.pstatus[bi] != 0) {  // oracle mass check (ot1d.py:133-136)
    if (threadIdx.x == 0) {
      A.status[bi] = 1;
      P.G.done[bi] = 1;
    }
    return;
  }
  const int E = P.G.pcount[bi];
  const int* pi = P.G.pi + (long)bi * L;
  const int* pj = P.G.pj + (long)bi * L;
  const double* pm = P.G.pm + (long)bi * L;
  // linear gap (fw.py:172) and the plan's transport cost (duality.py:331-332)
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n; i += GT) v[0] += P.G.ta[(long)bi * n + i] * (af[i] - f[i]);
  for (int j = threadIdx.x; j < m; j += GT) v[0] += P.G.tb[(long)bi * m + j] * (ag[j] - g[j]);
  for (int e = threadIdx.x; e < E; e += GT) v[1] += pm[e] * cost_at(A, bi, pi[e], pj[e]);
  block_sum<2>(v, scr);
  const double fw_gap = v[0];
  const double primal = v[1] + side_div(S.e1, S.r1, n, S.a, pi, pm, E, scr) +
                        side_div(S.e2, S.r2, m, S.b, pj, pm, E, scr);
  const double dual = P.G.dual[bi];
  const double pd = primal - dual;
  // the last oracle plan is the certificate (fw.py:246)
  for (int e = threadIdx.x; e < E; e += GT) {
    A.ei[(long)bi * L + e] = pi[e];
    A.ej[(long)bi * L + e] = pj[e];
    A.em[(long)bi * L + e] = pm[e];
  }
  if (threadIdx.x == 0) {
    A.fw_gap[(long)bi * A.max_iters + t] = fw_gap;
    A.pd_gap[(long)bi * A.max_iters + t] = pd;
    A.iterations[bi] = t + 1;
    A.count[bi] = E;
    A.summary[bi * 3 + 0] = primal;
    A.summary[bi * 3 + 1] = dual;
  }
  if (A.early_exit && pd < A.gap_tol) {  // converged: no step (fw.py:220-222)
    if (threadIdx.x == 0) P.G.done[bi] = 1;
    return;
  }
  double gm;
  if (A.step == UOT_STEP_HARMONIC) {
    gm = 2.0 / (2.0 + t);
  } else {  // line_search_h0 (fw.py:131-148); every value solves its own translation
    int err = 0;
    auto value = [&](double c) {
      auto pf = [&](int i) { return blend(f[i], af[i], c); };
      auto pg = [&](int j) { return blend(g[j], ag[j], c); };
      int e2 = 0;
      const double lam = newton_lambda(S, pf, pg, 0.0, scr, &e2);
      if (e2) err = e2;
      return e2 ? -CUDART_INF : h_value(S, pf, pg, lam, scr);
    };
    double lo = 0.0, hi = 1.0;
    for (int it = 0; it < 60; ++it) {  // ternary_max (fw.py:118-128)
      const double m1 = lo + (hi - lo) / 3.0, m2 = hi - (hi - lo) / 3.0;
      if (value(m1) < value(m2))
        lo = m1;
      else
        hi = m2;
    }
    gm = 0.5 * (lo + hi);
    double best = value(gm);
    const double v0 = value(0.0), v1 = value(1.0);
    if (v0 > best) {  // max() keeps the first of equal keys
      best = v0;
      gm = 0.0;
    }
    if (v1 > best) gm = 1.0;
    if (err) {
      if (threadIdx.x == 0) {
        A.status[bi] = 3;
        P.G.done[bi] = 1;
      }
      return;
    }
  }
  if (A.step_size != nullptr && threadIdx.x == 0) A.step_size[(long)bi * A.max_iters + t] = gm;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += GT) f[i] = blend(f[i], af[i], gm);
  for (int j = threadIdx.x; j < m; j += GT) g[j] = blend(g[j], ag[j], gm);
}

// the final translation lam* of the last iterate (fw.py:_finalize :235-252)
__global__ void __launch_bounds__(GT) fwg_finalize(GenArgs P) {
  __shared__ double scr[40];
  const int bi = blockIdx.x;
  const FwArgs& A = P.A;
  Sides S = P.S;
  S.a += (long)bi * S.n;
  S.b += (long)bi * S.m;
  double* f = A.f + (long)bi * S.n;
  double* g = A.g + (long)bi * S.m;
  if (A.status[bi] != 0) return;
  auto pf = [&](int i) { return f[i]; };
  auto pg = [&](int j) { return g[j]; };
  int err = 0;
  const double lam = newton_lambda(S, pf, pg, 0.0, scr, &err);
  if (err) {
    if (threadIdx.x == 0) A.status[bi] = 3;
    return;
  }
  if (threadIdx.x == 0) A.summary[bi * 3 + 2] = lam;
  for (int i = threadIdx.x; i < S.n; i += GT) f[i] += lam;
  for (int j = threadIdx.x; j < S.m; j += GT) g[j] -= lam;
}

}  // namespace

namespace fwk {

size_t generic_ws_bytes(int batch, int n, int m) {
  const size_t B = batch, L = (size_t)n + m - 1;
  return ot_scratch_bytes(batch, n, m) + 256 + sizeof(double) * B * (2 * (size_t)(n + m) + L + 1) +
         sizeof(int) * B * (2 * L + 3) + 256;
}

// FW for non-KL penalties: the host loop launches prep / oracle / step per
// iteration and reads the per-problem done flags every 16 iterations.
int run_fw_generic(const FwArgs& a, int batch, int e1, int e2, void* ws, size_t ws_bytes,
                   cudaStream_t st) {
  if (ws_bytes < generic_ws_bytes(batch, a.n, a.m)) {
    set_error("uot_fw1d_run: workspace too small");
    return UOT_INVALID;
  }
  const int n = a.n, m = a.m;
  const size_t B = batch, L = (size_t)n + m - 1;
  char* p = (char*)ws;
  FwArgs ot{};  // plain oracle on (ta, tb) into the scratch plan
  ot.scratch = (double*)p;
  ot.scratch_i = (int*)(p + sizeof(double) * B * (n + m));
  p += (ot_scratch_bytes(batch, n, m) + 255) / 256 * 256;
  GenArgs P{};
  P.A = a;
  P.S = Sides{n, m, a.a, a.b, e1, e2, a.r1, a.r2};
  P.G.ta = (double*)p;
  P.G.tb = P.G.ta + B * n;
  P.G.af = P.G.tb + B * m;
  P.G.ag = P.G.af + B * n;
  P.G.pm = P.G.ag + B * m;
  P.G.dual = P.G.pm + B * L;
  P.G.pi = (int*)(P.G.dual + B);
  P.G.pj = P.G.pi + B * L;
  P.G.pcount = P.G.pj + B * L;
  P.G.pstatus = P.G.pcount + B;
  P.G.done = P.G.pstatus + B;
  ot.n = n;
  ot.m = m;
  ot.p = a.p;
  ot.mode = 1;
  ot.x = a.x;
  ot.y = a.y;
  ot.a = P.G.ta;
  ot.b = P.G.tb;
  ot.f = P.G.af;
  ot.g = P.G.ag;
  ot.ei = P.G.pi;
  ot.ej = P.G.pj;
  ot.em = P.G.pm;
  ot.count = P.G.pcount;
  ot.status = P.G.pstatus;
  ot.C = a.C;
  UOT_CUDA_TRY(cudaMemsetAsync(P.G.done, 0, sizeof(int) * B, st));
  UOT_CUDA_TRY(cudaMemsetAsync(a.status, 0, sizeof(int) * B, st));
  UOT_CUDA_TRY(cudaMemsetAsync(a.iterations, 0, sizeof(int) * B, st));
  UOT_CUDA_TRY(cudaMemsetAsync(a.count, 0, sizeof(int) * B, st));
  std::vector<int> done(B);
  for (int t = 0; t < a.max_iters; ++t) {
    fwg_prep<<<batch, GT, 0, st>>>(P, t);
    UOT_CHECK_LAUNCH();
    const int rc = launch_fw_ot(ot, batch, st);
    if (rc != UOT_OK) return rc;
    fwg_step<<<batch, GT, 0, st>>>(P, t);
    UOT_CHECK_LAUNCH();
    if (a.early_exit && (t % 16 == 15)) {
      UOT_CUDA_TRY(cudaMemcpyAsync(done.data(), P.G.done, sizeof(int) * B,
                                   cudaMemcpyDeviceToHost, st));
      UOT_CUDA_TRY(cudaStreamSynchronize(st));
      if (std::all_of(done.begin(), done.end(), [](int v) { return v != 0; })) break;
    }
  }
  fwg_finalize<<<batch, GT, 0, st>>>(P);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

}  // namespace fwk
}  // namespace uot

using namespace uot;

extern "C" int uot_translation(int32_t batch, int32_t n, int32_t m, const double* a,
                               const double* b, const double* f, const double* g, int32_t ent1,
                               int32_t ent2, double rho1, double rho2, int32_t solve, double lam0,
                               double tol, int32_t max_iters, double* lam, double* ta, double* tb,
                               double* h, int32_t* status, void* stream) {
  if (batch < 1 || n < 1 || m < 1 || a == nullptr || b == nullptr || f == nullptr ||
      g == nullptr || !(rho1 > 0.0) || !(rho2 > 0.0) || !(tol > 0.0) || max_iters < 1) {
    set_error("uot_translation: invalid arguments");
    return UOT_INVALID;
  }
  if (solve && (ent1 == UOT_ENT_BALANCED || ent2 == UOT_ENT_BALANCED)) {
    set_error("optimal translation needs strictly convex conjugates (KL or Berg)");
    return UOT_UNSUPPORTED_ENTROPY;
  }
  Sides S{n, m, a, b, ent1, ent2, rho1, rho2};
  S.tol = tol;
  S.max_iters = max_iters;
  translation_kernel<<<batch, GT, 0, (cudaStream_t)stream>>>(S, f, g, solve, lam0, lam, ta, tb, h,
                                                             status);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
