// fw1d_kernel.cuh -- batched 1-D OT oracle (Algorithm 1) and batched Frank-Wolfe UOT
// at eps = 0 (K4/K5/K6 of SURVEY.md §2.2).
//
// Reference: src/ot1d.py:112-172 (solve_ot_1d), src/fw.py:106-232 (_h0,
// ternary line search, _lmo, fw_solve), src/duality.py:175-178, :279-303,
// :320-344 (lambda_star, _eval_h_kl, updated_marginals, eval_primal).
//
// Design: one CTA per problem, THREADS x EPT elements per side held in
// registers for the whole run (x, y and the cumulative masses live in shared
// memory for the random accesses of the oracle), so an FW iteration touches
// HBM only for its three trace scalars.  The monotone sweep is restated as a
// merge of cumulative masses: with A_k = sum_{i<=k} ta_i and B_l likewise,
// source event k happens after the target events with B_l < A_k (ties go to
// the source, ot1d.py:158), so its partner index is a binary search, and the
// dual potentials are prefix sums of cost differences along the staircase:
//   r_{k+1} = r_k + C(k+1, j_k) - C(k, j_k),  s_{l+1} = s_l + C(i_l, l+1) - C(i_l, l)
// starting from r_0 = 0, s_0 = C(0,0) (ot1d.py:138-166).  The line search
// minimises the convex log-partition phi(gamma) (H_0 = const - (r1+r2) e^phi,
// fw.py:106-148) by safeguarded Newton on three moments per pass instead of
// the reference's 123 ternary evaluations (FW parity).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#pragma once

#include "../../include/uot_b200.h"
#include "blockops.cuh"
#include "common.cuh"

namespace uot {
namespace fwk {
#ifdef UOT_NEWTON_STATS
static __device__ unsigned long long g_newton_stats[2];  // passes, line searches
#endif

constexpr int FW_THREADS = 256;
constexpr int FW_THREADS_BIG = 1024;  // large problems (n or m > 4096)
#ifndef FW_MINB
#define FW_MINB 2
#endif

struct FwArgs {
  int n, m;
  double p;
  double r1, r2;
  int step;
  int max_iters;
  double gap_tol;
  int early_exit;
  int mode;  // 0 = Frank-Wolfe, 1 = plain OT oracle on (a, b)
  const double* x;
  const double* y;
  const double* a;
  const double* b;
  double* f;
  double* g;
  double* h0;
  double* fw_gap;
  double* pd_gap;
  int* iterations;
  int* ei;
  int* ej;
  double* em;
  int* count;
  double* summary;
  int* status;
  double* step_size;
  double* scratch;  // [batch][n+m] doubles + [batch][n+m][2] ints (plan extraction)
  int* scratch_i;
  // pairwise FW atom store (fw.py:70-95), cap = max_iters + 1 slots per problem
  int cap;
  double* atoms;  // [batch][cap][n+m] (r | s) rows
  double* wts;    // [batch][cap] weight of each slot
  int* act;       // [batch][cap] active slots in insertion order
  int* natoms;    // optional [batch][max_iters] trace
  const double* ref_f;  // optional [batch][n]: reference potential
  double* err_f;        // optional [batch][max_iters]: sup error of the translated iterate
  const double* C;      // optional [batch][n][m]: explicit cost (PK = 3), else |x - y|^p
  // parity / trace mode (optional): replayed step sizes and away positions,
  // per-iteration plan-support hash and entry count
  const double* step_in;
  const int* away_in;
  unsigned long long* supp_hash;
  int* supp_nnz;
  // large problems (NT = FW_THREADS_BIG): the per-problem arrays that live in
  // shared memory on the resident path live here, big_stride bytes per problem
  char* big;
  size_t big_stride;
};

static __device__ __noinline__ double pow_abs(double d, double p) { return pow(fabs(d), p); }

__device__ __forceinline__ double pcost(double xi, double yj, double p) {
  const double d = xi - yj;
  if (p == 2.0) return d * d;
  const double ad = fabs(d);
  if (p == 1.0) return ad;
  return pow_abs(d, p);
}

// Cost kinds resolved at compile time for the FW kernels: PK = 0 -> p = 2,
// 1 -> p = 1, 2 -> general p (one out-of-line pow keeps the kernel small),
// 3 -> explicit matrix (ExplicitMatrix, src/ot1d.py:100-107; Cta::cost).
template <int PK>
__device__ __forceinline__ double pcost_k(double xi, double yj, double p) {
  const double d = xi - yj;
  if constexpr (PK == 0) return d * d;
  else if constexpr (PK == 1) return fabs(d);
  else return pow_abs(d, p);
}

template <int NW>
__device__ __forceinline__ int ibsum(int v, int* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  int s = 0;
  for (int w = 0; w < NW; ++w) s += scratch[w];
  __syncthreads();
  return s;
}

// Exclusive block max-scan of one int per thread (identity -1).
__device__ __forceinline__ int excl_max_scan(int v, int* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = max(incl, t);
  }
  int excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = -1;
  __syncthreads();
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  for (int w = 0; w < warp; ++w) excl = max(excl, scratch[w]);
  __syncthreads();
  return excl;
}

// Per-problem CTA.  Thread t owns source/target elements t*EPT .. t*EPT+EPT-1
// of each side.  Shared memory holds the supports, the constant weights, the
// breakpoints and the merge ranks; registers hold the potentials.

// Merge-rank type: 16-bit on the resident path (n, m <= 4096), 32-bit for
// large problems.
template <int NT>
using RankT = std::conditional_t<(NT > FW_THREADS), int, unsigned short>;

template <int EPT, int PK, int NT = FW_THREADS>
struct Cta {
  static constexpr int NW = NT / 32;
  using RK = RankT<NT>;
  int n, m;
  double p;
  const double* sx;
  const double* sy;
  double* sA;
  double* sB;
  RK* rkA;  // rkA[k] = #target events before source event k in the merge
  RK* rkB;  // rkB[l] = #source events before target event l
  double* zred;  // scratch of the zero-weight fix (own syncs)
  bool zeros;  // the problem has zero-weight atoms (exact-repeat fix needed)
  const double* cm = nullptr;  // PK == 3: this problem's [n][m] cost matrix

  // C(i, j): the cost at source i, target j (src/ot1d.py:92-109)
  __device__ __forceinline__ double cost(int i, int j) const {
    if constexpr (PK == 3) return __ldg(cm + (long)i * m + j);
    else return pcost_k<PK>(sx[i], sy[j], p);
  }

  __device__ int src(int e) const { return threadIdx.x * EPT + e; }

  // Merge path over the breakpoints: thread t emits merged positions
  // [2 EPT t, 2 EPT (t+1)) of the sweep order (source first on ties,
  // ot1d.py:158) after one diagonal binary search, recording for every event
  // its partner index -- the number of events of the other side before it.
  __device__ void merge_ranks() {
    const int na = n - 1, nb = m - 1, E = na + nb;
    constexpr int IPT = 2 * EPT;
    const int d0 = min((int)threadIdx.x * IPT, E);
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sA[mid] <= sB[d0 - 1 - mid])
        lo = mid + 1;
      else
        hi = mid;
    }
    int i = lo, j = d0 - lo;
#pragma unroll (EPT <= 32 ? IPT : 1)
    for (int s = 0; s < IPT; ++s) {
      if (d0 + s < E) {
        const double av = i < na ? sA[i] : CUDART_INF;
        const double bv = j < nb ? sB[j] : CUDART_INF;
        const bool takeA = av <= bv;
        RK* dst = takeA ? rkA + i : rkB + j;
        *dst = (RK)(takeA ? j : i);
        i += takeA;
        j += !takeA;
      }
    }
  }

  // Balanced 1-D OT oracle on (ta, tb): cumulative masses -> merge ranks ->
  // dual potentials (r, s).  Leaves sA/sB/rkA/rkB describing the plan.
  template <typename PING>
  __device__ void oracle(const double (&ta)[EPT], const double (&tb)[EPT], double (&r)[EPT],
                         double (&s)[EPT], double& mass_a, double& mass_b, PING& ping) {
    double pa[EPT], pb[EPT];
    double ca = 0.0, cb = 0.0;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      ca += ta[e];
      pa[e] = ca;
      cb += tb[e];
      pb[e] = cb;
    }
    double tot[2] = {ca, cb}, totals[2];
    bops::block_scan_excl<NW, 2>(tot, totals, ping.next());
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = src(e);
      if (i < n) sA[i] = tot[0] + pa[e];
      if (i < m) sB[i] = tot[1] + pb[e];
    }
    mass_a = totals[0];
    mass_b = totals[1];
    oracle_tail(ta, tb, r, s, ping);
  }

  // The oracle from breakpoints scanned before the tilt factors were known:
  // B = scale (offset + local inclusive prefix) of the unscaled weights (the
  // scan then doubles as the log-sum-exp reduction: one block sync less).
  template <typename PING>
  __device__ void oracle_scaled(const double (&ta)[EPT], const double (&tb)[EPT],
                                const double (&pa)[EPT], const double (&pb)[EPT], double offa,
                                double offb, double sca, double scb, double (&r)[EPT],
                                double (&s)[EPT], PING& ping) {
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = src(e);
      if (i < n) sA[i] = sca * (offa + pa[e]);
      if (i < m) sB[i] = scb * (offb + pb[e]);
    }
    oracle_tail(ta, tb, r, s, ping);
  }

  template <typename PING>
  __device__ __forceinline__ void oracle_tail(const double (&ta)[EPT], const double (&tb)[EPT],
                                              double (&r)[EPT], double (&s)[EPT], PING& ping) {
    if (zeros) {
      // A zero-weight atom must repeat its predecessor's breakpoint bit for
      // bit (the reference emits no entry for it, ot1d.py:149-153), but the
      // block scan associates differently across thread boundaries.
      int lza = -1, lzb = -1;
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = src(e);
        if (i < n && ta[e] > 0.0) lza = i;
        if (i < m && tb[e] > 0.0) lzb = i;
      }
      int pra = excl_max_scan(lza, reinterpret_cast<int*>(zred));
      int prb = excl_max_scan(lzb, reinterpret_cast<int*>(zred));
      __syncthreads();
      double fa[EPT], fb[EPT];
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = src(e);
        fa[e] = (i < n && ta[e] == 0.0) ? (pra >= 0 ? sA[pra] : 0.0) : -1.0;
        fb[e] = (i < m && tb[e] == 0.0) ? (prb >= 0 ? sB[prb] : 0.0) : -1.0;
        if (i < n && ta[e] > 0.0) pra = i;
        if (i < m && tb[e] > 0.0) prb = i;
      }
      __syncthreads();
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = src(e);
        if (fa[e] >= 0.0) sA[i] = fa[e];
        if (fb[e] >= 0.0) sB[i] = fb[e];
      }
    }
    __syncthreads();
    merge_ranks();
    __syncthreads();
    // cost increments along the staircase
    double da[EPT], db[EPT];
    double la = 0.0, lb = 0.0;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = src(e);
      da[e] = 0.0;
      db[e] = 0.0;
      if (i >= 1 && i < n) {
        const int j = rkA[i - 1];  // partner of source event i-1
        da[e] = cost(i, j) - cost(i - 1, j);
      }
      if (i >= 1 && i < m) {
        const int k = rkB[i - 1];  // partner of target event i-1
        db[e] = cost(k, i) - cost(k, i - 1);
      }
      la += da[e];
      lb += db[e];
    }
    double off[2] = {la, lb}, unused[2];
    bops::block_scan_excl<NW, 2>(off, unused, ping.next());
    const double s0 = cost(0, 0);
    double ra = off[0], rb = off[1];
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      ra += da[e];
      rb += db[e];
      r[e] = ra;
      s[e] = s0 + rb;
    }
  }

  // Plan of the current merge, compacted to positive-mass entries in sweep
  // order (ot1d.py:149-153).  vals: n+m doubles, codes: 2(n+m) ints.
  __device__ void extract_plan(double* vals, int* codes, int* ei, int* ej, double* em,
                               int* count, double total) {
    const int nev = (n - 1) + (m - 1);
    for (int i = threadIdx.x; i < n - 1; i += NT) {
      const int j = rkA[i];
      const int rank = i + j;
      vals[rank] = sA[i];
      codes[2 * rank] = i + 1;
      codes[2 * rank + 1] = j;
    }
    for (int l = threadIdx.x; l < m - 1; l += NT) {
      const int k = rkB[l];
      const int rank = l + k;
      vals[rank] = sB[l];
      codes[2 * rank] = k;
      codes[2 * rank + 1] = l + 1;
    }
    __syncthreads();
    int base = 0;
    int* iscr = reinterpret_cast<int*>(zred);
    for (int s0 = 0; s0 <= nev; s0 += NT) {
      const int s = s0 + threadIdx.x;
      double mass = 0.0;
      int ii = 0, jj = 0;
      if (s <= nev) {
        const double lo = s == 0 ? 0.0 : fmin(vals[s - 1], total);
        const double hi = s == nev ? total : fmin(vals[s], total);
        mass = hi - lo;
        if (s > 0) {
          ii = codes[2 * (s - 1)];
          jj = codes[2 * (s - 1) + 1];
        }
      }
      const int keep = (s <= nev && mass > 0.0) ? 1 : 0;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      int incl = keep;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      __syncthreads();
      if (lane == 31) iscr[warp] = incl;
      __syncthreads();
      int off = 0, tot = 0;
      for (int w = 0; w < NW; ++w) {
        if (w < warp) off += iscr[w];
        tot += iscr[w];
      }
      __syncthreads();
      if (keep) {
        const int pos = base + off + incl - 1;
        ei[pos] = ii;
        ej[pos] = jj;
        em[pos] = mass;
      }
      base += tot;
    }
    if (threadIdx.x == 0) *count = base;
    __syncthreads();
  }

  // Support hash and entry count of the current merge (trace mode): entry
  // after source event i is (i + 1, rkA[i]), after target event l is
  // (rkB[l], l + 1), the first is (0, 0); its mass is the next merged
  // breakpoint minus this one, both capped at the total (extract_plan's
  // rule), and the next breakpoint is the smaller of the two sides' next
  // unconsumed ones.
  __device__ void plan_hash(double total, unsigned long long* out_h, int* out_n) {
    __shared__ unsigned long long hs;
    __shared__ int ns;
    if (threadIdx.x == 0) {
      hs = 0ull;
      ns = 0;
    }
    __syncthreads();
    const int na = n - 1, nb = m - 1;
    unsigned long long h = 0ull;
    int cnt = 0;
    auto entry = [&](int i, int j, double lo, double nxt) {
      if (fmin(nxt, total) - fmin(lo, total) > 0.0) {
        h += pair_hash(i, j);
        ++cnt;
      }
    };
    auto va = [&](int i) { return i < na ? sA[i] : CUDART_INF; };
    auto vb = [&](int j) { return j < nb ? sB[j] : CUDART_INF; };
    if (threadIdx.x == 0) entry(0, 0, 0.0, fmin(va(0), vb(0)));
    for (int i = threadIdx.x; i < na; i += NT) {
      const int j = rkA[i];
      entry(i + 1, j, sA[i], fmin(va(i + 1), vb(j)));
    }
    for (int l = threadIdx.x; l < nb; l += NT) {
      const int k = rkB[l];
      entry(k, l + 1, sB[l], fmin(va(k), vb(l + 1)));
    }
    h = warp_sum(h);
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&hs, h);
      atomicAdd(&ns, cnt);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      *out_h = hs;
      *out_n = ns;
    }
  }
};

// Pairwise FW state shared by all threads of the CTA: active atoms and
// slots used so far (identical in every thread).
struct PfwState {
  int na, ntot;
  double* wts;  // weight of each slot: shared memory when cap <= PFW_CAP_S, else the workspace
  int* act;     // active slots in insertion order (likewise)
};
constexpr int PFW_CAP_S = 1024;
#ifndef PFW_CH
#define PFW_CH 2  // atoms scored per block reduction
#endif

// One pairwise step (fw.py:275-310) after the LMO of iteration t: scores of
// the active atoms against the tilted marginals (one warp per atom, coalesced
// rows from the workspace store) and their sup-norm distance to the new
// atom (r, s); the away atom = argmin score (lowest position on ties);
// safeguarded Newton on phi along (r, s) - away over [0, w_away] (fw.py:
// 295-297 runs a ternary search + endpoint check on the same concave H0);
// weight transfer, merge into an atom closer than 1e-12 (:260-272), drop of
// zero weights, and the iterate update d += gamma ((r, s) - away).  Returns
// gamma.  Slot weights and the active list live in shared memory (up to
// PFW_CAP_S slots, i.e. max_iters < 1024; the workspace beyond that); the atom
// rows in the workspace, each element read back by the thread that wrote it.
template <int EPT, int PK, int NT, typename PING>
__device__ double pfw_step(Cta<EPT, PK, NT>& c, const FwArgs& A, int b, int t, double (&f)[EPT],
                           double (&g)[EPT], const double (&r)[EPT], const double (&s)[EPT],
                           const double (&ta)[EPT], const double (&tb)[EPT], double mta,
                           double mtb, double& sha, double& shb, double i1, double i2, double t1,
                           double t2, const double* sal, const double* sbe, const double* tab,
                           PING& ping, PfwState& pst) {
  const int n = c.n, m = c.m, nm = n + m;
  using CT = Cta<EPT, PK, NT>;
  (void)sal;
  __shared__ int na_s;
  const long sb0 = (long)b * A.cap;
  const double* AT = A.atoms + sb0 * nm;
  double* wts = pst.wts;
  int* act = pst.act;
  // Scores <atom, (ta, tb)> and sup-norm distances to the new atom, all
  // threads sharing each stored row: a thread reads exactly the elements it
  // wrote (same ownership as the registers), PFW_CH atoms per block reduction
  // (sums only: the sup-norm test |atom - new| < 1e-12 is a count of the
  // elements that fail it), and every thread tracks the away atom (lowest
  // score, lowest position on ties) and the first atom within 1e-12 of the
  // new one from the bit-identical reduced values.
  constexpr int CH = PFW_CH;
  double best = CUDART_INF;
  int bp = 0x7fffffff, hp = 0x7fffffff;
  for (int p0 = 0; p0 < pst.na; p0 += CH) {
    double sd[2 * CH];  // scores, then counts of elements farther than 1e-12
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      double sck = 0.0;
      int far = 0;
      if (p0 + k < pst.na) {
        const double* row = AT + (long)act[p0 + k] * nm;
#pragma unroll (EPT <= 32 ? EPT : 1)
        for (int e = 0; e < EPT; ++e) {
          const int i = c.src(e);
          if (i < n) {
            const double v = row[i];
            sck = fma(v, ta[e], sck);
            far += !(fabs(v - r[e]) < 1e-12);
          }
          if (i < m) {
            const double v = row[n + i];
            sck = fma(v, tb[e], sck);
            far += !(fabs(v - s[e]) < 1e-12);
          }
        }
      }
      sd[k] = sck;
      sd[CH + k] = (double)far;
    }
    bops::block_sum<CT::NW, 2 * CH>(sd, ping.next());
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (p0 + k < pst.na) {
        if (sd[k] < best) {  // positions ascend: the first minimum is kept
          best = sd[k];
          bp = p0 + k;
        }
        if (hp == 0x7fffffff && sd[CH + k] == 0.0) hp = p0 + k;
      }
    }
  }
  const long tix = (long)b * A.max_iters + t;
  const bool replay = A.away_in != nullptr && A.step_in != nullptr;
  const int away = replay ? max(__ldg(A.away_in + tix), 0) : bp;
  const int hit = hp == 0x7fffffff ? -1 : hp;
  const int aslot = act[away];
  const double* ra = AT + (long)aslot * nm;
  double dA[EPT], dB[EPT];
  double mom[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // [4]: elements of the direction above 1e-12
  double mxs[2] = {-CUDART_INF, -CUDART_INF};
  int farn = 0;
#pragma unroll (EPT <= 32 ? EPT : 1)
  for (int e = 0; e < EPT; ++e) {
    const int i = c.src(e);
    dA[e] = i < n ? r[e] - ra[i] : 0.0;
    dB[e] = i < m ? s[e] - ra[n + i] : 0.0;
    const double va = dA[e] * i1, vb = dB[e] * i2;
    mom[0] += ta[e] * va;
    mom[1] += ta[e] * va * va;
    mom[2] += tb[e] * vb;
    mom[3] += tb[e] * vb * vb;
    farn += !(fabs(dA[e]) < 1e-12);
    farn += !(fabs(dB[e]) < 1e-12);
    if (i < n && sal[i] > 0.0) mxs[0] = bops::dmax(mxs[0], -va);
    if (i < m && sbe[i] > 0.0) mxs[1] = bops::dmax(mxs[1], -vb);
  }
  mom[4] = (double)farn;
  bops::block_red<Cta<EPT, PK, NT>::NW, 5, 2>(mom, mxs, ping.next());
  const double gmax = wts[aslot];
  double gam = 0.0;
  if (replay) {  // the reference's away atom and transfer (no step: away < 0)
    gam = __ldg(A.away_in + tix) < 0 ? 0.0 : __ldg(A.step_in + tix);
  } else if (!(gmax <= 0.0 || mom[4] == 0.0)) {  // fw.py:291-293
    // minimise phi(gamma) = t1 LSE_a(u - gamma va) + t2 LSE_b(u' - gamma vb)
    // on [0, gmax]; centred moments as in the FW line search
    const double ca = mom[0] / mta, cb = mom[2] / mtb;
    const double k0 = -(t1 * ca + t2 * cb);
    const double d2 = t1 * fmax(mom[1] / mta - ca * ca, 0.0) +
                      t2 * fmax(mom[3] / mtb - cb * cb, 0.0);
    if (k0 < 0.0) {
      double lo = 0.0, hi = gmax;
      gam = (d2 > 0.0) ? fmin(gmax, -k0 / d2) : gmax;
      for (int it = 0; it < 32; ++it) {
        const double pha = sha + gam * mxs[0];
        const double phb = shb + gam * mxs[1];
        double mm[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll (EPT <= 32 ? EPT : 1)
        for (int e = 0; e < EPT; ++e) {
          const int i = c.src(e);
          const double va = dA[e] * i1, vb = dB[e] * i2;
          const double wa0 = i < n ? sal[i] : 0.0, wb0 = i < m ? sbe[i] : 0.0;
          const double wa = bops::wexp(wa0, -f[e] * i1 - gam * va - pha, tab);
          const double wb = bops::wexp(wb0, -g[e] * i2 - gam * vb - phb, tab);
          const double xa = va - ca, xb = vb - cb;
          mm[0] += wa;
          mm[1] += wa * xa;
          mm[2] += wa * xa * xa;
          mm[3] += wb;
          mm[4] += wb * xb;
          mm[5] += wb * xb * xb;
        }
        bops::block_sum<Cta<EPT, PK, NT>::NW, 6>(mm, ping.next());
        const double a1 = mm[1] / mm[0], a2 = mm[2] / mm[0];
        const double b1 = mm[4] / mm[3], b2 = mm[5] / mm[3];
        const double g1 = k0 - t1 * a1 - t2 * b1;
        const double g2 = t1 * (a2 - a1 * a1) + t2 * (b2 - b1 * b1);
        if (g1 < 0.0)
          lo = gam;
        else
          hi = gam;
        if (gam >= gmax && g1 <= 0.0) {
          gam = gmax;
          break;
        }
        double nxt = (g2 > 0.0) ? gam - g1 / g2 : 0.5 * (lo + hi);
        const bool newton = nxt > lo && nxt < hi;
        if (!newton) nxt = 0.5 * (lo + hi);
        const bool conv = (newton && fabs(nxt - gam) <= 1e-9 * fmax(gmax, gam)) || g1 == 0.0 ||
                          hi - lo <= 1e-15 * fmax(1.0, gmax);
        gam = nxt;
        if (conv) break;
      }
    }
  }
  if (gam > 0.0) {
    // the new atom gets a slot unless it merges into an existing one
    const int nslot = pst.ntot;
    if (hit < 0) {
      double* row = A.atoms + (sb0 + nslot) * nm;
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = c.src(e);
        if (i < n) row[i] = r[e];
        if (i < m) row[n + i] = s[e];
      }
    }
    if (threadIdx.x == 0) {
      double* w = wts;
      int* ac = act;
      w[aslot] = fmax(w[aslot] - gam, 0.0);
      int na = pst.na;
      if (hit >= 0) {
        w[ac[hit]] += gam;
      } else {
        w[nslot] = gam;
        ac[na++] = nslot;
      }
      int k = 0;
      for (int q = 0; q < na; ++q) {
        const int sl = ac[q];
        if (w[sl] > 0.0) ac[k++] = sl;
      }
      na_s = k;
    }
    if (hit < 0) ++pst.ntot;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      f[e] += gam * dA[e];
      g[e] += gam * dB[e];
    }
    if (sha > -CUDART_INF) sha += gam * mxs[0];
    if (shb > -CUDART_INF) shb += gam * mxs[1];
    __syncthreads();
    pst.na = na_s;
  }
  if (A.natoms != nullptr && threadIdx.x == 0) A.natoms[(long)b * A.max_iters + t] = pst.na;
  return gam;
}

// NT = FW_THREADS: resident path (per-problem arrays in shared memory, two
// CTAs per SM).  NT = FW_THREADS_BIG: large problems -- the same arrays in the
// global workspace (L2-resident per problem), 32-bit merge ranks, one CTA of
// 1024 threads per problem.
// FULL: n = m = NT * EPT exactly (cfg2: 1024 = 256 x 4) -- the sizes are
// compile-time constants, so every bounds test on an owned element folds away
// and the shared-memory sub-array offsets are immediates.
template <int EPT, int PK, bool PW, int NT = FW_THREADS, bool FULL = false>
__global__ void __launch_bounds__(NT, NT == FW_THREADS ? FW_MINB : 1) fw1d_kernel(FwArgs A) {
  constexpr int NW = NT / 32;
  constexpr int BUF = 16 * NW;  // one reduction buffer (doubles)
  using RK = RankT<NT>;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(16) double red[3 * BUF];
  __shared__ double tab[32];
  const int b = blockIdx.x;
  const int n = FULL ? NT * EPT : A.n, m = FULL ? NT * EPT : A.m;
  if constexpr (FULL) __builtin_assume(threadIdx.x < NT);
  double* base = smem;
  if constexpr (NT != FW_THREADS) base = reinterpret_cast<double*>(A.big + (size_t)b * A.big_stride);
  double* sx = base;
  double* sy = sx + n;
  double* sA = sy + m;
  double* sB = sA + n;
  double* sal = sB + m;  // constant weights
  double* sbe = sal + n;
  RK* rkA = reinterpret_cast<RK*>(sbe + m);
  RK* rkB = rkA + n;
  Cta<EPT, PK, NT> c{n, m, A.p, sx, sy, sA, sB, rkA, rkB, red + 2 * BUF, false};
  if constexpr (PK == 3) c.cm = A.C + (long)b * n * m;
  bops::Ping<BUF> ping{red, 0};
  bops::load_exp_table(tab);

  int nz = 0;
  for (int i = threadIdx.x; i < n; i += NT) {
    sx[i] = A.x[(long)b * n + i];
    const double w = A.a[(long)b * n + i];
    sal[i] = w;
    nz += (w == 0.0);
  }
  for (int j = threadIdx.x; j < m; j += NT) {
    sy[j] = A.y[(long)b * m + j];
    const double w = A.b[(long)b * m + j];
    sbe[j] = w;
    nz += (w == 0.0);
  }
  c.zeros = ibsum<NW>(nz, reinterpret_cast<int*>(c.zred)) > 0;  // (syncs: smem now visible)

  double f[EPT], g[EPT];
#pragma unroll (EPT <= 32 ? EPT : 1)
  for (int e = 0; e < EPT; ++e) {
    const int i = c.src(e);
    f[e] = i < n ? A.f[(long)b * n + i] : 0.0;
    g[e] = i < m ? A.g[(long)b * m + i] : 0.0;
  }
  double* vals = A.scratch + (long)b * (n + m);
  int* codes = A.scratch_i + (long)b * 2 * (n + m);
  int* ei = A.ei + (long)b * (n + m - 1);
  int* ej = A.ej + (long)b * (n + m - 1);
  double* em = A.em + (long)b * (n + m - 1);

  if (A.mode == 1) {
    // Plain balanced OT on (a, b): src/ot1d.py:112-172.
    double ta[EPT], tb[EPT], r[EPT], s[EPT], ma, mb;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = c.src(e);
      ta[e] = i < n ? sal[i] : 0.0;
      tb[e] = i < m ? sbe[i] : 0.0;
    }
    c.oracle(ta, tb, r, s, ma, mb, ping);
    const int bad = fabs(ma - mb) > 1e-9 * fmax(ma, mb);  // ot1d.py:133-136
    if (threadIdx.x == 0) A.status[b] = bad ? UOT_MASS_BALANCE : 0;
    if (bad) return;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = c.src(e);
      if (i < n) A.f[(long)b * n + i] = r[e];
      if (i < m) A.g[(long)b * m + i] = s[e];
    }
    c.extract_plan(vals, codes, ei, ej, em, A.count + b, fmin(ma, mb));
    return;
  }

  const int lane = threadIdx.x & 31;
  const double r1 = A.r1, r2 = A.r2;
  const double i1 = 1.0 / r1, i2 = 1.0 / r2;
  const double t1 = r1 / (r1 + r2), t2 = r2 / (r1 + r2);
  double malpha, mbeta;
  // Shifts of the two log-sum-exps: exact maxima of u = -f/r1, u' = -g/r2
  // over the positive-weight atoms at t = 0, then the upper bound
  // (1-gamma) shift + gamma max(-r/r1) carried through each update, so no
  // per-iteration max reduction is needed (an underflowing sum falls back
  // to the exact maxima).
  double sha, shb;
  {
    double ms[2] = {0.0, 0.0}, mx[2] = {-CUDART_INF, -CUDART_INF};
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = c.src(e);
      if (i < n) ms[0] += sal[i];
      if (i < m) ms[1] += sbe[i];
      if (i < n && sal[i] > 0.0) mx[0] = bops::dmax(mx[0], -f[e] * i1);
      if (i < m && sbe[i] > 0.0) mx[1] = bops::dmax(mx[1], -g[e] * i2);
    }
    bops::block_red<NW, 2, 2>(ms, mx, ping.next());
    malpha = ms[0];
    mbeta = ms[1];
    sha = mx[0];
    shb = mx[1];
  }

  int status = 0;
  int iters = 0;
  double last_primal = 0.0, last_dual = 0.0;
  __shared__ double pfw_wts_s[PW ? PFW_CAP_S : 1];
  __shared__ int pfw_act_s[PW ? PFW_CAP_S : 1];
  PfwState pst{1, 1, nullptr, nullptr};
  if constexpr (PW) {  // store = {(f0, g0)} with weight 1 (fw.py:332)
    const bool ins = A.cap <= PFW_CAP_S;
    pst.wts = ins ? pfw_wts_s : A.wts + (long)b * A.cap;
    pst.act = ins ? pfw_act_s : A.act + (long)b * A.cap;
    double* row = A.atoms + (long)b * A.cap * (n + m);
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = c.src(e);
      if (i < n) row[i] = f[e];
      if (i < m) row[n + i] = g[e];
    }
    if (threadIdx.x == 0) {
      pst.act[0] = 0;
      pst.wts[0] = 1.0;
    }
    __syncthreads();
  }
  for (int t = 0; t < A.max_iters; ++t) {
    // --- lambda*, H_0 and the tilted marginals (duality.py:175-178, :279-303).
    // The exponentials are shared between the log-sum-exps and the tilt.
    double ta[EPT], tb[EPT], pa[EPT], pb[EPT];
    double sums[2], offs[2];
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      // exponentials, local prefixes and one block scan: the scan's totals are
      // the log-sum-exp sums, its offsets give the breakpoints (oracle_scaled)
      double ca = 0.0, cb = 0.0;
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = c.src(e);
        const double wa = i < n ? sal[i] : 0.0, wb = i < m ? sbe[i] : 0.0;
        ta[e] = bops::wexp(wa, -f[e] * i1 - sha, tab);
        tb[e] = bops::wexp(wb, -g[e] * i2 - shb, tab);
        ca += ta[e];
        pa[e] = ca;
        cb += tb[e];
        pb[e] = cb;
      }
      offs[0] = ca;
      offs[1] = cb;
      bops::block_scan_excl<NW, 2>(offs, sums, ping.next());
      // block-uniform: a stale shift far above the maximum underflowed
      if (!((sums[0] < 1e-280 && sha > -CUDART_INF) || (sums[1] < 1e-280 && shb > -CUDART_INF)))
        break;
      double mx[2] = {-CUDART_INF, -CUDART_INF};
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = c.src(e);
        if (i < n && sal[i] > 0.0) mx[0] = bops::dmax(mx[0], -f[e] * i1);
        if (i < m && sbe[i] > 0.0) mx[1] = bops::dmax(mx[1], -g[e] * i2);
      }
      bops::block_max<NW, 2>(mx, ping.next());
      sha = mx[0];
      shb = mx[1];
    }
    // Scalars, one transcendental per lane: lanes 0/1 take the logs, lanes
    // 0/1/2 the exponentials of H_0 and of the two tilt factors.
    const double lg = log((lane & 1) ? sums[1] : sums[0]);
    const double la = sha + __shfl_sync(bops::FULL, lg, 0);
    const double lb = shb + __shfl_sync(bops::FULL, lg, 1);
    const double lam = (r1 * r2 / (r1 + r2)) * (la - lb);
    const double earg = lane == 0 ? t1 * la + t2 * lb : lane == 1 ? sha - lam / r1 : shb + lam / r2;
    const double ev = exp(earg);  // (libdevice: arguments are not shifted here)
    const double dual = r1 * malpha + r2 * mbeta - (r1 + r2) * __shfl_sync(bops::FULL, ev, 0);
    if (A.err_f != nullptr) {  // fw.py:217-219: translated iterate vs the reference
      double em1[1] = {0.0};
#pragma unroll (EPT <= 32 ? EPT : 1)
      for (int e = 0; e < EPT; ++e) {
        const int i = c.src(e);
        if (i < n) em1[0] = bops::dmax(em1[0], fabs(f[e] + lam - A.ref_f[(long)b * n + i]));
      }
      bops::block_max<NW, 1>(em1, ping.next());
      if (threadIdx.x == 0) A.err_f[(long)b * A.max_iters + t] = em1[0];
    }
    const double sca = sha > -CUDART_INF ? __shfl_sync(bops::FULL, ev, 1) : 0.0;
    const double scb = shb > -CUDART_INF ? __shfl_sync(bops::FULL, ev, 2) : 0.0;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      ta[e] *= sca;
      tb[e] *= scb;
    }
    // --- linear oracle (ot1d.py:112-172 on the tilted marginals, fw.py:159-173)
    double r[EPT], s[EPT];
    const double mta = sca * sums[0], mtb = scb * sums[1];
    c.oracle_scaled(ta, tb, pa, pb, offs[0], offs[1], sca, scb, r, s, ping);
    if (fabs(mta - mtb) > 1e-9 * fmax(mta, mtb)) {  // fw.py:161-166
      status = UOT_MASS_BALANCE;
      break;
    }
    if (A.supp_hash != nullptr)
      c.plan_hash(fmin(mta, mtb), A.supp_hash + (long)b * A.max_iters + t,
                  A.supp_nnz + (long)b * A.max_iters + t);
    // --- gaps, primal and line-search moments at gamma = 0.  log(ta/alpha)
    // = -(f + lam)/r1 exactly, so the KL terms of the oracle plan (whose
    // marginals are ta, tb) need no logarithm (entropies.py:123-131).
    // mr: max of -r/r1, -s/r2 over the positive-weight atoms (shift bounds).
    double acc[9], mr[2] = {-CUDART_INF, -CUDART_INF};
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = c.src(e);
      const double va = (r[e] - f[e]) * i1, vb = (s[e] - g[e]) * i2;
      acc[0] += ta[e] * (r[e] - f[e]);
      acc[1] += tb[e] * (s[e] - g[e]);
      acc[2] += ta[e] * r[e] + tb[e] * s[e];
      if (ta[e] > 0.0) acc[3] += ta[e] * ((-f[e] - lam) * i1);
      if (tb[e] > 0.0) acc[4] += tb[e] * ((-g[e] + lam) * i2);
      if (i < n && sal[i] > 0.0) mr[0] = bops::dmax(mr[0], -r[e] * i1);
      if (i < m && sbe[i] > 0.0) mr[1] = bops::dmax(mr[1], -s[e] * i2);
      acc[5] += ta[e] * va;
      acc[6] += ta[e] * va * va;
      acc[7] += tb[e] * vb;
      acc[8] += tb[e] * vb * vb;
    }
    {
      // one-sync block reduction; the trace sums (0-4) are combined only
      // where they are needed (warp 0 writes the traces; every thread when
      // the early exit tests the primal-dual gap)
      double* rb = ping.next();
      bops::put_sums<NW, 9>(acc, rb);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double mx = bops::warp_dmax(mr[k]);
        if (lane == 0) rb[(9 + k) * NW + (threadIdx.x >> 5)] = mx;
      }
      __syncthreads();
      if (A.early_exit || threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[k] = bops::get_sum<NW>(rb + k * NW);
      }
#pragma unroll
      for (int k = 5; k < 9; ++k) acc[k] = bops::get_sum<NW>(rb + k * NW);
#pragma unroll
      for (int k = 0; k < 2; ++k) mr[k] = bops::get_max<NW>(rb + (9 + k) * NW);
    }
    const double fw_gap = acc[0] + acc[1];
    const double kl1 = acc[3] - mta + malpha, kl2 = acc[4] - mtb + mbeta;
    const double primal = acc[2] + r1 * kl1 + r2 * kl2;
    const double pd_gap = primal - dual;
    if (threadIdx.x == 0) {
      A.h0[(long)b * A.max_iters + t] = dual;
      A.fw_gap[(long)b * A.max_iters + t] = fw_gap;
      A.pd_gap[(long)b * A.max_iters + t] = pd_gap;
    }
    iters = t + 1;
    last_primal = primal;
    last_dual = dual;
    const bool stop = A.early_exit && pd_gap < A.gap_tol;  // fw.py:220-222
    if (stop || t == A.max_iters - 1) {
      c.extract_plan(vals, codes, ei, ej, em, A.count + b, fmin(mta, mtb));
    }
    if constexpr (PW) {
      // pairwise: the step of this iteration is taken before the exit test
      // (fw.py:341-353)
      const double gam = pfw_step(c, A, b, t, f, g, r, s, ta, tb, mta, mtb, sha, shb, i1, i2, t1,
                                  t2, sal, sbe, tab, ping, pst);
      if (A.step_size != nullptr && threadIdx.x == 0) A.step_size[(long)b * A.max_iters + t] = gam;
      if (stop) break;
      continue;
    }
    if (stop) break;
    // --- step size
    double gam;
    if (A.step_in != nullptr) {
      gam = __ldg(A.step_in + (long)b * A.max_iters + t);  // replayed gamma_t
    } else if (A.step == UOT_STEP_HARMONIC) {
      gam = 2.0 / (2.0 + t);  // fw.py:223-224
    } else {
      // minimise phi(gamma) = t1 LSE_a(u - gamma va) + t2 LSE_b(u' - gamma vb).
      // The FW direction carries a translation component (f + c, g - c) that
      // phi ignores exactly (H is translation invariant), so raw moments of
      // va and vb nearly cancel; moments are taken about the gamma = 0 means
      // (ca, cb) and the constant part of phi' is kept separately.
      const double ca = acc[5] / mta, cb = acc[7] / mtb;
      const double k0 = -(t1 * ca + t2 * cb);  // phi'(0)
      const double d2 = t1 * fmax(acc[6] / mta - ca * ca, 0.0) +
                        t2 * fmax(acc[8] / mtb - cb * cb, 0.0);  // starting curvature
      if (!(k0 < 0.0)) {
        gam = 0.0;
      } else {
        double lo = 0.0, hi = 1.0;
        gam = (d2 > 0.0) ? fmin(1.0, -k0 / d2) : 1.0;
#ifdef UOT_NEWTON_STATS
        if (threadIdx.x == 0) atomicAdd(&g_newton_stats[1], 1ull);
#endif
        for (int it = 0; it < 24; ++it) {
          // one pass: centred moments of va / vb under p_gamma, q_gamma; the
          // shift (1-gamma) sh + gamma max(-r/r1) bounds every exponent.
          const double pha = (1.0 - gam) * sha + gam * mr[0];
          const double phb = (1.0 - gam) * shb + gam * mr[1];
          double mom[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll (EPT <= 32 ? EPT : 1)
          for (int e = 0; e < EPT; ++e) {
            const int i = c.src(e);
            const double va = (r[e] - f[e]) * i1, vb = (s[e] - g[e]) * i2;
            const double wa0 = i < n ? sal[i] : 0.0, wb0 = i < m ? sbe[i] : 0.0;
            const double wa = bops::wexp(wa0, -f[e] * i1 - gam * va - pha, tab);
            const double wb = bops::wexp(wb0, -g[e] * i2 - gam * vb - phb, tab);
            const double xa = va - ca, xb = vb - cb;
            mom[0] += wa;
            mom[1] += wa * xa;
            mom[2] += wa * xa * xa;
            mom[3] += wb;
            mom[4] += wb * xb;
            mom[5] += wb * xb * xb;
          }
          bops::block_sum<NW, 6>(mom, ping.next());
#ifdef UOT_NEWTON_STATS
          if (threadIdx.x == 0) atomicAdd(&g_newton_stats[0], 1ull);
#endif
          const double a1 = mom[1] / mom[0], a2 = mom[2] / mom[0];
          const double b1 = mom[4] / mom[3], b2 = mom[5] / mom[3];
          const double g1 = k0 - t1 * a1 - t2 * b1;
          const double g2 = t1 * (a2 - a1 * a1) + t2 * (b2 - b1 * b1);
          if (g1 < 0.0)
            lo = gam;
          else
            hi = gam;
          if (gam >= 1.0 && g1 <= 0.0) {
            gam = 1.0;
            break;
          }
          double nxt = (g2 > 0.0) ? gam - g1 / g2 : 0.5 * (lo + hi);
          const bool newton = nxt > lo && nxt < hi;
          if (!newton) nxt = 0.5 * (lo + hi);
          // Newton converges quadratically: once a Newton step is below
          // 1e-9 the next iterate is exact to rounding (the reference's
          // ternary search resolves gamma to ~1e-5 on flat problems).
          const bool conv = (newton && fabs(nxt - gam) <= 1e-9 * fmax(1.0, gam)) ||
                            g1 == 0.0 || hi - lo <= 1e-15;
          gam = nxt;
          if (conv) break;
        }
      }
    }
    if (A.step_size != nullptr && threadIdx.x == 0) A.step_size[(long)b * A.max_iters + t] = gam;
    // --- update (fw.py:227-230) and the next shift bounds, rounded as numpy
    // rounds (1 - gamma) f + gamma r: two products and a sum, no FMA
    const double omg = 1.0 - gam;
#pragma unroll (EPT <= 32 ? EPT : 1)
    for (int e = 0; e < EPT; ++e) {
      f[e] = __dadd_rn(__dmul_rn(omg, f[e]), __dmul_rn(gam, r[e]));
      g[e] = __dadd_rn(__dmul_rn(omg, g[e]), __dmul_rn(gam, s[e]));
    }
    if (sha > -CUDART_INF) sha = (1.0 - gam) * sha + gam * mr[0];
    if (shb > -CUDART_INF) shb = (1.0 - gam) * shb + gam * mr[1];
  }
  // --- finalize: translate by lambda* (fw.py:235-252), exact maxima
  double mx[2] = {-CUDART_INF, -CUDART_INF};
#pragma unroll (EPT <= 32 ? EPT : 1)
  for (int e = 0; e < EPT; ++e) {
    const int i = c.src(e);
    if (i < n && sal[i] > 0.0) mx[0] = bops::dmax(mx[0], -f[e] * i1);
    if (i < m && sbe[i] > 0.0) mx[1] = bops::dmax(mx[1], -g[e] * i2);
  }
  bops::block_max<NW, 2>(mx, ping.next());
  double ls[2] = {0.0, 0.0};
#pragma unroll (EPT <= 32 ? EPT : 1)
  for (int e = 0; e < EPT; ++e) {
    const int i = c.src(e);
    if (i < n) ls[0] += bops::wexp(sal[i], -f[e] * i1 - mx[0], tab);
    if (i < m) ls[1] += bops::wexp(sbe[i], -g[e] * i2 - mx[1], tab);
  }
  bops::block_sum<NW, 2>(ls, ping.next());
  const double lam = (r1 * r2 / (r1 + r2)) * ((mx[0] + log(ls[0])) - (mx[1] + log(ls[1])));
#pragma unroll (EPT <= 32 ? EPT : 1)
  for (int e = 0; e < EPT; ++e) {
    const int i = c.src(e);
    if (i < n) A.f[(long)b * n + i] = f[e] + lam;
    if (i < m) A.g[(long)b * m + i] = g[e] - lam;
  }
  if (threadIdx.x == 0) {
    A.iterations[b] = iters;
    A.status[b] = status;
    A.summary[b * 3 + 0] = last_primal;
    A.summary[b * 3 + 1] = last_dual;
    A.summary[b * 3 + 2] = lam;
  }
}

inline int ept_for(int nm) {
  const int per = (nm + FW_THREADS - 1) / FW_THREADS;
  if (per <= 1) return 1;
  if (per <= 2) return 2;
  if (per <= 4) return 4;
  if (per <= 8) return 8;
  if (per <= 16) return 16;
  return -1;
}

// Large-problem path: elements per thread at FW_THREADS_BIG threads (EPT 8 /
// 16 in fw1d_big.cu; 32 -- arrays beyond the register budget live in local
// memory: a correctness path -- in fw1d_huge.cu).
// 64 / 128 / 256 -- fw1d_giant.cu: the per-atom loops stay rolled (#pragma
// unroll 1 above EPT 32), so these compile in seconds and run from local memory.
constexpr int FW_EPT_BIG_MAX = 256;  // n, m <= 262144 per problem
inline int ept_for_big(int nm) {
  const int per = (nm + FW_THREADS_BIG - 1) / FW_THREADS_BIG;
  for (int e = 8; e <= FW_EPT_BIG_MAX; e *= 2)
    if (per <= e) return e;
  return -1;
}

// Per-problem array bytes: supports, cumulative masses, weights (3 (n + m)
// doubles) and merge ranks (rk_bytes each).  (At n = m = 4096 that is 213,008 B
// of dynamic shared memory; with the kernels' static 3.3 KB -- 15.6 KB for
// pairwise, whose slot weights and active list sit there -- still under 227 KB.)
inline size_t fw_smem(int n, int m, bool pairwise, size_t rk_bytes = 2) {
  (void)pairwise;  // (the pairwise step no longer stages the new atom on chip)
  return sizeof(double) * 3 * (size_t)(n + m) + rk_bytes * (size_t)(n + m) + 16;
}

constexpr size_t FW_SMEM_MAX = 227 * 1024;

// Whether (n, m) takes the large-problem path (its arrays in the workspace).
// (UOT_FW_FORCE_BIG=1 sends every size there: parity of the two paths in tests.)
inline bool fw_force_big() {
  static const bool f = std::getenv("UOT_FW_FORCE_BIG") != nullptr;
  return f;
}
inline bool fw_big(int n, int m) {
  return fw_force_big() || ept_for(std::max(n, m)) < 0 || fw_smem(n, m, true) > FW_SMEM_MAX;
}
inline size_t fw_big_stride(int n, int m) { return (fw_smem(n, m, true, 4) + 255) / 256 * 256; }

// Large-problem instantiations live in their own translation units
// (fw1d_big.cu, fw1d_pfw_big.cu) so they compile in parallel with the rest.
template <bool PW, int PK>
int launch_fw_big(const FwArgs& a, int batch, cudaStream_t st, int ept) {
  if (ept == 8)
    fw1d_kernel<8, PK, PW, FW_THREADS_BIG><<<batch, FW_THREADS_BIG, 0, st>>>(a);
  else
    fw1d_kernel<16, PK, PW, FW_THREADS_BIG><<<batch, FW_THREADS_BIG, 0, st>>>(a);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
template <bool PW, int PK>
int launch_fw_huge(const FwArgs& a, int batch, cudaStream_t st, int ept) {
  (void)ept;  // 32
  fw1d_kernel<32, PK, PW, FW_THREADS_BIG><<<batch, FW_THREADS_BIG, 0, st>>>(a);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
template <bool PW, int PK>
int launch_fw_giant(const FwArgs& a, int batch, cudaStream_t st, int ept) {
  if (ept == 64)
    fw1d_kernel<64, PK, PW, FW_THREADS_BIG><<<batch, FW_THREADS_BIG, 0, st>>>(a);
  else if (ept == 128)
    fw1d_kernel<128, PK, PW, FW_THREADS_BIG><<<batch, FW_THREADS_BIG, 0, st>>>(a);
  else
    fw1d_kernel<256, PK, PW, FW_THREADS_BIG><<<batch, FW_THREADS_BIG, 0, st>>>(a);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
#define UOT_FW_GIANT(EXT, PW)                                                        \
  EXT template int launch_fw_giant<PW, 0>(const FwArgs&, int, cudaStream_t, int);   \
  EXT template int launch_fw_giant<PW, 1>(const FwArgs&, int, cudaStream_t, int);   \
  EXT template int launch_fw_giant<PW, 2>(const FwArgs&, int, cudaStream_t, int);   \
  EXT template int launch_fw_giant<PW, 3>(const FwArgs&, int, cudaStream_t, int);
#define UOT_FW_BIG(EXT, PW)                                                          \
  EXT template int launch_fw_big<PW, 0>(const FwArgs&, int, cudaStream_t, int);     \
  EXT template int launch_fw_big<PW, 1>(const FwArgs&, int, cudaStream_t, int);     \
  EXT template int launch_fw_big<PW, 2>(const FwArgs&, int, cudaStream_t, int);     \
  EXT template int launch_fw_big<PW, 3>(const FwArgs&, int, cudaStream_t, int);
#define UOT_FW_HUGE(EXT, PW)                                                         \
  EXT template int launch_fw_huge<PW, 0>(const FwArgs&, int, cudaStream_t, int);    \
  EXT template int launch_fw_huge<PW, 1>(const FwArgs&, int, cudaStream_t, int);    \
  EXT template int launch_fw_huge<PW, 2>(const FwArgs&, int, cudaStream_t, int);    \
  EXT template int launch_fw_huge<PW, 3>(const FwArgs&, int, cudaStream_t, int);
#ifndef UOT_FW_BIG_TU
UOT_FW_BIG(extern, false)
UOT_FW_BIG(extern, true)
UOT_FW_HUGE(extern, false)
UOT_FW_HUGE(extern, true)
UOT_FW_GIANT(extern, false)
UOT_FW_GIANT(extern, true)
#endif

template <bool PW>
int launch_fw_impl(const FwArgs& a0, int batch, cudaStream_t st) {
  FwArgs a = a0;
  const int mx = std::max(a.n, a.m);
  const int ept = ept_for(mx);
  const size_t smem = fw_smem(a.n, a.m, PW);
  const bool big = fw_force_big() || ept < 0 || smem > FW_SMEM_MAX;
  const int eptb = big ? ept_for_big(mx) : 0;
  if (big && eptb < 0) {
    set_error("1-D FW / OT kernel supports n, m <= %d per problem",
              FW_EPT_BIG_MAX * FW_THREADS_BIG);
    return UOT_INVALID;
  }
  if (big) {  // arrays after the plan-extraction scratch (fw1d.cu: fw_scratch_bytes)
    if (a.big == nullptr) {
      set_error("1-D FW / OT: workspace lacks the large-problem region");
      return UOT_INVALID;
    }
    a.big_stride = fw_big_stride(a.n, a.m);
  }
  auto go = [&](auto kern, int nt, size_t sm) -> int {
    if (sm > 0)
      UOT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)sm));
    kern<<<batch, nt, sm, st>>>(a);
    UOT_CHECK_LAUNCH();
    return UOT_OK;
  };
  auto by_ept = [&](auto pk) -> int {
    constexpr int PK = decltype(pk)::value;
    if (big)
      return eptb <= 16   ? launch_fw_big<PW, PK>(a, batch, st, eptb)
             : eptb <= 32 ? launch_fw_huge<PW, PK>(a, batch, st, eptb)
                          : launch_fw_giant<PW, PK>(a, batch, st, eptb);
    if constexpr (PK == 0) {  // exact power-of-two sizes: constant-size instantiations
      if (a.n == a.m && a.n == FW_THREADS * ept && !std::getenv("UOT_FW_NOFULL")) {
        if constexpr (!PW) {
          if (ept == 1) return go(fw1d_kernel<1, 0, PW, FW_THREADS, true>, FW_THREADS, smem);
          if (ept == 2) return go(fw1d_kernel<2, 0, PW, FW_THREADS, true>, FW_THREADS, smem);
        }
        if (ept == 4) return go(fw1d_kernel<4, 0, PW, FW_THREADS, true>, FW_THREADS, smem);
        if (ept == 8) return go(fw1d_kernel<8, 0, PW, FW_THREADS, true>, FW_THREADS, smem);
        if constexpr (!PW)
          if (ept == 16) return go(fw1d_kernel<16, 0, PW, FW_THREADS, true>, FW_THREADS, smem);
      }
    }
    switch (ept) {
      case 1: return go(fw1d_kernel<1, PK, PW>, FW_THREADS, smem);
      case 2: return go(fw1d_kernel<2, PK, PW>, FW_THREADS, smem);
      case 4: return go(fw1d_kernel<4, PK, PW>, FW_THREADS, smem);
      case 8: return go(fw1d_kernel<8, PK, PW>, FW_THREADS, smem);
      default: return go(fw1d_kernel<16, PK, PW>, FW_THREADS, smem);
    }
  };
  if (a.C != nullptr) return by_ept(std::integral_constant<int, 3>());
  if (a.p == 2.0) return by_ept(std::integral_constant<int, 0>());
  if (a.p == 1.0) return by_ept(std::integral_constant<int, 1>());
  return by_ept(std::integral_constant<int, 2>());
}

// pairwise instantiation lives in fw1d_pfw.cu (separate translation unit:
// the pairwise branch otherwise raises register pressure / spills of the
// FW and OT kernels)
int launch_fw_pairwise(const FwArgs& a, int batch, cudaStream_t st);
// non-KL penalties (fw1d_generic.cu)
size_t generic_ws_bytes(int batch, int n, int m);
int run_fw_generic(const FwArgs& a, int batch, int e1, int e2, void* ws, size_t ws_bytes,
                   cudaStream_t st);

}  // namespace fwk
}  // namespace uot
