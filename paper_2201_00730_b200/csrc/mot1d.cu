// mot1d.cu -- balanced K-marginal 1-D sweep (Algorithm 3) and the KL
// barycenter Frank-Wolfe (K7/K8/K9 of SURVEY.md §2.2).
//
// Reference: src/barycenter.py:148-233 (multimarginal_cost, solve_mot_1d),
// :236-240 (plan_cost), :298-327 (multimarginal_lambda, _h_value),
// :330-430 (fw_barycenter), :433-443 (extract_barycenter).
//
// Restatement.  With B_q[t] = sum_{s<=t} w_q[s] the
// cumulative masses of list q, the sweep advances coordinate p at its
// breakpoint B_p[t] in the order of the keys (B_p[t], p, t) (ties to the
// lowest coordinate, barycenter.py:218), and the advanced coordinate's dual
// grows by the change of the tuple cost
//   dCc = w_p d (x_p[t+1] + x_p[t] - Bb - Ba),  d = x_p[t+1] - x_p[t],
// where Bb, Ba = Bb + w_p d are the barycentres of the tuple before / after
// (Cc = sum w x^2 - B^2), so f_p[t+1] = f_p[t] + dCc (barycenter.py:225-229).
// Bb of every event is a prefix sum over the merged events of w_p d.
//
// Pipeline per FW iteration, all on device:
//   mot_prep   (cluster of K CTAs per problem, one CTA per list): log-sum-exps,
//              optimal zero-sum translation (DSMEM exchange), tilt, block scan
//              of the breakpoints, mass check, regular samples -> splitters ->
//              per-list split positions (sample sort).
//   mot_bucket (S CTAs per problem): gathers the events of one key range from
//              all K lists, bitonic-sorts them in shared memory, scans the
//              barycentre increments from the range's starting tuple and
//              writes every event's cost increment.
//   mot_update (cluster of K CTAs): per-list prefix sums -> dual atoms,
//              gaps / primal / dual (DSMEM reductions), safeguarded Newton
//              line search on sum_k rho_k LSE_k, update.
// The plan (tuples + masses) of the last iteration is materialised by
// mot_plan_count / mot_plan_write.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "../../include/uot_b200.h"
#include "blockops.cuh"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace uot {
namespace {

constexpr int MT = 512;           // threads of the per-list CTAs
#ifndef UOT_BT
#define UOT_BT 512
#endif
constexpr int BT = UOT_BT;  // threads of the bucket CTAs
#ifndef UOT_BT2
#define UOT_BT2 256
#endif
constexpr int BT2 = UOT_BT2;  // threads of the cost-increment bucket CTAs (mot_bucket)
constexpr int KMAX = 32;          // lists per problem (16-CTA clusters of two lists each)
constexpr int ST = 1024;          // threads of the per-problem splitter CTA
constexpr int SMAX = 768;         // buckets per problem

struct MotArgs {
  int batch, k, n;        // n = row stride (max list length)
  const int* lens;        // device [k] list lengths (shared by the batch)
  const double* omega;    // device [k]
  double rho;             // KL strength: rho_k = omega_k * rho
  int mode;               // 0 = barycenter FW, 1 = balanced sweep on a
  int step;               // UOT_STEP_*
  int max_iters;
  double gap_tol;
  int early_exit;
  int t;                  // iteration index (host loop)
  const double* x;        // [B][K][n]
  const double* a;        // [B][K][n]
  double* f;              // [B][K][n] potentials (untranslated iterate)
  double* ta;             // [B][K][n] tilted weights
  double* A;              // [B][K][n] breakpoints
  double* dcc;            // [B][K][n] cost increments
  int* split;             // [B][S+1][K]
  int S, SS;              // buckets per problem, samples per list
  double* scal;           // [B][4]: dual, (unused)
  double* lam;            // [B][K]
  double* h0;             // [B][max_iters]
  double* fw_gap;
  double* pd_gap;
  int* iterations;        // [B]
  int* done;              // [B]
  int* status;            // [B]
  double* summary;        // [B][2]
  double* out_f;          // [B][K][n] translated final potentials / sweep duals
  int* pidx;              // [B][cap_e][K]
  double* pmass;          // [B][cap_e]
  int* pcount;            // [B]
  int* bcount;            // [B][S]
  int cap_e;
  double* lse;            // [B][K][2] (max, q_k) of the current iterate
  double* mass;           // [B][K] input masses
  double* tmass;          // [B][K] tilted masses
  double* samp;           // [B][K][SS] regular samples (values)
  int* sampt;             // [B][K][SS] (indices)
  int cap;                // events per bucket: the regular-sampling bound (bucket_bound)
  int b0;                 // first problem of this launch (problem groups on streams)
  int upd_s;              // update by mot_update_s (the batch runs ungrouped: < 16 problems)
  int no_bin;             // 1: merge path only (UOT_MOT_NOBIN=1), 2: coarse bins only
                          // (UOT_MOT_COARSEBIN=1) -- parity tests
  int all_states;         // 1: mot_plan keeps every state (zero-mass ones too) and the
                          //    balanced sweep skips its duals (custom tuple costs)
  int cost_given;         // 1: mot_duals takes dcc[q][0] as given (custom tuple costs)
  // parity / trace mode (optional)
  const double* step_in;  // [B][max_iters] replayed gamma_t
  unsigned long long* supp_hash;  // [B][max_iters] plan-support hash
  int* supp_nnz;          // [B][max_iters] plan entry count
};

__device__ __forceinline__ int list_len(const MotArgs& A, int q) {
  return A.lens != nullptr ? A.lens[q] : A.n;
}

constexpr int MNW = MT / 32;
#ifdef UOT_NEWTON_STATS
__device__ unsigned long long g_mot_stats[2];  // Newton passes, line searches
#endif
constexpr int MBUF = 16 * MNW;  // one-sync reduction buffer (doubles)

// EPT consecutive doubles of a row starting at i0 (zero past nq); 16-byte
// vector loads when the run is complete and aligned.
template <int EPT>
__device__ __forceinline__ void load_run(const double* row, int i0, int nq, double (&v)[EPT]) {
  if (EPT % 2 == 0 && i0 + EPT <= nq && ((reinterpret_cast<uintptr_t>(row + i0) & 15) == 0)) {
    const double2* p = reinterpret_cast<const double2*>(row + i0);
#pragma unroll (EPT <= 32 ? (EPT / 2) : 1)
    for (int e = 0; e < EPT / 2; ++e) {
      const double2 u = p[e];
      v[2 * e] = u.x;
      v[2 * e + 1] = u.y;
    }
  } else {
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e) v[e] = i0 + e < nq ? row[i0 + e] : 0.0;
  }
}

template <int EPT>
__device__ __forceinline__ void store_run(double* row, int i0, int nq, const double (&v)[EPT]) {
  if (EPT % 2 == 0 && i0 + EPT <= nq && ((reinterpret_cast<uintptr_t>(row + i0) & 15) == 0)) {
    double2* p = reinterpret_cast<double2*>(row + i0);
#pragma unroll (EPT <= 32 ? (EPT / 2) : 1)
    for (int e = 0; e < EPT / 2; ++e) p[e] = make_double2(v[2 * e], v[2 * e + 1]);
  } else {
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e)
      if (i0 + e < nq) row[i0 + e] = v[e];
  }
}

// ---------------------------------------------------------------------------
// Block helpers (MT threads).

template <int K>
__device__ __forceinline__ void bsum_k(double (&v)[K], double* scr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) scr[k * 32 + warp] = v[k];
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += scr[k * 32 + w];
    v[k] = s;
  }
  __syncthreads();
}

template <int K>
__device__ __forceinline__ void bmax_k(double (&v)[K], double* scr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_max(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) scr[k * 32 + warp] = v[k];
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = -CUDART_INF;
    for (int w = 0; w < nw; ++w) s = fmax(s, scr[k * 32 + w]);
    v[k] = s;
  }
  __syncthreads();
}

// exclusive scan of one double per thread; returns the exclusive prefix and
// the block total.
__device__ __forceinline__ double bscan1(double v, double& total, double* scr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += t;
  }
  __syncthreads();
  if (lane == 31) scr[warp] = s;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double off = 0.0, tot = 0.0;
  for (int w = 0; w < nw; ++w) {
    const double t = scr[w];
    if (w < warp) off += t;
    tot += t;
  }
  __syncthreads();
  total = tot;
  return off + s - v;
}

__device__ __forceinline__ int bscan_maxi(int v, int* scr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s = max(s, t);
  }
  int ex = __shfl_up_sync(0xffffffffu, s, 1);
  if (lane == 0) ex = -1;
  __syncthreads();
  if (lane == 31) scr[warp] = s;
  __syncthreads();
  for (int w = 0; w < warp; ++w) ex = max(ex, scr[w]);
  __syncthreads();
  return ex;
}

// Cluster all-reduce (sum) of NV doubles: each CTA publishes its vector in
// its own shared slot; after the cluster barrier every warp reads the K
// slots in parallel (lane r <- CTA r) and butterfly-reduces them, so every
// thread of every CTA holds bit-identical sums.  `slot` alternates between
// two buffers so one cluster barrier per reduction suffices.
template <int NV>
__device__ __forceinline__ void cluster_sum(double (&v)[NV], double* slots, int& parity) {
  cg::cluster_group cl = cg::this_cluster();
  double* mine = slots + parity * 16;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) mine[k] = v[k];
  }
  cl.sync();
  const int nr = (int)cl.num_blocks();
  const int lane = threadIdx.x & 31;
  const double* other = cl.map_shared_rank(mine, lane < nr ? lane : 0);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = lane < nr ? other[k] : 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  parity ^= 1;
}

// Event codes: (list << 24) | index, ordered like (list, index).
__device__ __forceinline__ int ev_code(int q, int t) { return (q << 24) | t; }
__device__ __forceinline__ int ev_list(int c) { return c >> 24; }
__device__ __forceinline__ int ev_index(int c) { return c & 0xFFFFFF; }

// Composite event key order: (value, list, index) lexicographic.
__device__ __forceinline__ bool key_less(double va, int qa, int ta_, double vb, int qb, int tb) {
  if (va != vb) return va < vb;
  if (qa != qb) return qa < qb;
  return ta_ < tb;
}

// #{ t in [0, len) : (arr[t], q, t) < (v, qs, ts) }
__device__ __forceinline__ int count_keys_below(const double* arr, int len, int q, double v, int qs,
                                                int ts) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key_less(arr[mid], q, mid, v, qs, ts))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// mot_lse: per-list log-sum-exp of the potentials, q_k = LSE_{a_k}(-f_k/rho_k)
// (barycenter.py:307-313), stored as (max, q) with the input mass m_k.  Runs
// once before the loop; mot_update refreshes it for every new iterate.

template <int EPT>
__device__ __forceinline__ void list_lse(const double (&w)[EPT], const double (&fv)[EPT], double irq,
                                         const double* tab, double* red0, double* red1, double& mx,
                                         double& qk, double (&ew)[EPT]) {
  double m1[1] = {-CUDART_INF};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e)
    if (w[e] > 0.0) m1[0] = bops::dmax(m1[0], -fv[e] * irq);
  bops::block_max<MNW, 1>(m1, red0);
  double s1[1] = {0.0};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    ew[e] = bops::wexp(w[e], -fv[e] * irq - m1[0], tab);
    s1[0] += ew[e];
  }
  bops::block_sum<MNW, 1>(s1, red1);
  mx = m1[0];
  qk = m1[0] + log(s1[0]);
}

template <int EPT>
__global__ void __launch_bounds__(MT) mot_lse(MotArgs A) {
  __shared__ __align__(16) double red[2 * MBUF];
  __shared__ double tab[32];
  const int q = blockIdx.x, b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int nq = list_len(A, q);
  bops::load_exp_table(tab);
  __syncthreads();
  const long base = ((long)b * K + q) * n;
  const double irq = 1.0 / (A.omega[q] * A.rho);
  double w[EPT], fv[EPT];
  load_run<EPT>(A.a + base, threadIdx.x * EPT, nq, w);
  load_run<EPT>(A.f + base, threadIdx.x * EPT, nq, fv);
  double ms[1] = {0.0};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) ms[0] += w[e];
  double mx, qk;
  list_lse<EPT>(w, fv, irq, tab, red, red + MBUF, mx, qk, fv);
  bops::block_sum<MNW, 1>(ms, red);
  if (threadIdx.x == 0) {
    A.lse[((long)b * K + q) * 2 + 0] = mx;
    A.lse[((long)b * K + q) * 2 + 1] = qk;
    A.mass[(long)b * K + q] = ms[0];
  }
}

// Optimal zero-sum translation from the K per-list log-sum-exps
// (barycenter.py:316-317): lambda_q = rho_q q_q - (rho_q / rho_tot) sum_r rho_r q_r.
// Every warp computes the three problem sums with the same butterfly, so all
// lists of a problem see bit-identical values.  Returns lambda_q; ex0 / ex1
// / rtot = sum rho q, sum rho m, sum rho.
__device__ __forceinline__ double problem_lambda(const MotArgs& A, int b, int q, double& ex0,
                                                 double& ex1, double& rtot) {
  const int K = A.k, lane = threadIdx.x & 31;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  if (lane < K) {
    const double rr = A.omega[lane] * A.rho;
    a0 = rr * A.lse[((long)b * K + lane) * 2 + 1];
    a1 = rr * A.mass[(long)b * K + lane];
    a2 = rr;
  }
  ex0 = warp_sum(a0);
  ex1 = warp_sum(a1);
  rtot = warp_sum(a2);
  const double rq = A.omega[q] * A.rho;
  return rq * A.lse[((long)b * K + q) * 2 + 1] - (rq / rtot) * ex0;
}

// Exclusive block scan "last positive atom": (index, breakpoint) of the last
// atom with positive tilted weight owned by a lower thread (index -1: none).
__device__ __forceinline__ void excl_last_pos(int& idx, double& val, int* iscr, double* vscr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int si = idx;
  double sv = val;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ti = __shfl_up_sync(0xffffffffu, si, o);
    const double tv = __shfl_up_sync(0xffffffffu, sv, o);
    if (lane >= o && ti > si) {
      si = ti;
      sv = tv;
    }
  }
  int ei = __shfl_up_sync(0xffffffffu, si, 1);
  double ev = __shfl_up_sync(0xffffffffu, sv, 1);
  if (lane == 0) {
    ei = -1;
    ev = 0.0;
  }
  __syncthreads();
  if (lane == 31) {
    iscr[warp] = si;
    vscr[warp] = sv;
  }
  __syncthreads();
  for (int w = 0; w < warp; ++w) {
    if (iscr[w] > ei) {
      ei = iscr[w];
      ev = vscr[w];
    }
  }
  __syncthreads();
  idx = ei;
  val = ev;
}

// Coalesced staging of per-list rows for the run-per-thread kernels: a warp
// reads 512 consecutive bytes per instruction (instead of 32 lines, one per
// thread's 128-byte run) into shared memory laid out as runs of EPT + 2
// doubles (16-byte aligned, conflict-free per-thread 16-byte reads).
template <int EPT>
struct StageRun {
  static constexpr int RUN = EPT + 2;
  static constexpr size_t BYTES = (size_t)MT * RUN * sizeof(double);
  static constexpr bool ON = EPT >= 4 && EPT % 2 == 0 && 2 * BYTES <= 220000;
};

template <int EPT>
__device__ __forceinline__ void stage_store(double* buf, const double* row, int nq) {
  constexpr int RUN = StageRun<EPT>::RUN;
  const int nch = nq >> 1;
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
    for (int j = threadIdx.x; j < nch; j += MT) {
      const int i = 2 * j, r = i / EPT, c = i - r * EPT;
      *reinterpret_cast<double2*>(buf + r * RUN + c) = __ldg(r2 + j);
    }
    if ((nq & 1) && threadIdx.x == 0) {
      const int i = nq - 1, r = i / EPT;
      buf[r * RUN + (i - r * EPT)] = row[i];
    }
  } else {
    for (int i = threadIdx.x; i < nq; i += MT) {
      const int r = i / EPT;
      buf[r * RUN + (i - r * EPT)] = row[i];
    }
  }
}

template <int EPT>
__device__ __forceinline__ void stage_load(const double* buf, int nq, double (&v)[EPT]) {
  constexpr int RUN = StageRun<EPT>::RUN;
  const double2* p = reinterpret_cast<const double2*>(buf + threadIdx.x * RUN);
#pragma unroll (EPT <= 32 ? (EPT / 2) : 1)
  for (int e = 0; e < EPT / 2; ++e) {
    const double2 u = p[e];
    v[2 * e] = u.x;
    v[2 * e + 1] = u.y;
  }
  const int i0 = threadIdx.x * EPT;
  if (i0 + EPT > nq) {
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e)
      if (i0 + e >= nq) v[e] = 0.0;
  }
}

// The reverse: each thread puts its run into the staging buffer; after a
// __syncthreads the row leaves with coalesced 16-byte stores.
template <int EPT>
__device__ __forceinline__ void stage_put(double* buf, const double (&v)[EPT]) {
  double2* p = reinterpret_cast<double2*>(buf + threadIdx.x * StageRun<EPT>::RUN);
#pragma unroll (EPT <= 32 ? (EPT / 2) : 1)
  for (int e = 0; e < EPT / 2; ++e) p[e] = make_double2(v[2 * e], v[2 * e + 1]);
}

template <int EPT>
__device__ __forceinline__ void stage_out(const double* buf, double* row, int nq) {
  constexpr int RUN = StageRun<EPT>::RUN;
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    double2* r2 = reinterpret_cast<double2*>(row);
    const int nch = nq >> 1;
    for (int j = threadIdx.x; j < nch; j += MT) {
      const int i = 2 * j, r = i / EPT, c = i - r * EPT;
      r2[j] = *reinterpret_cast<const double2*>(buf + r * RUN + c);
    }
    if ((nq & 1) && threadIdx.x == 0) {
      const int i = nq - 1, r = i / EPT;
      row[i] = buf[r * RUN + (i - r * EPT)];
    }
  } else {
    for (int i = threadIdx.x; i < nq; i += MT) {
      const int r = i / EPT;
      row[i] = buf[r * RUN + (i - r * EPT)];
    }
  }
}

// Tilted weights ta of list q -> global; breakpoints A_q = cumsum(ta) by a
// one-sync block scan, zero-weight atoms repeating their predecessor's
// breakpoint bit for bit (barycenter.py:209-222); the tilted mass; and the
// list's SS regular samples (keys (A_q[t], q, t)), taken from registers by
// the owning threads.
template <int EPT>
__device__ __forceinline__ void tilt_tail(const MotArgs& A, int b, int q, int nq, const double (&ta)[EPT],
                          double* buf, int* iscr, double* vscr, double* sbuf = nullptr,
                          bool store_ta = true) {
  const int K = A.k, n = A.n;
  const long base = ((long)b * K + q) * n;
  const int i0 = threadIdx.x * EPT;
  const bool staged = StageRun<EPT>::ON && sbuf != nullptr;
  if (staged)
    stage_put<EPT>(sbuf, ta);
  else if (store_ta)
    store_run<EPT>(A.ta + base, i0, nq, ta);
  double av[EPT];
  double loc = 0.0;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    loc += ta[e];
    av[e] = loc;
  }
  double v[1] = {loc}, tot[1];
  bops::block_scan_excl<MNW, 1>(v, tot, buf);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) av[e] = v[0] + av[e];
  int any0 = 0, lz = -1;
  double lzv = 0.0;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    const int i = i0 + e;
    if (i < nq && ta[e] == 0.0) any0 = 1;
    if (i < nq && ta[e] > 0.0) {
      lz = i;
      lzv = av[e];
    }
  }
  if (__syncthreads_or(any0)) {
    int pi = lz;
    double pv = lzv;
    excl_last_pos(pi, pv, iscr, vscr);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = i0 + e;
      if (i < nq && ta[e] == 0.0) av[e] = pi >= 0 ? pv : 0.0;
      if (i < nq && ta[e] > 0.0) {
        pi = i;
        pv = av[e];
      }
    }
  }
  if (staged) {  // both rows leave coalesced
    double* sb1 = sbuf + MT * StageRun<EPT>::RUN;
    stage_put<EPT>(sb1, av);
    __syncthreads();
    stage_out<EPT>(sbuf, A.ta + base, nq);
    stage_out<EPT>(sb1, A.A + base, nq);
  } else {
    store_run<EPT>(A.A + base, i0, nq, av);
  }
  if (threadIdx.x == 0) A.tmass[(long)b * K + q] = tot[0];
  const int ne = nq - 1, SS = A.SS;
  double* sv = A.samp + ((long)b * K + q) * SS;
  int* st = A.sampt + ((long)b * K + q) * SS;
  if (ne <= 0) {
    for (int j = threadIdx.x; j < SS; j += MT) {
      sv[j] = CUDART_INF;
      st[j] = 0;
    }
    return;
  }
  // samples t_j = floor((j+1) ne / (SS+1)) falling in [i0, i0 + EPT)
  for (int j = max(0, (int)(((long)i0 * (SS + 1)) / ne) - 1); j < SS; ++j) {
    const int t = (int)(((long)(j + 1) * ne) / (SS + 1));
    if (t >= i0 + EPT) break;
    if (t >= i0) {
      double val = 0.0;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
      for (int e = 0; e < EPT; ++e)
        if (i0 + e == t) val = av[e];
      sv[j] = val;
      st[j] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// mot_tilt: one CTA per list (no cluster).  Tilted weights, breakpoints by
// block scan, the list's tilted mass and its regular samples.

template <int EPT>
__global__ void __launch_bounds__(MT) mot_tilt(MotArgs A) {
  __shared__ __align__(16) double red[MBUF];
  __shared__ double tab[32];
  __shared__ int iscr[MNW];
  __shared__ double vscr[MNW];
  const int q = blockIdx.x, b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int nq = list_len(A, q);
  if (A.done != nullptr && A.done[b]) return;
  bops::load_exp_table(tab);
  const long base = ((long)b * K + q) * n;
  double w[EPT], ta[EPT];
  load_run<EPT>(A.a + base, threadIdx.x * EPT, nq, w);
  __syncthreads();
  if (A.mode == 0) {
    const double rq = A.omega[q] * A.rho, irq = 1.0 / rq;
    double fv[EPT];
    load_run<EPT>(A.f + base, threadIdx.x * EPT, nq, fv);
    double ex0, ex1, rtot;
    const double lamq = problem_lambda(A, b, q, ex0, ex1, rtot);
    const double mx = A.lse[((long)b * K + q) * 2 + 0];
    if (threadIdx.x == 0) {
      A.lam[(long)b * K + q] = lamq;
      if (q == 0) A.scal[b * 4 + 0] = ex1 - rtot * exp(ex0 / rtot);  // H_0, :320-327
    }
    const double sc = exp(mx - lamq * irq);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e) ta[e] = bops::wexp(w[e], -fv[e] * irq - mx, tab) * sc;
  } else {
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e) ta[e] = w[e];
  }
  tilt_tail<EPT>(A, b, q, nq, ta, red, iscr, vscr);
}

// ---------------------------------------------------------------------------
// mot_split: one CTA per problem.  Mass balance across the K inputs
// (barycenter.py:187-191, :368-370), global ranks of the K*SS regular samples
// (binary searches between the sorted per-list sample arrays), the S-1
// splitters (the samples of rank floor(s K SS / S)) and every list's split
// positions (binary searches in its breakpoints).

__device__ int merge_runs16(const double* key, uint16_t* code0, uint16_t* code1, const int* rb,
                            int K, int total);

__global__ void __launch_bounds__(ST) mot_split(MotArgs A) {
  extern __shared__ __align__(16) double ssm[];
  __shared__ double splk[SMAX + 1];
  __shared__ int splc[SMAX + 1], splr[SMAX + 1];
  __shared__ int rb[KMAX + 1];
  __shared__ int bad_s;
  const int b = blockIdx.x + A.b0;
  const int K = A.k, n = A.n, S = A.S, SS = A.SS, KSS = K * SS;
  if (A.done != nullptr && A.done[b]) return;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const double tm = lane < K ? A.tmass[(long)b * K + lane] : 0.0;
    const double mxm = warp_max(lane < K ? tm : -CUDART_INF);
    const double mnm = warp_min(lane < K ? tm : CUDART_INF);
    if (lane == 0) {
      const bool bad = (mxm - mnm) > 1e-9 * mxm;
      A.status[b] = bad ? UOT_MASS_BALANCE : 0;
      if (bad && A.done != nullptr) A.done[b] = 1;
      A.scal[b * 4 + 1] = mnm;  // common total (min)
      bad_s = bad && A.done != nullptr;
    }
  }
  for (int i = threadIdx.x; i <= K; i += ST) rb[i] = i * SS;
  int* sp = A.split + (long)b * (S + 1) * K;
  if (S == 1) {
    for (int q = threadIdx.x; q < K; q += ST) {
      sp[q] = 0;
      sp[K + q] = max(list_len(A, q) - 1, 0);
    }
    return;
  }
  // the K sorted sample lists, merged in (value, list, index) order: a
  // sample's merged position is its global rank
  double* key0 = ssm;
  uint16_t* code0 = reinterpret_cast<uint16_t*>(key0 + KSS);
  uint16_t* code1 = code0 + KSS;
  uint16_t* pos = code1 + KSS;  // merged position of sample slot q SS + j
  for (int idx = threadIdx.x; idx < KSS; idx += ST) {
    key0[idx] = A.samp[(long)b * KSS + idx];
    code0[idx] = (uint16_t)idx;
  }
  __syncthreads();
  if (bad_s) return;
  const uint16_t* mc = merge_runs16(key0, code0, code1, rb, K, KSS) ? code1 : code0;
  for (int r = threadIdx.x; r < KSS; r += ST) pos[mc[r]] = (uint16_t)r;
  // splitters: the samples of rank floor(s K SS / S)
  for (int s = 1 + threadIdx.x; s < S; s += ST) {
    const int R = (int)(((long)s * KSS) / S);
    const int slot = mc[R], q = slot / SS;
    splk[s] = key0[slot];
    splc[s] = ev_code(q, A.sampt[(long)b * KSS + slot]);
    splr[s] = R;
  }
  __syncthreads();
  // split positions: list q's samples bracket the position (merged ranks
  // below R: binary search in pos), then a short search in the breakpoints
  int top = 1;
  while (top * 2 <= SS) top *= 2;
  for (int pr = threadIdx.x; pr < (S + 1) * K; pr += ST) {
    const int s = pr / K, q = pr - s * K;
    const int ne = max(list_len(A, q) - 1, 0);
    int p;
    if (s == 0) {
      p = 0;
    } else if (s == S) {
      p = ne;
    } else {
      const int R = splr[s];
      const uint16_t* pq = pos + q * SS;
      int c = 0;  // #{j : pos(q, j) < R}
      for (int step = top; step > 0; step >>= 1)
        if (c + step <= SS && pq[c + step - 1] < R) c += step;
      const int* tq = A.sampt + (long)b * KSS + q * SS;
      // events below sample c-1's index are below the splitter, events from
      // sample c's index on are not (sample c is the splitter or after it)
      const int lo = min(c > 0 ? tq[c - 1] : 0, ne);
      const int hi = c < SS ? tq[c] : ne;
      const double* Aq = A.A + ((long)b * K + q) * n;
      const double v = splk[s];
      const int qs = ev_list(splc[s]), ts = ev_index(splc[s]);
      int l = lo, h = max(lo, min(hi, ne));
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (key_less(Aq[mid], q, mid, v, qs, ts))
          l = mid + 1;
        else
          h = mid;
      }
      p = l;
    }
    sp[(long)s * K + q] = p;
  }
}

// ---------------------------------------------------------------------------
// mot_bucket: events of one key range, sorted; cost increments.

#ifdef UOT_MOT_TIMING
// timing build only (scripts/mot_timeline.py): %globaltimer stamps of one
// thread per CTA at the phase boundaries of mot_update
__device__ unsigned long long g_mot_stamps[1 << 14][8];
__device__ __forceinline__ unsigned long long mtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MOT_STAMP(k)                                     \
  if (threadIdx.x == 0 && A.t + 2 == A.max_iters) /* the last update with a tilt */ \
  g_mot_stamps[blockIdx.y * gridDim.x + blockIdx.x][k] = mtimer()
__device__ unsigned long long g_bkt_stamps[1 << 14][6];
#define BKT_STAMP(k) \
  if (threadIdx.x == 0) g_bkt_stamps[blockIdx.y * gridDim.x + blockIdx.x][k] = mtimer()
#else
#define MOT_STAMP(k)
#define BKT_STAMP(k)
#endif

// Stable merge of the bucket's K sorted runs (run q = the events of list q,
// at [rb[q], rb[q+1])) in ceil(log2 K) pairwise rounds.  Groups of runs are
// contiguous list ranges, so on equal values the left (lower-list) group goes
// first -- exactly the (value, list, index) key order (barycenter.py:218).
// Each round is a merge path: thread t emits output positions
// [t P, (t+1) P) after one diagonal binary search per group it touches.
// Ping-pongs between the two buffers; returns the buffer holding the result.
__device__ int merge_runs(double* key0, int* code0, double* key1, int* code1, const int* rb, int K,
                          int total) {
  int cur = 0;
  const int P = (total + blockDim.x - 1) / blockDim.x;
  for (int w = 1; w < K; w <<= 1) {
    const double* ks = cur ? key1 : key0;
    const int* cs = cur ? code1 : code0;
    double* kd = cur ? key0 : key1;
    int* cd = cur ? code0 : code1;
    int o = threadIdx.x * P;
    const int oend = min(total, o + P);
    int g = 0;
    while (o < oend) {
      int r1 = rb[min(2 * w, K)];
      while (o >= r1) {
        ++g;
        r1 = rb[min((2 * g + 2) * w, K)];
      }
      const int l0 = rb[min(2 * g * w, K)], m0 = rb[min((2 * g + 1) * w, K)];
      const int nL = m0 - l0, nR = r1 - m0;
      const int d = o - l0;
      int lo = max(0, d - nR), hi = min(d, nL);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ks[l0 + mid] <= ks[m0 + d - 1 - mid])
          lo = mid + 1;
        else
          hi = mid;
      }
      int i = lo, j = d - lo;
      double lv = i < nL ? ks[l0 + i] : CUDART_INF;
      double rv = j < nR ? ks[m0 + j] : CUDART_INF;
      const int stop = min(oend, r1);
      for (; o < stop; ++o) {
        const bool takeL = lv <= rv;
        kd[o] = takeL ? lv : rv;
        cd[o] = cs[takeL ? l0 + i : m0 + j];
        if (takeL) {
          ++i;
          lv = i < nL ? ks[l0 + i] : CUDART_INF;
        } else {
          ++j;
          rv = j < nR ? ks[m0 + j] : CUDART_INF;
        }
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

// Gathers the events of range s from all K lists into shared memory and
// merges them; key/code point at the merged buffer on return.
__device__ __forceinline__ int bucket_gather(const MotArgs& A, int b, int s, double* buf,
                                             double*& key, int*& code, int* lo_s, int* cnt_s) {
  const int K = A.k, n = A.n;
  const int* sp = A.split + (long)b * (A.S + 1) * K;
  if (threadIdx.x < 32) {  // lane q: list q's range, offsets by a warp scan
    const int lane = threadIdx.x;
    const int lo = lane < K ? sp[(long)s * K + lane] : 0;
    const int len = lane < K ? sp[(long)(s + 1) * K + lane] - lo : 0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane < K) {
      lo_s[lane] = lo;
      cnt_s[lane] = incl - len;
    }
    if (lane == K - 1) cnt_s[K] = incl;
  }
  __syncthreads();
  const int total = cnt_s[K];
  const int cap = A.cap;
  if (total > cap) return -1;
  double* key0 = buf;
  double* key1 = buf + cap;
  int* code0 = reinterpret_cast<int*>(buf + 2 * cap);
  int* code1 = code0 + cap;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int q = 0, hi = K - 1;  // last run starting at or before e
    while (q < hi) {
      const int mid = (q + hi + 1) >> 1;
      if (cnt_s[mid] <= e)
        q = mid;
      else
        hi = mid - 1;
    }
    const int t = lo_s[q] + (e - cnt_s[q]);
    key0[e] = A.A[((long)b * K + q) * n + t];
    code0[e] = ev_code(q, t);
  }
  __syncthreads();
  const int which = merge_runs(key0, code0, key1, code1, cnt_s, K, total);
  key = which ? key1 : key0;
  code = which ? code1 : code0;
  return total;
}

// Stable pairwise merge rounds of the bucket's K sorted runs, moving each
// event's key with a 16-bit code (its gather position: the run layout is the
// lists' ranges concatenated in list order, so the position identifies list
// and index).  Same merge path and tie rule as merge_runs.
__device__ int merge_runs16(const double* key, uint16_t* code0, uint16_t* code1, const int* rb,
                            int K, int total) {
  // codes are gather positions; keys are read through them (key[code])
  int cur = 0;
  const int P = (total + blockDim.x - 1) / blockDim.x;
  for (int w = 1; w < K; w <<= 1) {
    const uint16_t* cs = cur ? code1 : code0;
    uint16_t* cd = cur ? code0 : code1;
    int o = threadIdx.x * P;
    const int oend = min(total, o + P);
    int g = 0;
    while (o < oend) {
      int r1 = rb[min(2 * w, K)];
      while (o >= r1) {
        ++g;
        r1 = rb[min((2 * g + 2) * w, K)];
      }
      const int l0 = rb[min(2 * g * w, K)], m0 = rb[min((2 * g + 1) * w, K)];
      const int nL = m0 - l0, nR = r1 - m0;
      const int d = o - l0;
      int lo = max(0, d - nR), hi = min(d, nL);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key[cs[l0 + mid]] <= key[cs[m0 + d - 1 - mid]])
          lo = mid + 1;
        else
          hi = mid;
      }
      int il = l0 + lo, ir = m0 + (d - lo);
      uint16_t lc = cs[min(il, total - 1)], rc = cs[min(ir, total - 1)];
      double lv = il < m0 ? key[lc] : CUDART_INF;
      double rv = ir < r1 ? key[rc] : CUDART_INF;
      const int stop = min(oend, r1);
      for (; o < stop; ++o) {
        const bool takeL = lv <= rv;
        cd[o] = takeL ? lc : rc;
        il += takeL;
        ir += !takeL;
        const int ni = takeL ? il : ir;
        const bool in = takeL ? (il < m0) : (ir < r1);
        const uint16_t nc = cs[min(ni, total - 1)];
        const double nv = in ? key[nc] : CUDART_INF;
        lv = takeL ? nv : lv;
        lc = takeL ? nc : lc;
        rv = takeL ? rv : nv;
        rc = takeL ? rc : nc;
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

// Bucket sort of the gathered events by value (one bin per two events on
// average, bins by linear interpolation between the smallest and largest key
// -- monotone, so bin order is key order), then an insertion sort of every
// bin by (value, gather position); the gather layout is (list, index) order,
// so the result is exactly the (value, list, index) merge of merge_runs16.
// Counting and scattering use shared-memory atomics (the order inside a bin
// before its sort is irrelevant: the key order is total).  Returns 1 with the
// result in key1 / code1, or 0 when a bin would hold more than BINMAX events
// (heavily tied or clustered keys): the caller then merges instead.
constexpr int BINMAX = 64;

// Fast path (total <= BIN_EV events per thread, the cfg5 regime): one bin per
// event on average, two 16-bit counters packed per word (same buffer as the
// coarse path); the counting atomic's return value is the event's arrival
// rank in its bin, so the scatter needs no second atomic pass, and most bins
// hold one event, so little is left for the insertion sort.
constexpr int BIN_EV = 8;

__device__ __forceinline__ int bin_get(const int* binc, int i) {
  return (binc[i >> 1] >> ((i & 1) * 16)) & 0xffff;
}

__device__ int bin_sort_fine(const double* key0, uint16_t* code1, int* binc, int total, double kmin,
                             double span, int* over_s, int* wsum) {
  const int tid = threadIdx.x, bd = blockDim.x;
  const int NB = total;
  for (int i = tid; i < ((NB + 1) >> 1); i += bd) binc[i] = 0;
  __syncthreads();
  const double scale = (double)NB / span;
  int bi_r[BIN_EV], rk_r[BIN_EV];
#pragma unroll
  for (int u = 0; u < BIN_EV; ++u) {
    const int e = tid + u * bd;
    bi_r[u] = 0;
    rk_r[u] = 0;
    if (e < total) {
      const int bi = min(NB - 1, (int)((key0[e] - kmin) * scale));
      const int sh = (bi & 1) * 16;
      const int old = atomicAdd(&binc[bi >> 1], 1 << sh);
      bi_r[u] = bi;
      rk_r[u] = (old >> sh) & 0xffff;
    }
  }
  __syncthreads();
  // exclusive scan of the bin counts: an even number of bins per thread, so no
  // two threads share a packed word
  const int per = (((NB + bd - 1) / bd) + 1) & ~1;
  const int b0 = min(NB, tid * per), b1 = min(NB, b0 + per);
  int loc = 0, big = 0;
  for (int i = b0; i < b1; ++i) {
    const int c = bin_get(binc, i);
    loc += c;
    big = max(big, c);
  }
  if (big > BINMAX) *over_s = 1;
  const int lane = tid & 31, warp = tid >> 5;
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (*over_s) return 0;
  int off = incl - loc;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  for (int i = b0; i < b1; i += 2) {  // counts -> starts, a packed word at a time
    const int wv = binc[i >> 1];
    const int c0 = wv & 0xffff, c1 = (wv >> 16) & 0xffff;
    binc[i >> 1] = off | ((off + c0) << 16);
    off += c0 + c1;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BIN_EV; ++u) {
    const int e = tid + u * bd;
    if (e < total) code1[bin_get(binc, bi_r[u]) + rk_r[u]] = (uint16_t)e;
  }
  __syncthreads();
  // insertion sort of every bin by (key, gather position)
  for (int i = tid; i < NB; i += bd) {
    const int st = bin_get(binc, i), en = i + 1 < NB ? bin_get(binc, i + 1) : total;
    for (int a = st + 1; a < en; ++a) {
      const uint16_t c = code1[a];
      const double k = key0[c];
      int j = a - 1;
      while (j >= st) {
        const uint16_t cj = code1[j];
        const double kj = key0[cj];
        if (!(kj > k || (kj == k && cj > c))) break;
        code1[j + 1] = cj;
        --j;
      }
      code1[j + 1] = c;
    }
  }
  __syncthreads();
  return 1;
}

__device__ int bin_sort(const double* key0, uint16_t* code1, int* binc, const int* rb, int K,
                        int total, bool bin_coarse) {
  __shared__ double kmin_s, kmax_s;
  __shared__ int over_s;
  const int tid = threadIdx.x;
  if (tid < 32) {
    double mn = CUDART_INF, mx = -CUDART_INF;
    if (tid < K && rb[tid + 1] > rb[tid]) {
      mn = key0[rb[tid]];
      mx = key0[rb[tid + 1] - 1];
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (tid == 0) {
      kmin_s = mn;
      kmax_s = mx;
      over_s = 0;
    }
  }
  __shared__ int wsum[32];
  if (total <= BIN_EV * (int)blockDim.x && total < 65536 && !bin_coarse) {
    __syncthreads();
    const double kmin = kmin_s, span = kmax_s - kmin_s;
    if (!(span > 0.0)) return 0;
    return bin_sort_fine(key0, code1, binc, total, kmin, span, &over_s, wsum);
  }
  const int NB = max(1, total >> 1);
  for (int i = tid; i < NB; i += blockDim.x) binc[i] = 0;
  __syncthreads();
  const double kmin = kmin_s, span = kmax_s - kmin_s;
  if (!(span > 0.0)) return 0;
  const double scale = (double)NB / span;
  for (int e = tid; e < total; e += blockDim.x) {
    const int bi = min(NB - 1, (int)((key0[e] - kmin) * scale));
    atomicAdd(&binc[bi], 1);
  }
  __syncthreads();
  // exclusive scan of the bin counts (contiguous chunk per thread) + overflow check
  const int per = (NB + blockDim.x - 1) / blockDim.x;
  const int b0 = tid * per, b1 = min(NB, b0 + per);
  int loc = 0, big = 0;
  for (int i = b0; i < b1; ++i) {
    loc += binc[i];
    big = max(big, binc[i]);
  }
  if (big > BINMAX) over_s = 1;
  const int lane = tid & 31, warp = tid >> 5;
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (over_s) return 0;
  int off = incl - loc;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  for (int i = b0; i < b1; ++i) {
    const int c = binc[i];
    binc[i] = off;
    off += c;
  }
  __syncthreads();
  for (int e = tid; e < total; e += blockDim.x) {
    const int bi = min(NB - 1, (int)((key0[e] - kmin) * scale));
    code1[atomicAdd(&binc[bi], 1)] = (uint16_t)e;
  }
  __syncthreads();
  // binc[i] is now the end of bin i; insertion sort by (key, gather position)
  for (int i = tid; i < NB; i += blockDim.x) {
    const int st = i == 0 ? 0 : binc[i - 1], en = binc[i];
    for (int a = st + 1; a < en; ++a) {
      const uint16_t c = code1[a];
      const double k = key0[c];
      int j = a - 1;
      while (j >= st) {
        const uint16_t cj = code1[j];
        const double kj = key0[cj];
        if (!(kj > k || (kj == k && cj > c))) break;
        code1[j + 1] = cj;
        --j;
      }
      code1[j + 1] = c;
    }
  }
  __syncthreads();
  return 1;
}

// Shared memory of one mot_bucket CTA: two key buffers, the supports of the
// ranges (one more per list), two code buffers and the position -> list table.
__host__ __device__ __forceinline__ size_t bucket_smem_bytes(int cap, int k) {
  return (size_t)cap * (2 * sizeof(double) + 2 * sizeof(uint16_t) + 1) + (size_t)k * sizeof(double) +
         16 + (size_t)(cap / 2 + 2) * sizeof(int);
}

// mot_bucket: the events of key range s of problem b, merged in shared
// memory, and their cost increments.  Gather: the lists' ranges (keys, and
// the supports x_q[lo_q .. hi_q]) concatenated in list order, one warp per
// list (coalesced).
// After the merge every thread owns a contiguous run of sorted events: the
// barycentre before each event is bstart + an exclusive scan of the
// increments w_q (x_q[t+1] - x_q[t]), and dCc = inc (x_q[t+1] + x_q[t] - Bb -
// Ba) (barycenter.py:223-229) lands at the event's gather position, so each
// list's increments leave with coalesced stores.
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
// all but the most recent committed group have landed
__device__ __forceinline__ void cp_async_wait_but_last() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

__global__ void __launch_bounds__(BT2) mot_bucket(MotArgs A) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ int lo_s[KMAX + 1], cnt_s[KMAX + 1];
  __shared__ double om_s[KMAX];
  __shared__ double scr[32];
  __shared__ double bstart_s;
  __shared__ int done_s;
  BKT_STAMP(0);
  const int s = blockIdx.x, b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n, cap = A.cap;
  const int* sp = A.split + (long)b * (A.S + 1) * K;
  if (threadIdx.x < 32) {  // lane q: list q's range, offsets by a warp scan (one latency)
    const int lane = threadIdx.x;
    const int dn = (lane == 0 && A.done != nullptr) ? A.done[b] : 0;
    const int lo = lane < K ? sp[(long)s * K + lane] : 0;
    const int len = lane < K ? sp[(long)(s + 1) * K + lane] - lo : 0;
    const double om = lane < K ? A.omega[lane] : 0.0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane < K) {
      lo_s[lane] = lo;
      cnt_s[lane] = incl - len;
      om_s[lane] = om;
    }
    if (lane == K - 1) cnt_s[K] = incl;
    if (lane == 0) done_s = dn;
  }
  __syncthreads();
  if (done_s) return;
  const int total = cnt_s[K];
  if (total > cap) {  // excluded by bucket_bound; kept as a guard
    if (threadIdx.x == 0) A.status[b] = UOT_INVALID;
    return;
  }
  if (total == 0) return;
  double* key0 = bsm;
  double* xs = bsm + cap;  // list q's supports at [cnt_q + q, cnt_{q+1} + q]
  uint16_t* c0 = reinterpret_cast<uint16_t*>(xs + cap + K);
  uint16_t* c1 = c0 + cap;
  uint8_t* qt = reinterpret_cast<uint8_t*>(c1 + cap);
  const long rowb = (long)b * K * n;
  {  // warp w gathers lists w, w + NW, ...: keys and supports by cp.async (all
     // loads in flight at once), codes and list tags
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = BT2 / 32;
    for (int q = warp; q < K; q += NW) {
      const int c = cnt_s[q], len = cnt_s[q + 1] - c;
      const double* Aq = A.A + rowb + (long)q * n + lo_s[q];
      const double* xq = A.x + rowb + (long)q * n + lo_s[q];
      double* xd = xs + c + q;
      for (int j = lane; j < len; j += 32) {
        cp_async8(key0 + c + j, Aq + j);
        cp_async8(xd + j, xq + j);
        c0[c + j] = (uint16_t)(c + j);
        qt[c + j] = (uint8_t)q;
      }
      if (lane == 0) cp_async8(xd + len, xq + len);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // barycentre of the tuple before the range: idx_q = lo_q
    const int lane = threadIdx.x;
    const double bs = warp_sum(lane < K ? om_s[lane] * xs[cnt_s[lane] + lane] : 0.0);
    if (lane == 0) bstart_s = bs;
  }
  BKT_STAMP(1);
  int* binc = reinterpret_cast<int*>(
      (reinterpret_cast<uintptr_t>(qt + cap) + 15) & ~static_cast<uintptr_t>(15));
  const uint16_t* code = c1;
  if (A.no_bin == 1 || !bin_sort(key0, c1, binc, cnt_s, K, total, A.no_bin == 2))
    code = merge_runs16(key0, c0, c1, cnt_s, K, total) ? c1 : c0;
  BKT_STAMP(2);
  const int per = (total + BT2 - 1) / BT2;
  const int e0 = threadIdx.x * per, e1 = min(total, e0 + per);
  double loc = 0.0;
  for (int e = e0; e < e1; ++e) {
    const int g = code[e], q = qt[g];
    loc += om_s[q] * (xs[g + q + 1] - xs[g + q]);
  }
  double tot;
  double run = bscan1(loc, tot, scr) + bstart_s;
  double* out = key0;  // keys are dead after the merge: dCc by gather position
  for (int e = e0; e < e1; ++e) {
    const int g = code[e], q = qt[g];
    const double xo = xs[g + q], xn = xs[g + q + 1];
    const double inc = om_s[q] * (xn - xo);
    const double bb = run, ba = bb + inc;
    out[g] = inc * (xn + xo - bb - ba);
    run += inc;
  }
  __syncthreads();
  BKT_STAMP(3);
  for (int e = threadIdx.x; e < total; e += BT2) {
    const int q = qt[e];
    A.dcc[rowb + (long)q * n + lo_s[q] + (e - cnt_s[q]) + 1] = out[e];
  }
  BKT_STAMP(4);
}

// ---------------------------------------------------------------------------
// mot_update: dual atoms, gaps, line search, update (cluster of K CTAs).



template <int EPT>
__global__ void __launch_bounds__(MT) mot_update(MotArgs A) {
  MOT_STAMP(0);
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double stg[];  // 2 staging buffers (StageRun)
  __shared__ double scr[32 * 8];
  __shared__ __align__(16) double red[2 * MBUF];
  __shared__ double tab[32];
  __shared__ double slots[32];
  __shared__ int done_s;
  __shared__ double cc0_s;
  __shared__ int iscr[MNW];
  __shared__ double vscr[MNW];
  const int q = (int)cl.block_rank();
  const int b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int nq = list_len(A, q);
  int parity = 0;
  bops::Ping<MBUF> ping{red, 0};
  bops::load_exp_table(tab);
  if (threadIdx.x == 0) done_s = (A.done != nullptr) ? A.done[b] : 0;
  __syncthreads();
  if (done_s) return;
  const long base = ((long)b * K + q) * n;
  // Issue every per-list load up front (cost increments, potentials, tilted
  // and input weights) so their latencies overlap each other and the scan.
  double rv[EPT], fv[EPT], tv[EPT], wv[EPT];
  double loc = 0.0;
  if constexpr (StageRun<EPT>::ON) {
    // two rounds of two coalesced rows through the staging buffers
    double* b0 = stg;
    double* b1 = stg + MT * StageRun<EPT>::RUN;
    stage_store<EPT>(b0, A.dcc + base, nq);
    if (A.mode != 1) stage_store<EPT>(b1, A.f + base, nq);
    __syncthreads();
    stage_load<EPT>(b0, nq, rv);
    if (A.mode != 1) stage_load<EPT>(b1, nq, fv);
    __syncthreads();
    if (A.mode != 1) {
      stage_store<EPT>(b0, A.ta + base, nq);
      stage_store<EPT>(b1, A.a + base, nq);
      __syncthreads();
      stage_load<EPT>(b0, nq, tv);
      stage_load<EPT>(b1, nq, wv);
    }
  } else {
    load_run<EPT>(A.dcc + base, threadIdx.x * EPT, nq, rv);
    if (A.mode != 1) {
      load_run<EPT>(A.f + base, threadIdx.x * EPT, nq, fv);
      load_run<EPT>(A.ta + base, threadIdx.x * EPT, nq, tv);
      load_run<EPT>(A.a + base, threadIdx.x * EPT, nq, wv);
    }
  }
  MOT_STAMP(1);
  // initial potential: f_1[0] = Cc(first tuple), f_k[0] = 0 (barycenter.py:206-207)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double c = 0.0;
    if (q == 0) {
      const double x0 = lane < K ? A.x[((long)b * K + lane) * n] : 0.0;
      const double om = lane < K ? A.omega[lane] : 0.0;
      const double bb = warp_sum(om * x0);
      c = warp_sum(om * ((x0 - bb) * (x0 - bb)));
    }
    if (lane == 0) cc0_s = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) rv[0] = 0.0;  // dcc[0] is not an event
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    loc += rv[e];
    rv[e] = loc;
  }
  double tot;
  const double off = bscan1(loc, tot, scr) + cc0_s;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) rv[e] += off;

  if (A.mode == 1) {  // balanced sweep: the duals are the output
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e) {
      const int i = threadIdx.x * EPT + e;
      if (i < nq) A.out_f[base + i] = rv[e];
    }
    return;
  }
  const double rq = A.omega[q] * A.rho;
  const double lamq = A.lam[(long)b * K + q];
  const double irq = 1.0 / rq;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  double mxs[2] = {-CUDART_INF, -CUDART_INF};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    const double d = rv[e] - fv[e];
    acc[0] += tv[e] * d;                 // fw_gap part (barycenter.py:376-381)
    acc[1] += tv[e] * rv[e];             // plan cost via complementary slackness
    if (tv[e] > 0.0) acc[2] += tv[e] * (-(fv[e] + lamq) * irq);  // sum ta log(ta/a)
    acc[3] += tv[e];                     // tilted mass
    acc[4] += wv[e];                     // input mass
    acc[5] += tv[e] * d;                 // first moment of d under p_0
    acc[6] += tv[e] * d * d;             // second moment
    if (wv[e] > 0.0) {
      mxs[0] = bops::dmax(mxs[0], -fv[e] * irq);
      mxs[1] = bops::dmax(mxs[1], -rv[e] * irq);
    }
  }
  bops::block_red<MNW, 7, 2>(acc, mxs, ping.next());
  MOT_STAMP(2);
  // cluster sums: fw_gap, plan cost + rho KL terms, sum of centres
  const double cq = acc[5] / acc[3];
  // (the line search's starting curvature rides along: one cluster barrier
  // instead of two)
  double cs[4] = {acc[0], acc[1] + rq * (acc[2] - acc[3] + acc[4]), cq,
                  fmax(acc[6] / acc[3] - cq * cq, 0.0) / rq};
  cluster_sum<4>(cs, slots, parity);
  const double fw_gap = cs[0];
  const double primal = cs[1];
  const double dual = A.scal[b * 4 + 0];
  const double pd_gap = primal - dual;
  const int t = A.t;
  if (q == 0 && threadIdx.x == 0) {
    A.h0[(long)b * A.max_iters + t] = dual;
    A.fw_gap[(long)b * A.max_iters + t] = fw_gap;
    A.pd_gap[(long)b * A.max_iters + t] = pd_gap;
    A.iterations[b] = t + 1;
    A.summary[b * 2 + 0] = primal;
    A.summary[b * 2 + 1] = dual;
  }
  MOT_STAMP(3);
  const bool stop = A.early_exit && pd_gap < A.gap_tol;  // barycenter.py:394-396
  if (stop) {
    if (q == 0 && threadIdx.x == 0) A.done[b] = 2;  // converged (plan of this iteration kept)
    cl.sync();
    return;
  }
  double gam;
  if (A.step_in != nullptr) {
    gam = __ldg(A.step_in + (long)b * A.max_iters + t);  // replayed gamma_t
  } else if (A.step == UOT_STEP_HARMONIC) {
    gam = 2.0 / (2.0 + t);
  } else {
    // minimise Phi(gamma) = sum_k rho_k LSE_{a_k}(-(f_k + gamma d_k)/rho_k):
    // Phi' = -sum_k E_k[d_k], Phi'' = sum_k Var_k[d_k] / rho_k; moments are
    // centred at the gamma = 0 means (translation invariance, see fw1d.cu).
    const double k0 = -cs[2];
    const double vs[1] = {cs[3]};
    if (!(k0 < 0.0)) {
      gam = 0.0;
    } else {
      double lo = 0.0, hi = 1.0;
      gam = vs[0] > 0.0 ? fmin(1.0, -k0 / vs[0]) : 1.0;
#ifdef UOT_NEWTON_STATS
      if (threadIdx.x == 0 && q == 0) atomicAdd(&g_mot_stats[1], 1ull);
#endif
      for (int it = 0; it < 24; ++it) {
        const double sh = (1.0 - gam) * mxs[0] + gam * mxs[1];
        double mom[3] = {0.0, 0.0, 0.0};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
        for (int e = 0; e < EPT; ++e) {
          const double d = rv[e] - fv[e];
          const double ww = bops::wexp(wv[e], -(fv[e] + gam * d) * irq - sh, tab);
          const double xc = d - cq;
          mom[0] += ww;
          mom[1] += ww * xc;
          mom[2] += ww * xc * xc;
        }
        bops::block_sum<MNW, 3>(mom, ping.next());
#ifdef UOT_NEWTON_STATS
        if (threadIdx.x == 0 && q == 0) atomicAdd(&g_mot_stats[0], 1ull);
#endif
        const double e1 = mom[1] / mom[0];
        double gv[2] = {e1, (mom[2] / mom[0] - e1 * e1) / rq};
        cluster_sum<2>(gv, slots, parity);
        const double g1 = k0 - gv[0], g2 = gv[1];
        if (g1 < 0.0)
          lo = gam;
        else
          hi = gam;
        if (gam >= 1.0 && g1 <= 0.0) {
          gam = 1.0;
          break;
        }
        double nxt = g2 > 0.0 ? gam - g1 / g2 : 0.5 * (lo + hi);
        const bool newton = nxt > lo && nxt < hi;
        if (!newton) nxt = 0.5 * (lo + hi);
        const bool conv = (newton && fabs(nxt - gam) <= 1e-9 * fmax(1.0, gam)) || g1 == 0.0 ||
                          hi - lo <= 1e-15;
        gam = nxt;
        if (conv) break;
      }
    }
  }
  // barycenter.py:409-411, rounded as numpy rounds it (two products, a sum)
  const double omg = 1.0 - gam;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) fv[e] = __dadd_rn(__dmul_rn(omg, fv[e]), __dmul_rn(gam, rv[e]));
  MOT_STAMP(4);
  if constexpr (StageRun<EPT>::ON) {  // coalesced: the stage buffer is free here
    stage_put<EPT>(stg, fv);
    __syncthreads();
    stage_out<EPT>(stg, A.f + base, nq);  // list_lse's barriers order the reuse below
  } else {
    store_run<EPT>(A.f + base, threadIdx.x * EPT, nq, fv);
  }
  {  // log-sum-exp of the new iterate for the next tilt / the final translation
    double mx, qk;
    double* r0 = ping.next();
    double* r1 = ping.next();
    list_lse<EPT>(wv, fv, irq, tab, r0, r1, mx, qk, tv);  // tv <- w exp(-f/rho - mx)
    MOT_STAMP(5);
    if (threadIdx.x == 0) {
      A.lse[((long)b * K + q) * 2 + 0] = mx;
      A.lse[((long)b * K + q) * 2 + 1] = qk;
    }
    if (t + 1 < A.max_iters) {
      // the next iteration's tilt, fused: lambda from the cluster's
      // log-sum-exps (barycenter.py:316-317), H_0 (:320-327), breakpoints.
      double ex[3] = {rq * qk, rq * acc[4], rq};
      cluster_sum<3>(ex, slots, parity);
      const double lam1 = rq * qk - (rq / ex[2]) * ex[0];
      if (threadIdx.x == 0) {
        A.lam[(long)b * K + q] = lam1;
        if (q == 0) A.scal[b * 4 + 0] = ex[1] - ex[2] * exp(ex[0] / ex[2]);
      }
      const double sc = exp(mx - lam1 * irq);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
      for (int e = 0; e < EPT; ++e) tv[e] *= sc;
      tilt_tail<EPT>(A, b, q, nq, tv, ping.next(), iscr, vscr,
                     StageRun<EPT>::ON ? stg : nullptr);
    }
    MOT_STAMP(6);
  }
  cl.sync();  // slots stay valid until every CTA read them
  MOT_STAMP(7);
}

// ---------------------------------------------------------------------------
// mot_update2: the same update with TWO lists per CTA (clusters of K/2 CTAs),
// so twice as many problems are co-resident as with one 16-CTA cluster per
// problem (16-CTA clusters of 512-thread CTAs: at most 7 in flight).  List A
// (2c) lives in registers exactly as in mot_update; list B (2c+1) keeps its
// rows (dual atoms, potentials, input weights) in shared memory, staged by
// cp.async in a swizzled run layout (thread t's 16-byte chunk c of a row at
// t EPT + 2 (c ^ sw(t)): conflict-free per-thread vector reads, coalesced
// fills).  Per-list reductions are formed per list as before; cluster sums
// read list l's value in lane l, in the same order as cluster_sum.

template <int EPT>
struct Swz {
  static constexpr int PAIRS = EPT / 2;
  __device__ static __forceinline__ int chunk(int t, int c) {
    if constexpr (PAIRS >= 8) return c ^ (t & 7);
    else if constexpr (PAIRS == 4) return c ^ ((t >> 1) & 3);
    else if constexpr (PAIRS == 2) return c ^ ((t >> 2) & 1);
    else return c;
  }
  __device__ static __forceinline__ double2* at(double* row, int t, int c) {
    return reinterpret_cast<double2*>(row + t * EPT + 2 * chunk(t, c));
  }
  __device__ static __forceinline__ const double2* at(const double* row, int t, int c) {
    return reinterpret_cast<const double2*>(row + t * EPT + 2 * chunk(t, c));
  }
  // global row (16-byte aligned, nq valid entries) -> swizzled shared row, async
  __device__ static __forceinline__ void fill(double* srow, const double* grow, int nq) {
    if ((reinterpret_cast<uintptr_t>(grow) & 15) != 0) {  // odd row stride: 8-byte copies
      for (int i = threadIdx.x; i < MT * EPT; i += MT) {
        const int t = i / EPT, e = i - t * EPT;
        double* dst = reinterpret_cast<double*>(at(srow, t, e >> 1)) + (e & 1);
        *dst = i < nq ? grow[i] : 0.0;
      }
      return;
    }
    for (int j = threadIdx.x; j < MT * PAIRS; j += MT) {
      const int t = j / PAIRS, c = j - t * PAIRS;
      const int rem = nq - 2 * j;
      const int bytes = rem >= 2 ? 16 : rem == 1 ? 8 : 0;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(at(srow, t, c));
      const double* src = bytes > 0 ? grow + 2 * j : grow;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                   "r"(bytes));
    }
  }
  // swizzled shared row -> global row (coalesced)
  __device__ static __forceinline__ void drain(const double* srow, double* grow, int nq) {
    if ((reinterpret_cast<uintptr_t>(grow) & 15) != 0) {
      for (int i = threadIdx.x; i < nq; i += MT) {
        const int t = i / EPT, e = i - t * EPT;
        grow[i] = reinterpret_cast<const double*>(at(srow, t, e >> 1))[e & 1];
      }
      return;
    }
    for (int j = threadIdx.x; j < MT * PAIRS && 2 * j < nq; j += MT) {
      const int t = j / PAIRS, c = j - t * PAIRS;
      const double2 v = *at(srow, t, c);
      if (2 * j + 1 < nq)
        *reinterpret_cast<double2*>(grow + 2 * j) = v;
      else
        grow[2 * j] = v.x;
    }
  }
};


// Cluster all-reduce over the K lists of a two-lists-per-CTA cluster: CTA c
// publishes (list 2c, list 2c+1); lane l reads list l; butterfly over the warp.
template <int NV>
__device__ __forceinline__ void cluster_sum2(double (&va)[NV], const double (&vb)[NV],
                                             double* slots, int& parity, int K) {
  static_assert(NV <= 8, "cluster_sum2: NV <= 8");
  cg::cluster_group cl = cg::this_cluster();
  double* mine = slots + parity * 16;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      mine[k] = va[k];
      mine[8 + k] = vb[k];
    }
  }
  cl.sync();
  const int lane = threadIdx.x & 31;
  const bool act = lane < K;
  const double* other = cl.map_shared_rank(mine, act ? (lane >> 1) : 0);
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = act ? other[(lane & 1) * 8 + k] : 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) va[k] = warp_sum(v[k]);
  parity ^= 1;
}

template <int EPT>
constexpr size_t upd2_smem() {
  return 3 * (size_t)MT * EPT * sizeof(double);
}

// tilt_tail for a list whose row sits in shared memory (swizzled, holding
// w exp(-f/rho - mx)): scaled in place to the tilted weights, then turned in
// place into the breakpoints with tilt_tail's association (local prefix,
// plus the block offset) and zero-weight fix-up; the row leaves coalesced.
template <int EPT>
__device__ __forceinline__ void tilt_tail_smem(const MotArgs& A, int b, int q, int nq, double* row,
                                               double scale, double* buf, int* iscr,
                                               double* vscr) {
  using SW = Swz<EPT>;
  constexpr int PAIRS = EPT / 2;
  const int K = A.k, n = A.n, tid = threadIdx.x;
  const int i0 = tid * EPT;
  double loc = 0.0;
#pragma unroll 2
  for (int cc = 0; cc < PAIRS; ++cc) {
    double2* p = SW::at(row, tid, cc);
    double2 v = *p;
    v.x *= scale;
    v.y *= scale;
    *p = v;
    loc += v.x;
    loc += v.y;
  }
  double v1[1] = {loc}, tot[1];
  bops::block_scan_excl<MNW, 1>(v1, tot, buf);
  const double off = v1[0];
  int any0 = 0, lz = -1;
  double lzv = 0.0;
  loc = 0.0;
#pragma unroll 2
  for (int cc = 0; cc < PAIRS; ++cc) {
    double2* p = SW::at(row, tid, cc);
    const double2 t2 = *p;
    double2 a2;
    loc += t2.x;
    a2.x = off + loc;
    loc += t2.y;
    a2.y = off + loc;
    const int i = i0 + 2 * cc;
    if (i < nq && t2.x == 0.0) any0 = 1;
    if (i < nq && t2.x > 0.0) {
      lz = i;
      lzv = a2.x;
    }
    if (i + 1 < nq && t2.y == 0.0) any0 = 1;
    if (i + 1 < nq && t2.y > 0.0) {
      lz = i + 1;
      lzv = a2.y;
    }
    // zero-weight atoms are marked by a negative value (breakpoints are >= 0)
    // until the fix-up below gives them their predecessor's breakpoint
    *p = make_double2(t2.x == 0.0 ? -a2.x - 1.0 : a2.x, t2.y == 0.0 ? -a2.y - 1.0 : a2.y);
  }
  if (__syncthreads_or(any0)) {
    int pi = lz;
    double pv = lzv;
    excl_last_pos(pi, pv, iscr, vscr);
#pragma unroll 1
    for (int cc = 0; cc < PAIRS; ++cc) {
      double2* p = SW::at(row, tid, cc);
      double2 a2 = *p;
      const int i = i0 + 2 * cc;
      if (i < nq && a2.x < 0.0) a2.x = pi >= 0 ? pv : 0.0;
      else if (i < nq) { pi = i; pv = a2.x; }
      if (i + 1 < nq && a2.y < 0.0) a2.y = pi >= 0 ? pv : 0.0;
      else if (i + 1 < nq) { pi = i + 1; pv = a2.y; }
      *p = a2;
    }
  }
  __syncthreads();
  const long base = ((long)b * K + q) * n;
  SW::drain(row, A.A + base, nq);
  if (tid == 0) A.tmass[(long)b * K + q] = tot[0];
  const int ne = nq - 1, SS = A.SS;
  double* sv = A.samp + ((long)b * K + q) * SS;
  int* st = A.sampt + ((long)b * K + q) * SS;
  if (ne <= 0) {
    for (int j = tid; j < SS; j += MT) {
      sv[j] = CUDART_INF;
      st[j] = 0;
    }
    return;
  }
  for (int j = tid; j < SS; j += MT) {  // samples t_j = floor((j+1) ne / (SS+1))
    const int t = (int)(((long)(j + 1) * ne) / (SS + 1));
    const int th = t / EPT, e = t - th * EPT;
    const double2 a2 = *SW::at(row, th, e >> 1);
    sv[j] = (e & 1) ? a2.y : a2.x;
    st[j] = t;
  }
}

template <int EPT>
__global__ void __launch_bounds__(MT, 1) mot_update2(MotArgs A) {
  MOT_STAMP(0);
  using SW = Swz<EPT>;
  constexpr int PAIRS = EPT / 2;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double rows[];  // list B: r (dcc first), f, w
  constexpr int RBUF = 8 * MNW;  // the 6 + 2 gap reductions are the widest
  __shared__ __align__(16) double red[2 * RBUF];
  __shared__ double tab[32];
  __shared__ double slots[32];
  __shared__ int done_s;
  __shared__ double cc0_s;
  __shared__ int iscr[MNW];
  __shared__ double vscr[MNW];
  const int c = (int)cl.block_rank();
  const int b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int qa = 2 * c;
  const bool hasB = 2 * c + 1 < K;  // odd K: the last CTA holds one list
  const int qb = hasB ? 2 * c + 1 : qa;
  const int na = list_len(A, qa), nb = hasB ? list_len(A, qb) : 0;
  const int tid = threadIdx.x, i0 = tid * EPT;
  int parity = 0;
  bops::Ping<RBUF> ping{red, 0};
  bops::load_exp_table(tab);
  if (tid == 0) done_s = (A.done != nullptr) ? A.done[b] : 0;
  __syncthreads();
  if (done_s) return;
  const long basea = ((long)b * K + qa) * n, baseb = ((long)b * K + qb) * n;
  double* rB = rows;
  double* fB = rows + MT * EPT;
  double* wB = rows + 2 * MT * EPT;
  SW::fill(rB, A.dcc + baseb, nb);
  cp_async_commit();  // the increments first: the prefix scan starts while f and w are in flight
  SW::fill(fB, A.f + baseb, nb);
  SW::fill(wB, A.a + baseb, nb);
  cp_async_commit();
  double rv[EPT], fv[EPT], wv[EPT];
  load_run<EPT>(A.dcc + basea, i0, na, rv);
  load_run<EPT>(A.f + basea, i0, na, fv);
  load_run<EPT>(A.a + basea, i0, na, wv);
  if (tid < 32) {  // f_1[0] = Cc(first tuple) (barycenter.py:206-207); list 0 is list A of CTA 0
    const int lane = tid;
    double cc = 0.0;
    if (c == 0) {
      const double x0 = lane < K ? A.x[((long)b * K + lane) * n] : 0.0;
      const double om = lane < K ? A.omega[lane] : 0.0;
      const double bb = warp_sum(om * x0);
      cc = warp_sum(om * ((x0 - bb) * (x0 - bb)));
    }
    if (lane == 0) cc0_s = cc;
  }
  cp_async_wait_but_last();
  __syncthreads();
  MOT_STAMP(1);
  // dual atoms: prefix sums of the cost increments (dcc[0] is not an event)
  if (tid == 0) rv[0] = 0.0;
  double sc2[2] = {0.0, 0.0};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    sc2[0] += rv[e];
    rv[e] = sc2[0];
  }
  if (tid == 0) SW::at(rB, 0, 0)->x = 0.0;
#pragma unroll 2
  for (int cc = 0; cc < PAIRS; ++cc) {
    const double2 d = *SW::at(rB, tid, cc);
    sc2[1] += d.x;
    sc2[1] += d.y;
  }
  {
    double tot2[2];
    bops::block_scan_excl<MNW, 2>(sc2, tot2, ping.next());
  }
  const double offa = sc2[0] + cc0_s, offb = sc2[1];
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) rv[e] += offa;
  {
    double lb = 0.0;  // list B: local inclusive prefix + offset, in place
#pragma unroll 2
    for (int cc = 0; cc < PAIRS; ++cc) {
      double2* p = SW::at(rB, tid, cc);
      const double2 d = *p;
      lb += d.x;
      const double x0 = lb + offb;
      lb += d.y;
      *p = make_double2(x0, lb + offb);
    }
  }
  cp_async_wait_all();  // f and w rows
  __syncthreads();
  const double rqa = A.omega[qa] * A.rho, rqb = A.omega[qb] * A.rho;
  const double irqa = 1.0 / rqa, irqb = 1.0 / rqb;
  const double lama = A.lam[(long)b * K + qa], lamb = A.lam[(long)b * K + qb];
  // (without a list B, qb aliases qa: its rows are empty (nb = 0), its
  // sums zero, its slot past lane K - 1 never read, and nothing is stored)
  // gap sums (barycenter.py:376-381), plan cost by complementary slackness,
  // KL terms, masses, second moment of d under the current tilt (its first
  // moment is the gap term); shift bounds.  One block reduction per list
  // keeps the accumulators of only one list live.
  double acc[6] = {0, 0, 0, 0, 0, 0};
  double mxs[2] = {-CUDART_INF, -CUDART_INF};
  // The tilted weights are recomputed exactly as the tilt formed them,
  // ta = wexp(w, -f/rho - mx) * exp(mx - lambda/rho), with the stored mx and
  // lambda (bit-identical; no row round trip through HBM).
  const double mxa = A.lse[((long)b * K + qa) * 2 + 0], mxb = A.lse[((long)b * K + qb) * 2 + 0];
  const double tsa = exp(mxa - lama * irqa), tsb = exp(mxb - lamb * irqb);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    const double r = rv[e], f = fv[e], w = wv[e];
    const double tv = bops::wexp(w, -f * irqa - mxa, tab) * tsa;
    const double d = r - f;
    acc[0] += tv * d;
    acc[1] += tv * r;
    if (tv > 0.0) acc[2] += tv * (-(f + lama) * irqa);
    acc[3] += tv;
    acc[4] += w;
    acc[5] += tv * d * d;
    if (w > 0.0) {
      mxs[0] = bops::dmax(mxs[0], -f * irqa);
      mxs[1] = bops::dmax(mxs[1], -r * irqa);
    }
  }
  bops::block_red<MNW, 6, 2>(acc, mxs, ping.next());
  const double cqa = acc[0] / acc[3];
  double cs[4] = {acc[0], acc[1] + rqa * (acc[2] - acc[3] + acc[4]), cqa,
                  fmax(acc[5] / acc[3] - cqa * cqa, 0.0) / rqa};
  const double mass_a = acc[4];
  const double mxa0 = mxs[0], mxa1 = mxs[1];
  {
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] = 0.0;
    mxs[0] = mxs[1] = -CUDART_INF;
#pragma unroll 2
    for (int cc = 0; cc < PAIRS; ++cc) {
      const double2 r2 = *SW::at(rB, tid, cc), f2 = *SW::at(fB, tid, cc), w2 = *SW::at(wB, tid, cc);
      const double rr[2] = {r2.x, r2.y}, ff[2] = {f2.x, f2.y}, ww[2] = {w2.x, w2.y};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double t = bops::wexp(ww[h], -ff[h] * irqb - mxb, tab) * tsb;
        const double d = rr[h] - ff[h];
        acc[0] += t * d;
        acc[1] += t * rr[h];
        if (t > 0.0) acc[2] += t * (-(ff[h] + lamb) * irqb);
        acc[3] += t;
        acc[4] += ww[h];
        acc[5] += t * d * d;
        if (ww[h] > 0.0) {
          mxs[0] = bops::dmax(mxs[0], -ff[h] * irqb);
          mxs[1] = bops::dmax(mxs[1], -rr[h] * irqb);
        }
      }
    }
  }
  bops::block_red<MNW, 6, 2>(acc, mxs, ping.next());
  const double cqb = hasB ? acc[0] / acc[3] : 0.0;
  const double csb[4] = {acc[0], acc[1] + rqb * (acc[2] - acc[3] + acc[4]), cqb,
                         fmax(acc[5] / acc[3] - cqb * cqb, 0.0) / rqb};
  const double mass_b = acc[4];
  const double mxb0 = mxs[0], mxb1 = mxs[1];
  MOT_STAMP(2);
  cluster_sum2<4>(cs, csb, slots, parity, K);
  MOT_STAMP(3);
  const double fw_gap = cs[0];
  const double primal = cs[1];
  const double dual = A.scal[b * 4 + 0];
  const double pd_gap = primal - dual;
  const int t = A.t;
  if (c == 0 && tid == 0) {
    A.h0[(long)b * A.max_iters + t] = dual;
    A.fw_gap[(long)b * A.max_iters + t] = fw_gap;
    A.pd_gap[(long)b * A.max_iters + t] = pd_gap;
    A.iterations[b] = t + 1;
    A.summary[b * 2 + 0] = primal;
    A.summary[b * 2 + 1] = dual;
  }
  const bool stop = A.early_exit && pd_gap < A.gap_tol;  // barycenter.py:394-396
  if (stop) {
    if (c == 0 && tid == 0) A.done[b] = 2;
    cl.sync();
    return;
  }
  double gam;
  if (A.step_in != nullptr) {
    gam = __ldg(A.step_in + (long)b * A.max_iters + t);  // replayed gamma_t
  } else if (A.step == UOT_STEP_HARMONIC) {
    gam = 2.0 / (2.0 + t);
  } else {  // safeguarded Newton on Phi(gamma) (see mot_update)
    const double k0 = -cs[2];
    const double vs = cs[3];
    if (!(k0 < 0.0)) {
      gam = 0.0;
    } else {
      double lo = 0.0, hi = 1.0;
      gam = vs > 0.0 ? fmin(1.0, -k0 / vs) : 1.0;
#ifdef UOT_NEWTON_STATS
      if (tid == 0 && c == 0) atomicAdd(&g_mot_stats[1], 1ull);
#endif
      for (int it = 0; it < 24; ++it) {
        const double sha = (1.0 - gam) * mxa0 + gam * mxa1;
        const double shb = (1.0 - gam) * mxb0 + gam * mxb1;
        double mom[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
        for (int e = 0; e < EPT; ++e) {
          const double d = rv[e] - fv[e];
          const double ww = bops::wexp(wv[e], -(fv[e] + gam * d) * irqa - sha, tab);
          const double xc = d - cqa;
          mom[0] += ww;
          mom[1] += ww * xc;
          mom[2] += ww * xc * xc;
        }
#pragma unroll 2
        for (int cc = 0; cc < PAIRS; ++cc) {
          const double2 r2 = *SW::at(rB, tid, cc), f2 = *SW::at(fB, tid, cc),
                        w2 = *SW::at(wB, tid, cc);
          const double rr[2] = {r2.x, r2.y}, ff[2] = {f2.x, f2.y}, wq[2] = {w2.x, w2.y};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double d = rr[h] - ff[h];
            const double ww = bops::wexp(wq[h], -(ff[h] + gam * d) * irqb - shb, tab);
            const double xc = d - cqb;
            mom[3] += ww;
            mom[4] += ww * xc;
            mom[5] += ww * xc * xc;
          }
        }
        bops::block_sum<MNW, 6>(mom, ping.next());
#ifdef UOT_NEWTON_STATS
        if (tid == 0 && c == 0) atomicAdd(&g_mot_stats[0], 1ull);
#endif
        const double e1a = mom[1] / mom[0], e1b = mom[4] / mom[3];
        double gv[2] = {e1a, (mom[2] / mom[0] - e1a * e1a) / rqa};
        const double gvb[2] = {e1b, (mom[5] / mom[3] - e1b * e1b) / rqb};
        cluster_sum2<2>(gv, gvb, slots, parity, K);
        const double g1 = k0 - gv[0], g2 = gv[1];
        if (g1 < 0.0)
          lo = gam;
        else
          hi = gam;
        if (gam >= 1.0 && g1 <= 0.0) {
          gam = 1.0;
          break;
        }
        double nxt = g2 > 0.0 ? gam - g1 / g2 : 0.5 * (lo + hi);
        const bool newton = nxt > lo && nxt < hi;
        if (!newton) nxt = 0.5 * (lo + hi);
        const bool conv = (newton && fabs(nxt - gam) <= 1e-9 * fmax(1.0, gam)) || g1 == 0.0 ||
                          hi - lo <= 1e-15;
        gam = nxt;
        if (conv) break;
      }
    }
  }
  MOT_STAMP(4);
  // barycenter.py:409-411, rounded as numpy rounds it (two products, a sum)
  const double omg = 1.0 - gam;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) fv[e] = __dadd_rn(__dmul_rn(omg, fv[e]), __dmul_rn(gam, rv[e]));
  store_run<EPT>(A.f + basea, i0, na, fv);
#pragma unroll 2
  for (int cc = 0; cc < PAIRS; ++cc) {
    const double2 r2 = *SW::at(rB, tid, cc), f2 = *SW::at(fB, tid, cc);
    *SW::at(fB, tid, cc) = make_double2(__dadd_rn(__dmul_rn(omg, f2.x), __dmul_rn(gam, r2.x)),
                                        __dadd_rn(__dmul_rn(omg, f2.y), __dmul_rn(gam, r2.y)));
  }
  // log-sum-exps of the new iterate (both lists; list_lse's arithmetic)
  double m2[2] = {-CUDART_INF, -CUDART_INF};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e)
    if (wv[e] > 0.0) m2[0] = bops::dmax(m2[0], -fv[e] * irqa);
#pragma unroll 2
  for (int cc = 0; cc < PAIRS; ++cc) {
    const double2 f2 = *SW::at(fB, tid, cc), w2 = *SW::at(wB, tid, cc);
    if (w2.x > 0.0) m2[1] = bops::dmax(m2[1], -f2.x * irqb);
    if (w2.y > 0.0) m2[1] = bops::dmax(m2[1], -f2.y * irqb);
  }
  bops::block_max<MNW, 2>(m2, ping.next());
  double tv[EPT];
  double s2[2] = {0.0, 0.0};
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    tv[e] = bops::wexp(wv[e], -fv[e] * irqa - m2[0], tab);
    s2[0] += tv[e];
  }
#pragma unroll 2
  for (int cc = 0; cc < PAIRS; ++cc) {  // list B's w exp(-f/rho - mx) replaces its dual atoms
    const double2 f2 = *SW::at(fB, tid, cc), w2 = *SW::at(wB, tid, cc);
    const double ex = bops::wexp(w2.x, -f2.x * irqb - m2[1], tab);
    const double ey = bops::wexp(w2.y, -f2.y * irqb - m2[1], tab);
    s2[1] += ex;
    s2[1] += ey;
    *SW::at(rB, tid, cc) = make_double2(ex, ey);
  }
  bops::block_sum<MNW, 2>(s2, ping.next());
  const double qka = m2[0] + log(s2[0]), qkb = m2[1] + log(s2[1]);
  if (tid == 0) {
    A.lse[((long)b * K + qa) * 2 + 0] = m2[0];
    A.lse[((long)b * K + qa) * 2 + 1] = qka;
    if (hasB) {
      A.lse[((long)b * K + qb) * 2 + 0] = m2[1];
      A.lse[((long)b * K + qb) * 2 + 1] = qkb;
    }
  }
  Swz<EPT>::drain(fB, A.f + baseb, nb);
  MOT_STAMP(5);
  if (t + 1 < A.max_iters) {
    // the next iteration's tilt, fused: lambda from the cluster's
    // log-sum-exps (barycenter.py:316-317), H_0 (:320-327), breakpoints.
    double ex[3] = {rqa * qka, rqa * mass_a, rqa};
    const double exb[3] = {rqb * qkb, rqb * mass_b, rqb};
    cluster_sum2<3>(ex, exb, slots, parity, K);
    const double lam1a = rqa * qka - (rqa / ex[2]) * ex[0];
    const double lam1b = rqb * qkb - (rqb / ex[2]) * ex[0];
    if (tid == 0) {
      A.lam[(long)b * K + qa] = lam1a;
      if (hasB) A.lam[(long)b * K + qb] = lam1b;
      if (c == 0) A.scal[b * 4 + 0] = ex[1] - ex[2] * exp(ex[0] / ex[2]);
    }
    const double sca = exp(m2[0] - lam1a * irqa), scb = exp(m2[1] - lam1b * irqb);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
    for (int e = 0; e < EPT; ++e) tv[e] *= sca;
    tilt_tail<EPT>(A, b, qa, na, tv, ping.next(), iscr, vscr, nullptr, false);
    if (hasB) tilt_tail_smem<EPT>(A, b, qb, nb, rB, scb, ping.next(), iscr, vscr);
  }
  MOT_STAMP(6);
  cl.sync();  // slots stay valid until every CTA read them
  MOT_STAMP(7);
}

// mot_update_s: ONE list per CTA (clusters of K CTAs, K <= 16) with the list's
// three rows in shared memory (mot_update2's list-B path on its own).  No row
// lives in registers, so the per-atom loops unroll four wide and the fp64
// exp chains of consecutive atoms interleave (mot_update / mot_update2 keep
// 96 state registers per thread and run them one after the other).
// Chosen by use_update_s (small, ungrouped batches; even n, N <= 16 MT).
#ifndef UPDS_UNROLL
#define UPDS_UNROLL 4
#endif
template <int EPT>
__global__ void __launch_bounds__(MT, 1) mot_update_s(MotArgs A) {
  MOT_STAMP(0);
  using SW = Swz<EPT>;
  constexpr int PAIRS = EPT / 2;
  constexpr int UNR = PAIRS < UPDS_UNROLL ? PAIRS : UPDS_UNROLL;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double rows[];  // r (dcc first), f, w
  constexpr int RBUF = 8 * MNW;
  __shared__ __align__(16) double red[2 * RBUF];
  __shared__ double tab[32];
  __shared__ double slots[32];
  __shared__ int done_s;
  __shared__ double cc0_s;
  __shared__ int iscr[MNW];
  __shared__ double vscr[MNW];
  const int q = (int)cl.block_rank();
  const int b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int nq = list_len(A, q);
  const int tid = threadIdx.x;
  int parity = 0;
  bops::Ping<RBUF> ping{red, 0};
  bops::load_exp_table(tab);
  if (tid == 0) done_s = (A.done != nullptr) ? A.done[b] : 0;
  __syncthreads();
  if (done_s) return;
  const long base = ((long)b * K + q) * n;
  double* rB = rows;
  double* fB = rows + MT * EPT;
  double* wB = rows + 2 * MT * EPT;
  SW::fill(rB, A.dcc + base, nq);
  cp_async_commit();  // the increments first: the prefix scan starts while f and w are in flight
  SW::fill(fB, A.f + base, nq);
  SW::fill(wB, A.a + base, nq);
  cp_async_commit();
  if (tid < 32) {  // f_1[0] = Cc(first tuple) (barycenter.py:206-207)
    const int lane = tid;
    double cc = 0.0;
    if (q == 0) {
      const double x0 = lane < K ? A.x[((long)b * K + lane) * n] : 0.0;
      const double om = lane < K ? A.omega[lane] : 0.0;
      const double bb = warp_sum(om * x0);
      cc = warp_sum(om * ((x0 - bb) * (x0 - bb)));
    }
    if (lane == 0) cc0_s = cc;
  }
  cp_async_wait_but_last();
  __syncthreads();
  MOT_STAMP(1);
  // dual atoms: prefix sums of the cost increments (dcc[0] is not an event)
  if (tid == 0) SW::at(rB, 0, 0)->x = 0.0;
  double sc1[1] = {0.0};
#pragma unroll UNR
  for (int cc = 0; cc < PAIRS; ++cc) {
    const double2 d = *SW::at(rB, tid, cc);
    sc1[0] += d.x;
    sc1[0] += d.y;
  }
  {
    double tot1[1];
    bops::block_scan_excl<MNW, 1>(sc1, tot1, ping.next());
  }
  const double offb = sc1[0] + cc0_s;
  {
    double lb = 0.0;
#pragma unroll UNR
    for (int cc = 0; cc < PAIRS; ++cc) {
      double2* p = SW::at(rB, tid, cc);
      const double2 d = *p;
      lb += d.x;
      const double x0 = lb + offb;
      lb += d.y;
      *p = make_double2(x0, lb + offb);
    }
  }
  cp_async_wait_all();  // f and w rows
  __syncthreads();
  const double rq = A.omega[q] * A.rho, irq = 1.0 / rq;
  const double lamq = A.lam[(long)b * K + q];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  double mxs[2] = {-CUDART_INF, -CUDART_INF};
  const double mxq = A.lse[((long)b * K + q) * 2 + 0];
  const double tsq = exp(mxq - lamq * irq);
#pragma unroll UNR
  for (int cc = 0; cc < PAIRS; ++cc) {
    const double2 r2 = *SW::at(rB, tid, cc), f2 = *SW::at(fB, tid, cc), w2 = *SW::at(wB, tid, cc);
    const double rr[2] = {r2.x, r2.y}, ff[2] = {f2.x, f2.y}, ww[2] = {w2.x, w2.y};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double t = bops::wexp(ww[h], -ff[h] * irq - mxq, tab) * tsq;
      const double d = rr[h] - ff[h];
      acc[0] += t * d;
      acc[1] += t * rr[h];
      if (t > 0.0) acc[2] += t * (-(ff[h] + lamq) * irq);
      acc[3] += t;
      acc[4] += ww[h];
      acc[5] += t * d * d;
      if (ww[h] > 0.0) {
        mxs[0] = bops::dmax(mxs[0], -ff[h] * irq);
        mxs[1] = bops::dmax(mxs[1], -rr[h] * irq);
      }
    }
  }
  bops::block_red<MNW, 6, 2>(acc, mxs, ping.next());
  const double cq = acc[0] / acc[3];
  double cs[4] = {acc[0], acc[1] + rq * (acc[2] - acc[3] + acc[4]), cq,
                  fmax(acc[5] / acc[3] - cq * cq, 0.0) / rq};
  const double mass_q = acc[4];
  const double mx0 = mxs[0], mx1 = mxs[1];
  MOT_STAMP(2);
  cluster_sum<4>(cs, slots, parity);
  MOT_STAMP(3);
  const double fw_gap = cs[0];
  const double primal = cs[1];
  const double dual = A.scal[b * 4 + 0];
  const double pd_gap = primal - dual;
  const int t = A.t;
  if (q == 0 && tid == 0) {
    A.h0[(long)b * A.max_iters + t] = dual;
    A.fw_gap[(long)b * A.max_iters + t] = fw_gap;
    A.pd_gap[(long)b * A.max_iters + t] = pd_gap;
    A.iterations[b] = t + 1;
    A.summary[b * 2 + 0] = primal;
    A.summary[b * 2 + 1] = dual;
  }
  const bool stop = A.early_exit && pd_gap < A.gap_tol;  // barycenter.py:394-396
  if (stop) {
    if (q == 0 && tid == 0) A.done[b] = 2;
    cl.sync();
    return;
  }
  double gam;
  if (A.step_in != nullptr) {
    gam = __ldg(A.step_in + (long)b * A.max_iters + t);  // replayed gamma_t
  } else if (A.step == UOT_STEP_HARMONIC) {
    gam = 2.0 / (2.0 + t);
  } else {  // safeguarded Newton on Phi(gamma) (see mot_update)
    const double k0 = -cs[2];
    const double vs = cs[3];
    if (!(k0 < 0.0)) {
      gam = 0.0;
    } else {
      double lo = 0.0, hi = 1.0;
      gam = vs > 0.0 ? fmin(1.0, -k0 / vs) : 1.0;
      for (int it = 0; it < 24; ++it) {
        const double sh = (1.0 - gam) * mx0 + gam * mx1;
        double mom[3] = {0.0, 0.0, 0.0};
#pragma unroll UNR
        for (int cc = 0; cc < PAIRS; ++cc) {
          const double2 r2 = *SW::at(rB, tid, cc), f2 = *SW::at(fB, tid, cc),
                        w2 = *SW::at(wB, tid, cc);
          const double rr[2] = {r2.x, r2.y}, ff[2] = {f2.x, f2.y}, wq[2] = {w2.x, w2.y};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double d = rr[h] - ff[h];
            const double ww = bops::wexp(wq[h], -(ff[h] + gam * d) * irq - sh, tab);
            const double xc = d - cq;
            mom[0] += ww;
            mom[1] += ww * xc;
            mom[2] += ww * xc * xc;
          }
        }
        bops::block_sum<MNW, 3>(mom, ping.next());
        const double e1 = mom[1] / mom[0];
        double gv[2] = {e1, (mom[2] / mom[0] - e1 * e1) / rq};
        cluster_sum<2>(gv, slots, parity);
        const double g1 = k0 - gv[0], g2 = gv[1];
        if (g1 < 0.0)
          lo = gam;
        else
          hi = gam;
        if (gam >= 1.0 && g1 <= 0.0) {
          gam = 1.0;
          break;
        }
        double nxt = g2 > 0.0 ? gam - g1 / g2 : 0.5 * (lo + hi);
        const bool newton = nxt > lo && nxt < hi;
        if (!newton) nxt = 0.5 * (lo + hi);
        const bool conv = (newton && fabs(nxt - gam) <= 1e-9 * fmax(1.0, gam)) || g1 == 0.0 ||
                          hi - lo <= 1e-15;
        gam = nxt;
        if (conv) break;
      }
    }
  }
  MOT_STAMP(4);
  // barycenter.py:409-411, rounded as numpy rounds it (two products, a sum);
  // the maximum of the new iterate's exponents in the same pass
  const double omg = 1.0 - gam;
  double m1[1] = {-CUDART_INF};
#pragma unroll UNR
  for (int cc = 0; cc < PAIRS; ++cc) {
    const double2 r2 = *SW::at(rB, tid, cc), f2 = *SW::at(fB, tid, cc), w2 = *SW::at(wB, tid, cc);
    const double2 fn = make_double2(__dadd_rn(__dmul_rn(omg, f2.x), __dmul_rn(gam, r2.x)),
                                    __dadd_rn(__dmul_rn(omg, f2.y), __dmul_rn(gam, r2.y)));
    *SW::at(fB, tid, cc) = fn;
    if (w2.x > 0.0) m1[0] = bops::dmax(m1[0], -fn.x * irq);
    if (w2.y > 0.0) m1[0] = bops::dmax(m1[0], -fn.y * irq);
  }
  bops::block_max<MNW, 1>(m1, ping.next());
  double s1[1] = {0.0};
#pragma unroll UNR
  for (int cc = 0; cc < PAIRS; ++cc) {  // w exp(-f/rho - mx) replaces the dual atoms
    const double2 f2 = *SW::at(fB, tid, cc), w2 = *SW::at(wB, tid, cc);
    const double ex = bops::wexp(w2.x, -f2.x * irq - m1[0], tab);
    const double ey = bops::wexp(w2.y, -f2.y * irq - m1[0], tab);
    s1[0] += ex;
    s1[0] += ey;
    *SW::at(rB, tid, cc) = make_double2(ex, ey);
  }
  bops::block_sum<MNW, 1>(s1, ping.next());
  const double qk = m1[0] + log(s1[0]);
  if (tid == 0) {
    A.lse[((long)b * K + q) * 2 + 0] = m1[0];
    A.lse[((long)b * K + q) * 2 + 1] = qk;
  }
  Swz<EPT>::drain(fB, A.f + base, nq);
  MOT_STAMP(5);
  if (t + 1 < A.max_iters) {
    double ex[3] = {rq * qk, rq * mass_q, rq};
    cluster_sum<3>(ex, slots, parity);
    const double lam1 = rq * qk - (rq / ex[2]) * ex[0];
    if (tid == 0) {
      A.lam[(long)b * K + q] = lam1;
      if (q == 0) A.scal[b * 4 + 0] = ex[1] - ex[2] * exp(ex[0] / ex[2]);
    }
    const double sc = exp(m1[0] - lam1 * irq);
    tilt_tail_smem<EPT>(A, b, q, nq, rB, sc, ping.next(), iscr, vscr);
  }
  MOT_STAMP(6);
  cl.sync();  // slots stay valid until every CTA read them
  MOT_STAMP(7);
}

// Balanced sweep (solve_mot_1d, mode 1): the duals are prefix sums of the
// cost increments, f_1[0] = Cc(first tuple), f_k[0] = 0 (barycenter.py:206-229);
// no cross-list reduction, so one plain CTA per list (any K).
template <int EPT>
__global__ void __launch_bounds__(MT) mot_duals(MotArgs A) {
  __shared__ double scr[32];
  __shared__ double cc0_s;
  const int q = blockIdx.x, b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int nq = list_len(A, q);
  const long base = ((long)b * K + q) * n;
  double rv[EPT];
  load_run<EPT>(A.dcc + base, threadIdx.x * EPT, nq, rv);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double c = 0.0;
    if (q == 0 && !A.cost_given) {
      const double x0 = lane < K ? A.x[((long)b * K + lane) * n] : 0.0;
      const double om = lane < K ? A.omega[lane] : 0.0;
      const double bb = warp_sum(om * x0);
      c = warp_sum(om * ((x0 - bb) * (x0 - bb)));
    }
    if (lane == 0) cc0_s = c;
  }
  __syncthreads();
  // dcc[0] is not an event (custom costs: it holds f_q[0] = Cc(first tuple) or 0)
  if (threadIdx.x == 0 && !A.cost_given) rv[0] = 0.0;
  double loc = 0.0;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) {
    loc += rv[e];
    rv[e] = loc;
  }
  double tot;
  const double off = bscan1(loc, tot, scr) + cc0_s;
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) rv[e] += off;
  store_run<EPT>(A.out_f + base, threadIdx.x * EPT, nq, rv);
}

// Custom tuple costs (solve_mot_1d with costfn, barycenter.py:195-229): the
// sweep's state sequence is cost-independent, so the caller evaluates its
// costfn on the visited tuples and the duals follow from the increments:
// state t advances exactly one list p to index i, and
// f_p[i] = f_p[i-1] + cost[t] - cost[t-1]  (new = cost - (pot_sum - old), :225-228),
// f_1[0] = cost[0], f_k[0] = 0.  This kernel scatters the increments into dcc
// at (p, i); mot_duals (cost_given) turns them into prefix sums.
__global__ void mot_cost_dcc(MotArgs A, const double* cost) {
  const int b = blockIdx.y, K = A.k, n = A.n;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int cnt = A.pcount[b];
  const int* ib = A.pidx + (long)b * A.cap_e * K;
  const double* cb = cost + (long)b * A.cap_e;
  double* db = A.dcc + (long)b * K * n;
  if (t == 0) {
    for (int q = 0; q < K; ++q) db[(long)q * n] = (q == 0) ? cb[0] : 0.0;
    return;
  }
  if (t >= cnt) return;
  for (int q = 0; q < K; ++q) {
    const int i = ib[(long)t * K + q];
    if (i != ib[(long)(t - 1) * K + q]) {
      db[(long)q * n + i] = cb[t] - cb[t - 1];
      return;
    }
  }
}

// Final translation by the optimal zero-sum lambda (barycenter.py:413-414),
// from the log-sum-exps the last update stored for the final iterate.
template <int EPT>
__global__ void __launch_bounds__(MT) mot_finalize(MotArgs A) {
  const int q = blockIdx.x, b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  const int nq = list_len(A, q);
  const long base = ((long)b * K + q) * n;
  double ex0, ex1, rtot;
  const double lamq = problem_lambda(A, b, q, ex0, ex1, rtot);
  double fv[EPT];
  load_run<EPT>(A.f + base, threadIdx.x * EPT, nq, fv);
#pragma unroll (EPT <= 32 ? (EPT) : 1)
  for (int e = 0; e < EPT; ++e) fv[e] += lamq;
  store_run<EPT>(A.out_f + base, threadIdx.x * EPT, nq, fv);
}

// ---------------------------------------------------------------------------
// Plan of the current breakpoints: tuples and masses of the positive-mass
// states (barycenter.py:209-222), in sweep order.

__device__ __forceinline__ double next_event_value(const MotArgs& A, int b, int s) {
  // smallest key among the lists' first events of range s (or +inf)
  const int K = A.k, n = A.n;
  const int* sp = A.split + (long)b * (A.S + 1) * K;
  double v = CUDART_INF;
  for (int q = 0; q < K; ++q) {
    const int lo = sp[(long)s * K + q];
    const int ne = list_len(A, q) - 1;
    if (lo < ne) v = fmin(v, A.A[((long)b * K + q) * n + lo]);
  }
  return v;
}

// WRITE: materialise tuples + masses; HASH (trace mode, WRITE false): add
// every kept entry's tuple hash and the entry count into supp_hash / supp_nnz
// of iteration A.t (zeroed by the host before the run).
template <bool WRITE, bool HASH = false>
__global__ void __launch_bounds__(BT) mot_plan(MotArgs A) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ int lo_s[KMAX + 1], cnt_s[KMAX + 1];
  __shared__ int scan_s[BT / 32];
  __shared__ int kept_s;
  const int s = blockIdx.x, b = blockIdx.y + A.b0;
  const int K = A.k, n = A.n;
  double* key;
  int* code;
  const int total = bucket_gather(A, b, s, bsm, key, code, lo_s, cnt_s);
  if (total < 0) return;
  const double tot_mass = A.scal[b * 4 + 1];
  const double nxt = (s + 1 < A.S) ? next_event_value(A, b, s + 1) : CUDART_INF;
  // states: the state after each event (and, in range 0, the initial state)
  const int first = (s == 0) ? -1 : 0;
  const int nst = total - first;  // number of states emitted by this range
  int out_base = 0;
  if (WRITE) {
    for (int r = 0; r < s; ++r) out_base += A.bcount[(long)b * A.S + r];
  }
  int kept_run = 0;
  unsigned long long hacc = 0ull;
  for (int c0 = 0; c0 < nst; c0 += BT) {
    const int c = c0 + threadIdx.x;
    const int e = c + first;  // state after event e (e = -1: initial state)
    double mass = 0.0;
    if (c < nst) {
      const double lo = (e < 0) ? 0.0 : fmin(key[e], tot_mass);
      double hi = (e + 1 < total) ? key[e + 1] : nxt;
      hi = fmin(hi, tot_mass);
      mass = hi - lo;
    }
    const int keep = (c < nst && (mass > 0.0 || A.all_states)) ? 1 : 0;
    // block exclusive scan of keep
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = keep;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int tt = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += tt;
    }
    if (lane == 31) scan_s[warp] = incl;
    __syncthreads();
    int offw = 0, tot = 0;
    for (int w = 0; w < BT / 32; ++w) {
      if (w < warp) offw += scan_s[w];
      tot += scan_s[w];
    }
    __syncthreads();
    const int pos = out_base + kept_run + offw + incl - 1;
    if ((WRITE && keep && pos < A.cap_e) || (HASH && keep)) {
      if (WRITE) A.pmass[(long)b * A.cap_e + pos] = mass;
      // tuple: lo_q + #{events of list q among sorted events [0, e]}; the
      // events of one list are ordered, so the count is a binary search of
      // (key[e], list, index) among list q's keys in this range.
      unsigned long long tkey = 0ull;
      for (int q = 0; q < K; ++q) {
        int cnt = 0;
        const int c_lo = cnt_s[q], c_len = cnt_s[q + 1] - c_lo;
        if (e >= 0 && c_len > 0) {
          const double* Aq = A.A + ((long)b * K + q) * n + lo_s[q];
          const int eq = ev_list(code[e]);
          const int et = ev_index(code[e]);
          int lo2 = 0, hi2 = c_len;
          while (lo2 < hi2) {  // #{j : (Aq[j], q, lo+j) <= (key[e], eq, et)}
            const int mid = (lo2 + hi2) >> 1;
            const bool le = !key_less(key[e], eq, et, Aq[mid], q, lo_s[q] + mid);
            if (le)
              lo2 = mid + 1;
            else
              hi2 = mid;
          }
          cnt = lo2;
        }
        if (WRITE) A.pidx[((long)b * A.cap_e + pos) * K + q] = lo_s[q] + cnt;
        if (HASH) tkey += coord_key(q, lo_s[q] + cnt);
      }
      if (HASH) hacc += mix64(tkey);
    }
    kept_run += tot;
  }
  if (HASH) {
    hacc = warp_sum(hacc);
    if ((threadIdx.x & 31) == 0) atomicAdd(A.supp_hash + (long)b * A.max_iters + A.t, hacc);
    if (threadIdx.x == 0) atomicAdd(A.supp_nnz + (long)b * A.max_iters + A.t, kept_run);
    return;
  }
  if (!WRITE && threadIdx.x == 0) A.bcount[(long)b * A.S + s] = kept_run;
  if (WRITE && threadIdx.x == 0 && s == A.S - 1) A.pcount[b] = min(out_base + kept_run, A.cap_e);
  (void)kept_s;
}

// ---------------------------------------------------------------------------
// Certificate of a balanced multi-marginal solution (barycenter.py:236-295):
// one CTA per problem.  primal = sum_e mass_e Cc(tuple_e) (plan_cost), dual =
// sum_k <a_k, f_k>, support = max_e |sum_k f_k[i_ek] - Cc(tuple_e)|, marginal
// = max_{k,i} |sum_{e: i_ek = i} mass_e - a_k[i]| (the plan is monotone, so
// the entries of atom i of list k are one contiguous run: two binary
// searches), and, when the grid has at most 1e5 tuples, the exhaustive dual
// feasibility sweep (:243-258).  Fixed reduction order: deterministic.
constexpr int CT = 1024;

__device__ __forceinline__ int run_bound(const int* idx, int K, int q, int cnt, int v, bool upper) {
  int lo = 0, hi = cnt;  // first e with idx[e][q] > v (upper) or >= v (lower)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int x = idx[(long)mid * K + q];
    if (upper ? (x <= v) : (x < v))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(CT) mot_certify_kernel(int K, int n, const int* lens,
                                                         const double* omega, const double* x,
                                                         const double* a, const double* f,
                                                         const int* idx, const double* mass,
                                                         const int* count, int cap_e,
                                                         int exhaustive, double* out,
                                                         const double* ecost = nullptr,
                                                         const double* gcost = nullptr,
                                                         long gstride = 0) {
  __shared__ double scr[32];
  const int b = blockIdx.x;
  const int cnt = count[b];
  const int* ib = idx + (long)b * cap_e * K;
  const double* mb = mass + (long)b * cap_e;
  const double* xb = x + (long)b * K * n;
  const double* ab = a + (long)b * K * n;
  const double* fb = f + (long)b * K * n;
  double primal = 0.0, sup = 0.0;
  for (int e = threadIdx.x; e < cnt; e += CT) {
    double bc = 0.0, fs = 0.0;
    for (int q = 0; q < K; ++q) {
      const int i = ib[(long)e * K + q];
      if (ecost == nullptr) bc += omega[q] * xb[(long)q * n + i];
      fs += fb[(long)q * n + i];
    }
    double cc = 0.0;
    if (ecost != nullptr) {  // caller-evaluated tuple cost (custom costfn)
      cc = ecost[(long)b * cap_e + e];
    } else {
      for (int q = 0; q < K; ++q) {
        const double dx = xb[(long)q * n + ib[(long)e * K + q]] - bc;
        cc += omega[q] * (dx * dx);
      }
    }
    primal += mb[e] * cc;
    sup = fmax(sup, fabs(fs - cc));
  }
  double dual = 0.0, marg = 0.0;
  for (int q = 0; q < K; ++q) {
    const int nq = lens != nullptr ? lens[q] : n;
    for (int i = threadIdx.x; i < nq; i += CT) {
      dual += ab[(long)q * n + i] * fb[(long)q * n + i];
      const int lo = run_bound(ib, K, q, cnt, i, false), hi = run_bound(ib, K, q, cnt, i, true);
      double m = 0.0;
      for (int e = lo; e < hi; ++e) m += mb[e];
      marg = fmax(marg, fabs(m - ab[(long)q * n + i]));
    }
  }
  double feas = 0.0;
  if (exhaustive) {
    long total = 1;
    for (int q = 0; q < K; ++q) total *= (lens != nullptr ? lens[q] : n);
    double worst = -CUDART_INF;
    for (long t = threadIdx.x; t < total; t += CT) {
      long r = t;
      double bc = 0.0, fs = 0.0;
      for (int q = K - 1; q >= 0; --q) {  // C order: the last list varies fastest
        const int nq = lens != nullptr ? lens[q] : n;
        const int i = (int)(r % nq);
        r /= nq;
        if (gcost == nullptr) bc += omega[q] * xb[(long)q * n + i];
        fs += fb[(long)q * n + i];
      }
      r = t;
      double cc = 0.0;
      if (gcost != nullptr) {
        cc = gcost[(long)b * gstride + t];
      } else {
        for (int q = K - 1; q >= 0; --q) {
          const int nq = lens != nullptr ? lens[q] : n;
          const int i = (int)(r % nq);
          r /= nq;
          const double dx = xb[(long)q * n + i] - bc;
          cc += omega[q] * (dx * dx);
        }
      }
      worst = fmax(worst, fs - cc);
    }
    worst = block_reduce(worst, scr, MaxOp(), -CUDART_INF);
    feas = fmax(0.0, worst);
  }
  primal = block_reduce(primal, scr, SumOp(), 0.0);
  dual = block_reduce(dual, scr, SumOp(), 0.0);
  sup = block_reduce(sup, scr, MaxOp(), 0.0);
  marg = block_reduce(marg, scr, MaxOp(), 0.0);
  if (threadIdx.x == 0) {
    out[b * 6 + 0] = primal;
    out[b * 6 + 1] = dual;
    out[b * 6 + 2] = sup;
    out[b * 6 + 3] = marg;
    out[b * 6 + 4] = feas;
    out[b * 6 + 5] = exhaustive ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Host driver.

struct MotPlan {
  int S, SS, ept, cap;
  size_t tilt_smem, split_smem, bucket_smem, plan_smem;
};

int ept_for(int n) {
  const int per = (n + MT - 1) / MT;
  if (per <= 1) return 1;
  if (per <= 2) return 2;
  if (per <= 4) return 4;
  if (per <= 8) return 8;
  if (per <= 16) return 16;
  if (per <= 32) return 32;
  // beyond 32 atoms per thread the per-atom loops stay rolled and the per-thread
  // arrays live in local memory (a correctness path; K <= 16 only)
  if (per <= 64) return 64;
  if (per <= 128) return 128;
  if (per <= 256) return 256;
  return -1;
}
constexpr int EPT_MAX = 256;

// Largest possible bucket under regular sampling: list q has
// SS samples at t_j = floor((j+1) ne / (SS+1)), consecutive samples (and the
// list ends) at most gmax = ceil(ne / (SS+1)) + 1 events apart; bucket s holds
// the samples of global rank [R_s, R_{s+1}), at most ceil(K SS / S) of them,
// and list q's events in the bucket lie strictly between the two list-q
// samples just outside it: <= (c_q + 1) gmax - 1 events for c_q samples
// inside.  Summed over the lists: (ceil(K SS / S) + K) gmax - K.
long bucket_bound(int k, int ne, int S, int SS) {
  if (S == 1) return (long)k * ne;
  const long per = ((long)k * SS + S - 1) / S;
  const long gmax = ((long)ne + SS) / (SS + 1) + 1;
  return std::max(1L, (per + k) * gmax - k);
}

MotPlan plan_for(int k, int n) {
  MotPlan p;
  const long events = (long)k * (n - 1);
  p.S = (int)std::min((long)SMAX, std::max(1L, (events + 1535) / 1536));
  // samples per list: enough that the bucket bound stays ~1.25x the average
  // (K SS <= 8192 keeps mot_split's sample merge in shared memory)
  p.SS = (p.S > 1) ? std::max(1, std::min({16 * p.S, n - 1, 8192 / k})) : 1;
  p.ept = ept_for(n);
  if (k > 16 && p.ept == 1) p.ept = 2;  // mot_update2 needs whole 16-byte pairs
  p.cap = (int)std::min(bucket_bound(k, std::max(n - 1, 0), p.S, p.SS), 60000L);
  p.tilt_smem = sizeof(double) * (size_t)n;
  p.split_smem = (sizeof(double) + 3 * sizeof(uint16_t)) * (size_t)k * p.SS;
  p.bucket_smem = bucket_smem_bytes(p.cap, k);
  p.plan_smem = 2 * (sizeof(double) + sizeof(int)) * (size_t)p.cap;
  return p;
}

// Two lists per CTA (mot_update2) when K is even, the cluster stays portable
// and rows are 16-byte aligned; UOT_MOT_UPDATE1=1 forces the one-list kernel.
bool env_flag(const char* name) {
  const char* e = getenv(name);
  return e != nullptr && e[0] == '1';
}

// Two lists per CTA (mot_update2, EPT 2..16): whenever K > 16 (clusters of
// up to 16 CTAs), and by default for even K <= 16 with 16-byte rows (the
// faster choice at cfg5 scale); UOT_MOT_UPDATE1=1 forces the one-list kernel
// where it applies (K <= 16).
bool use_update2(const MotArgs& a) {
  if (a.mode != 0) return false;
  if (a.k > 16) return true;
  return !env_flag("UOT_MOT_UPDATE1") && a.k % 2 == 0 && a.n % 2 == 0;
}

// mot_update_s (one list per CTA, rows in shared memory, clusters of K CTAs)
// finishes a list in ~33 us where mot_update2 takes ~79 us for two, but only 7
// sixteen-CTA clusters are co-resident against 15 eight-CTA ones.  It wins
// whenever the batch is small enough to run ungrouped (a single problem -- the
// reference's own fw_barycenter call -- 75 -> 48 us per iteration at cfg5 size,
// 7 problems 139 -> 84 us); the grouped cfg5 batch stays on mot_update2 (0.435
// vs 0.46 ms per iteration).  UOT_MOT_UPDATES=1 / 0 forces / forbids it.
bool use_update_s(const MotArgs& a) {
  if (a.mode != 0 || a.k > 16 || a.n % 2 != 0) return false;
  const char* e = getenv("UOT_MOT_UPDATES");
  if (e != nullptr) return atoi(e) != 0;
  return a.upd_s != 0 && !env_flag("UOT_MOT_UPDATE1");
}

template <class Kern>
int launch_cluster(Kern kern, int k, int batch, size_t smem, cudaStream_t st, const MotArgs& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(k, batch, 1);
  cfg.blockDim = dim3(MT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = k;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  UOT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  UOT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  UOT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  return UOT_OK;
}

int launch_bucket(const MotArgs& a, const MotPlan& p, cudaStream_t st) {
  UOT_CUDA_TRY(cudaFuncSetAttribute(mot_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)p.bucket_smem));
  mot_bucket<<<dim3(p.S, a.batch), BT2, p.bucket_smem, st>>>(a);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

// tilt -> splitters -> buckets (the K-marginal sweep); then the update.
template <int EPT>
int run_sweep(const MotArgs& a, const MotPlan& p, cudaStream_t st, bool tilt) {
  if (tilt) {  // otherwise the previous mot_update already tilted (fused)
    mot_tilt<EPT><<<dim3(a.k, a.batch), MT, 0, st>>>(a);
    UOT_CHECK_LAUNCH();
  }
  UOT_CUDA_TRY(cudaFuncSetAttribute(mot_split, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)p.split_smem));
  mot_split<<<a.batch, ST, p.split_smem, st>>>(a);
  UOT_CHECK_LAUNCH();
  UOT_TRY(launch_bucket(a, p, st));
  if (a.supp_hash != nullptr) {  // trace mode: this iteration's plan support
    UOT_CUDA_TRY(cudaFuncSetAttribute(mot_plan<false, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)p.plan_smem));
    mot_plan<false, true><<<dim3(p.S, a.batch), BT, p.plan_smem, st>>>(a);
    UOT_CHECK_LAUNCH();
  }
  if (a.mode == 1) {
    if (!a.all_states) {
      mot_duals<EPT><<<dim3(a.k, a.batch), MT, 0, st>>>(a);
      UOT_CHECK_LAUNCH();
    }
    return UOT_OK;
  }
  if constexpr (EPT >= 2 && EPT <= 16) {
    if (use_update_s(a)) {
      UOT_TRY(launch_cluster(mot_update_s<EPT>, a.k, a.batch, 3 * (size_t)MT * EPT * sizeof(double),
                             st, a));
      return UOT_OK;
    }
    if (use_update2(a)) {
      UOT_TRY(launch_cluster(mot_update2<EPT>, (a.k + 1) / 2, a.batch, upd2_smem<EPT>(), st, a));
      return UOT_OK;
    }
  }
  if (a.k > 16) {
    set_error("barycenter FW with more than 16 inputs needs lists of at most %d atoms", 16 * MT);
    return UOT_INVALID;
  }
  UOT_TRY(launch_cluster(mot_update<EPT>, a.k, a.batch,
                         StageRun<EPT>::ON ? 2 * StageRun<EPT>::BYTES : 0, st, a));
  return UOT_OK;
}

int run_plan(const MotArgs& a, const MotPlan& p, cudaStream_t st) {
  UOT_CUDA_TRY(cudaFuncSetAttribute(mot_plan<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)p.plan_smem));
  UOT_CUDA_TRY(cudaFuncSetAttribute(mot_plan<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)p.plan_smem));
  mot_plan<false><<<dim3(p.S, a.batch), BT, p.plan_smem, st>>>(a);
  UOT_CHECK_LAUNCH();
  mot_plan<true><<<dim3(p.S, a.batch), BT, p.plan_smem, st>>>(a);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

// Problem groups: the batch runs as G independent groups on their own
// streams (their iterations interleave on the device, so one group's bucket
// sorts fill the SMs another group's last update wave leaves idle).
int mot_groups(int batch) {
  const char* e = getenv("UOT_MOT_GROUPS");
  const int g = e ? atoi(e) : std::min(8, std::max(1, batch / 8));
  return std::max(1, std::min(g, std::min(batch, 16)));
}

template <int EPT>
int run_all(MotArgs a, const MotPlan& p, cudaStream_t st, bool fw) {
  if (fw) {
    const int G = mot_groups(a.batch);
    a.upd_s = G == 1;
    std::vector<MotArgs> ga(G, a);
    std::vector<cudaStream_t> gs(G, st);
    cudaEvent_t fork = nullptr;
    std::vector<cudaEvent_t> join(G, nullptr);
    if (G > 1) {
      UOT_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      UOT_CUDA_TRY(cudaEventRecord(fork, st));
      for (int g = 0; g < G; ++g) {
        ga[g].b0 = (int)((long)a.batch * g / G);
        ga[g].batch = (int)((long)a.batch * (g + 1) / G) - ga[g].b0;
        UOT_CUDA_TRY(cudaStreamCreateWithFlags(&gs[g], cudaStreamNonBlocking));
        UOT_CUDA_TRY(cudaEventCreateWithFlags(&join[g], cudaEventDisableTiming));
        UOT_CUDA_TRY(cudaStreamWaitEvent(gs[g], fork, 0));
      }
    }
    for (int g = 0; g < G; ++g) {
      mot_lse<EPT><<<dim3(a.k, ga[g].batch), MT, 0, gs[g]>>>(ga[g]);
      UOT_CHECK_LAUNCH();
    }
    for (int t = 0; t < a.max_iters; ++t)
      for (int g = 0; g < G; ++g) {
        ga[g].t = t;
        UOT_TRY(run_sweep<EPT>(ga[g], p, gs[g], t == 0));
      }
    for (int g = 0; g < G; ++g) {
      // plan of the last recorded iteration: its breakpoints are still in A.
      // (Converged problems stopped before updating; the others updated f
      // after the last oracle call, exactly like the reference loop.)
      MotArgs ap = ga[g];
      ap.done = nullptr;
      UOT_TRY(run_plan(ap, p, gs[g]));
      mot_finalize<EPT><<<dim3(a.k, ga[g].batch), MT, 0, gs[g]>>>(ga[g]);
      UOT_CHECK_LAUNCH();
    }
    if (G > 1) {
      for (int g = 0; g < G; ++g) {
        UOT_CUDA_TRY(cudaEventRecord(join[g], gs[g]));
        UOT_CUDA_TRY(cudaStreamWaitEvent(st, join[g], 0));
      }
      for (int g = 0; g < G; ++g) {
        cudaStreamDestroy(gs[g]);  // released once its work completes
        cudaEventDestroy(join[g]);
      }
      cudaEventDestroy(fork);
    }
  } else {
    a.mode = 1;
    UOT_TRY(run_sweep<EPT>(a, p, st, true));
    UOT_TRY(run_plan(a, p, st));
  }
  return UOT_OK;
}

int dispatch(const MotArgs& a, const MotPlan& p, cudaStream_t st, bool fw) {
  switch (p.ept) {
    case 1: return run_all<1>(a, p, st, fw);
    case 2: return run_all<2>(a, p, st, fw);
    case 4: return run_all<4>(a, p, st, fw);
    case 8: return run_all<8>(a, p, st, fw);
    case 16: return run_all<16>(a, p, st, fw);
    case 32: return run_all<32>(a, p, st, fw);
    case 64: return run_all<64>(a, p, st, fw);
    case 128: return run_all<128>(a, p, st, fw);
    case 256: return run_all<256>(a, p, st, fw);
  }
  set_error("lists longer than %d atoms are not supported", EPT_MAX * MT);
  return UOT_INVALID;
}

// Workspace: ta, A, dcc [B][K][n] doubles; split [B][S+1][K] ints; scal
// [B][4]; lam [B][K]; bcount [B][S]; done [B]; omega [K]; lens [K];
// h0/fw/pd [B][T] + iterations (for the plain sweep).
struct MotWs {
  size_t off[17];
  size_t total;
};

MotWs ws_layout(int batch, int k, int n, int S, int SS) {
  MotWs w;
  size_t sz[17];
  const size_t bkn = (size_t)batch * k * n;
  sz[0] = sizeof(double) * bkn;
  sz[1] = sizeof(double) * bkn;
  sz[2] = sizeof(double) * bkn;
  sz[3] = sizeof(int) * (size_t)batch * (S + 1) * k;
  sz[4] = sizeof(double) * 4 * (size_t)batch;
  sz[5] = sizeof(double) * (size_t)batch * k;
  sz[6] = sizeof(int) * (size_t)batch * S;
  sz[7] = sizeof(int) * (size_t)batch;
  sz[8] = sizeof(double) * (size_t)k;
  sz[9] = sizeof(int) * (size_t)k;
  sz[10] = sizeof(double) * 3 * (size_t)batch + sizeof(int) * (size_t)batch;
  sz[11] = sizeof(double) * bkn;  // working copy of the potentials
  sz[12] = sizeof(double) * 2 * (size_t)batch * k;   // lse
  sz[13] = sizeof(double) * (size_t)batch * k;       // mass
  sz[14] = sizeof(double) * (size_t)batch * k;       // tmass
  sz[15] = sizeof(double) * (size_t)batch * k * SS;  // samples
  sz[16] = sizeof(int) * (size_t)batch * k * SS;     // sample indices
  size_t o = 0;
  for (int i = 0; i < 17; ++i) {
    w.off[i] = o;
    o += (sz[i] + 255) / 256 * 256;
  }
  w.total = o;
  return w;
}

MotArgs make_args(int batch, int k, int n, const MotPlan& p, char* ws, const double* omega_host,
                  const int32_t* lens_host, double rho, cudaStream_t st, int* rc) {
  MotArgs a{};
  MotWs L = ws_layout(batch, k, n, p.S, p.SS);
  a.batch = batch;
  a.k = k;
  a.n = n;
  a.rho = rho;
  a.S = p.S;
  a.SS = p.SS;
  a.cap = p.cap;
  a.no_bin = env_flag("UOT_MOT_NOBIN") ? 1 : env_flag("UOT_MOT_COARSEBIN") ? 2 : 0;
  a.ta = (double*)(ws + L.off[0]);
  a.A = (double*)(ws + L.off[1]);
  a.dcc = (double*)(ws + L.off[2]);
  a.split = (int*)(ws + L.off[3]);
  a.scal = (double*)(ws + L.off[4]);
  a.lam = (double*)(ws + L.off[5]);
  a.bcount = (int*)(ws + L.off[6]);
  a.done = (int*)(ws + L.off[7]);
  a.lse = (double*)(ws + L.off[12]);
  a.mass = (double*)(ws + L.off[13]);
  a.tmass = (double*)(ws + L.off[14]);
  a.samp = (double*)(ws + L.off[15]);
  a.sampt = (int*)(ws + L.off[16]);
  double* om = (double*)(ws + L.off[8]);
  a.omega = om;
  a.lens = nullptr;
  *rc = UOT_OK;
  if (lens_host != nullptr) {
    int* ld = (int*)(ws + L.off[9]);
    if (cudaMemcpyAsync(ld, lens_host, sizeof(int) * k, cudaMemcpyHostToDevice, st) !=
        cudaSuccess) {
      set_error("workspace initialisation failed");
      *rc = UOT_CUDA;
    }
    a.lens = ld;
  }
  if (cudaMemcpyAsync(om, omega_host, sizeof(double) * k, cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaMemsetAsync(a.done, 0, sizeof(int) * batch, st) != cudaSuccess) {
    set_error("workspace initialisation failed");
    *rc = UOT_CUDA;
  }
  return a;
}

int check_sizes(int batch, int k, int n) {
  if (batch < 1 || k < 2 || n < 1) {
    set_error("need batch >= 1, k >= 2 inputs, n >= 1 atoms");
    return UOT_INVALID;
  }
  if (k > KMAX) {
    set_error("at most %d input measures per problem", KMAX);
    return UOT_INVALID;
  }
  if (ept_for(n) < 0) {
    set_error("lists longer than %d atoms are not supported", EPT_MAX * MT);
    return UOT_INVALID;
  }
  const MotPlan p = plan_for(k, n);
  if (p.plan_smem > 227 * 1024 || p.bucket_smem > 227 * 1024) {
    set_error("bucket capacity %d exceeds shared memory", p.cap);
    return UOT_INVALID;
  }
  return UOT_OK;
}

}  // namespace
}  // namespace uot

using namespace uot;

extern "C" int uot_mot1d_workspace_size(int32_t batch, int32_t k, int32_t n, size_t* bytes) {
  UOT_TRY(check_sizes(batch, k, n));
  MotPlan p = plan_for(k, n);
  *bytes = ws_layout(batch, k, n, p.S, p.SS).total;
  return UOT_OK;
}

extern "C" int uot_mot1d_batched(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                                 const double* x, const double* a, const double* omega_host,
                                 double* f, int32_t* idx, double* mass, int32_t* count,
                                 int32_t* status, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  UOT_TRY(check_sizes(batch, k, n));
  MotPlan p = plan_for(k, n);
  if (workspace_bytes < ws_layout(batch, k, n, p.S, p.SS).total) {
    set_error("uot_mot1d_batched: workspace too small");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  MotArgs A = make_args(batch, k, n, p, (char*)workspace, omega_host, lens, 1.0, st, &rc);
  UOT_TRY(rc);
  A.mode = 1;
  A.x = x;
  A.a = a;
  A.f = f;
  A.out_f = f;
  A.status = status;
  A.pidx = idx;
  A.pmass = mass;
  A.pcount = count;
  A.cap_e = k * (n - 1) + 1;
  A.max_iters = 1;
  return dispatch(A, p, st, false);
}

extern "C" int uot_bary_workspace_size(const uot_bary_desc* d, size_t* bytes) {
  if (d == nullptr) {
    set_error("null descriptor");
    return UOT_INVALID;
  }
  return uot_mot1d_workspace_size(d->batch, d->k, d->n, bytes);
}

extern "C" int uot_bary_run(const uot_bary_desc* d, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (d == nullptr) {
    set_error("null descriptor");
    return UOT_INVALID;
  }
  UOT_TRY(check_sizes(d->batch, d->k, d->n));
  if (!(d->rho > 0.0) || d->max_iters < 1) {
    set_error("uot_bary_run: need rho > 0 and max_iters >= 1");
    return UOT_INVALID;
  }
  if (d->k > 16 && plan_for(d->k, d->n).ept > 16) {
    set_error("barycenter FW with more than 16 inputs needs lists of at most %d atoms", 16 * MT);
    return UOT_INVALID;
  }
  MotPlan p = plan_for(d->k, d->n);
  MotWs L = ws_layout(d->batch, d->k, d->n, p.S, p.SS);
  if (workspace_bytes < L.total) {
    set_error("uot_bary_run: workspace too small");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  MotArgs A = make_args(d->batch, d->k, d->n, p, (char*)workspace, d->omega, d->lens, d->rho, st,
                        &rc);
  UOT_TRY(rc);
  A.mode = 0;
  A.step = d->step;
  A.max_iters = d->max_iters;
  A.gap_tol = d->gap_tol;
  A.early_exit = d->early_exit;
  A.x = d->x;
  A.a = d->a;
  // iterate on a working copy; the caller's f receives the translated result
  double* work = (double*)((char*)workspace + L.off[11]);
  UOT_CUDA_TRY(cudaMemcpyAsync(work, d->f, sizeof(double) * (size_t)d->batch * d->k * d->n,
                               cudaMemcpyDeviceToDevice, st));
  A.f = work;
  A.out_f = d->f;
  A.h0 = d->h0;
  A.fw_gap = d->fw_gap;
  A.pd_gap = d->pd_gap;
  A.iterations = d->iterations;
  A.status = d->status;
  A.summary = d->summary;
  A.pidx = d->idx;
  A.pmass = d->mass;
  A.pcount = d->count;
  A.cap_e = d->k * (d->n - 1) + 1;
  A.step_in = d->step_in;
  A.supp_hash = reinterpret_cast<unsigned long long*>(d->supp_hash);
  A.supp_nnz = d->supp_nnz;
  if ((A.supp_hash == nullptr) != (A.supp_nnz == nullptr)) {
    set_error("uot_bary_run: supp_hash and supp_nnz go together");
    return UOT_INVALID;
  }
  if (A.supp_hash != nullptr) {
    const size_t bt = (size_t)d->batch * d->max_iters;
    UOT_CUDA_TRY(cudaMemsetAsync(A.supp_hash, 0, sizeof(unsigned long long) * bt, st));
    UOT_CUDA_TRY(cudaMemsetAsync(A.supp_nnz, 0, sizeof(int) * bt, st));
  }
  return dispatch(A, p, st, true);
}

extern "C" int uot_mot_certify(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                               const double* x, const double* a, const double* omega_host,
                               const double* f, const int32_t* idx, const double* mass,
                               const int32_t* count, double* out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  UOT_TRY(check_sizes(batch, k, n));
  if (workspace_bytes < sizeof(double) * (size_t)k + sizeof(int) * (size_t)k + 256) {
    set_error("uot_mot_certify: workspace too small");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* om = (double*)workspace;
  int* ld = (int*)((char*)workspace + (sizeof(double) * (size_t)k + 15) / 16 * 16);
  long grid = 1;
  for (int q = 0; q < k; ++q) {
    grid *= (lens != nullptr ? lens[q] : n);
    if (grid > 100000) break;
  }
  UOT_CUDA_TRY(cudaMemcpyAsync(om, omega_host, sizeof(double) * k, cudaMemcpyHostToDevice, st));
  if (lens != nullptr)
    UOT_CUDA_TRY(cudaMemcpyAsync(ld, lens, sizeof(int) * k, cudaMemcpyHostToDevice, st));
  const int cap_e = k * (n - 1) + 1;
  mot_certify_kernel<<<batch, CT, 0, st>>>(k, n, lens != nullptr ? ld : nullptr, om, x, a, f, idx,
                                           mass, count, cap_e, grid <= 100000 ? 1 : 0, out);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

// Custom tuple costs (solve_mot_1d / plan_cost / mot_certificate with a
// caller costfn).  States: the sweep of uot_mot1d_batched with every visited
// tuple kept (zero-mass states included), count[b] = 1 + sum_q (len_q - 1).
extern "C" int uot_mot1d_states(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                                const double* a, int32_t* idx, double* mass, int32_t* count,
                                int32_t* status, void* workspace, size_t workspace_bytes,
                                void* stream) {
  UOT_TRY(check_sizes(batch, k, n));
  MotPlan p = plan_for(k, n);
  if (workspace_bytes < ws_layout(batch, k, n, p.S, p.SS).total) {
    set_error("uot_mot1d_states: workspace too small");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> om(k, 1.0 / k);  // the cost increments of the sweep are discarded
  int rc;
  MotArgs A = make_args(batch, k, n, p, (char*)workspace, om.data(), lens, 1.0, st, &rc);
  UOT_TRY(rc);
  A.mode = 1;
  A.all_states = 1;
  A.x = a;  // positions do not enter the state sequence
  A.a = a;
  A.status = status;
  A.pidx = idx;
  A.pmass = mass;
  A.pcount = count;
  A.cap_e = k * (n - 1) + 1;
  A.max_iters = 1;
  UOT_TRY(dispatch(A, p, st, false));
  // make_args staged om/lens from host memory that dies with this frame
  UOT_CUDA_TRY(cudaStreamSynchronize(st));
  return UOT_OK;
}

// Duals of the custom-cost sweep from the caller's state costs cost [batch][cap]
// (cap = k (n-1) + 1, the states of uot_mot1d_states in order).
extern "C" int uot_mot1d_cost_duals(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                                    const int32_t* idx, const int32_t* count, const double* cost,
                                    double* f, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  UOT_TRY(check_sizes(batch, k, n));
  MotPlan p = plan_for(k, n);
  if (workspace_bytes < ws_layout(batch, k, n, p.S, p.SS).total) {
    set_error("uot_mot1d_cost_duals: workspace too small");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> om(k, 1.0 / k);
  int rc;
  MotArgs A = make_args(batch, k, n, p, (char*)workspace, om.data(), lens, 1.0, st, &rc);
  UOT_TRY(rc);
  A.mode = 1;
  A.cost_given = 1;
  A.pidx = const_cast<int32_t*>(idx);
  A.pcount = const_cast<int32_t*>(count);
  A.cap_e = k * (n - 1) + 1;
  A.out_f = f;
  mot_cost_dcc<<<dim3((A.cap_e + 255) / 256, batch), 256, 0, st>>>(A, cost);
  UOT_CHECK_LAUNCH();
  switch (p.ept) {
    case 1: mot_duals<1><<<dim3(k, batch), MT, 0, st>>>(A); break;
    case 2: mot_duals<2><<<dim3(k, batch), MT, 0, st>>>(A); break;
    case 4: mot_duals<4><<<dim3(k, batch), MT, 0, st>>>(A); break;
    case 8: mot_duals<8><<<dim3(k, batch), MT, 0, st>>>(A); break;
    case 16: mot_duals<16><<<dim3(k, batch), MT, 0, st>>>(A); break;
    default: mot_duals<32><<<dim3(k, batch), MT, 0, st>>>(A); break;
  }
  UOT_CHECK_LAUNCH();
  UOT_CUDA_TRY(cudaStreamSynchronize(st));
  return UOT_OK;
}

// Certificate with caller-evaluated tuple costs: ecost [batch][cap] at the plan
// entries, gcost [batch][grid] over the whole index grid (C order) when the
// grid holds at most 1e5 tuples (else may be NULL; the sweep is skipped).
extern "C" int uot_mot_certify_costs(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                                     const double* a, const double* f, const int32_t* idx,
                                     const double* mass, const int32_t* count,
                                     const double* ecost, const double* gcost, double* out,
                                     void* workspace, size_t workspace_bytes, void* stream) {
  UOT_TRY(check_sizes(batch, k, n));
  if (ecost == nullptr) {
    set_error("uot_mot_certify_costs: ecost is required");
    return UOT_INVALID;
  }
  if (workspace_bytes < sizeof(double) * (size_t)k + sizeof(int) * (size_t)k + 256) {
    set_error("uot_mot_certify_costs: workspace too small");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* om = (double*)workspace;
  int* ld = (int*)((char*)workspace + (sizeof(double) * (size_t)k + 15) / 16 * 16);
  long grid = 1;
  for (int q = 0; q < k; ++q) {
    grid *= (lens != nullptr ? lens[q] : n);
    if (grid > 100000) break;
  }
  const int exhaustive = (grid <= 100000 && gcost != nullptr) ? 1 : 0;
  UOT_CUDA_TRY(cudaMemsetAsync(om, 0, sizeof(double) * k, st));
  if (lens != nullptr)
    UOT_CUDA_TRY(cudaMemcpyAsync(ld, lens, sizeof(int) * k, cudaMemcpyHostToDevice, st));
  const int cap_e = k * (n - 1) + 1;
  mot_certify_kernel<<<batch, CT, 0, st>>>(k, n, lens != nullptr ? ld : nullptr, om, a, a, f, idx,
                                           mass, count, cap_e, exhaustive, out, ecost, gcost,
                                           exhaustive ? grid : 0);
  UOT_CHECK_LAUNCH();
  if (lens != nullptr) UOT_CUDA_TRY(cudaStreamSynchronize(st));
  return UOT_OK;
}

#ifdef UOT_NEWTON_STATS
// scripts/newton_stats.py (stats build only): Newton passes / line searches
extern "C" int uot_debug_mot_stats(unsigned long long* out, int reset) {
  unsigned long long h[2];
  cudaMemcpyFromSymbol(h, uot::g_mot_stats, sizeof(h));
  out[0] = h[0];
  out[1] = h[1];
  if (reset) {
    h[0] = h[1] = 0;
    cudaMemcpyToSymbol(uot::g_mot_stats, h, sizeof(h));
  }
  return 0;
}
#endif

#ifdef UOT_MOT_TIMING
extern "C" int uot_debug_bkt_stamps(unsigned long long* out, int n) {
  cudaMemcpyFromSymbol(out, uot::g_bkt_stamps, sizeof(unsigned long long) * 6 * (size_t)n);
  return 0;
}
// scripts/mot_timeline.py (timing build only)
extern "C" int uot_debug_mot_stamps(unsigned long long* out, int n) {
  cudaMemcpyFromSymbol(out, uot::g_mot_stamps, sizeof(unsigned long long) * 8 * (size_t)n);
  return 0;
}
#endif
