// blockops.cuh -- fp64 building blocks shared by the 1-D FW kernels
// (fw1d.cu, mot1d.cu): a table-driven exp, and block reductions / scans that
// cost ONE __syncthreads each.
//
// One-sync reductions: every warp reduces its partials, one lane per value
// writes them to a scratch buffer, the block syncs once, and every thread
// re-reads the NW partials (vector loads) and combines them in a fixed
// order, so all threads hold bit-identical results.  Consecutive reductions
// must alternate between two buffers (the next write of a buffer can only
// happen after the sync of the reduction in between, which every thread
// reaches after it finished reading) -- `Ping` hands them out.
#pragma once

#include "common.cuh"

namespace uot {
namespace bops {

constexpr unsigned FULL = 0xffffffffu;

// 2^(j/32), j = 0..31, correctly rounded.
__device__ __constant__ double kExp2Tab[32] = {
    1.0,                1.0218971486541166, 1.0442737824274138, 1.0671404006768237,
    1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775,
    1.189207115002721,  1.215247359980469,  1.241857812073484,  1.2690509571917332,
    1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965,
    1.681792830507429,  1.718619298122478,  1.7562521603732995, 1.7947090750031072,
    1.8340080864093424, 1.8741676341103,    1.9152065613971474, 1.9571441241754002};

// Copy the table into shared memory (call before the first exp_fast, then sync).
__device__ __forceinline__ void load_exp_table(double* tab) {
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Tab[threadIdx.x];
}

// max without NaN handling (DSETP + 2 FSEL instead of the ~6-instruction
// IEEE fmax); arguments are never NaN on the FW paths.
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }

// exp(x) for x <= ~700 (FW arguments are shifted by an upper bound of their
// maximum, so x <= 0 up to rounding).  x = k ln2/32 + r, |r| <= ln2/64;
// k by the 1.5*2^52 rounding trick (no conversion instructions), r by a
// two-constant Cody-Waite fma reduction, e^r - 1 by a degree-6 Estrin
// polynomial (truncation 3.5e-18), 2^(k mod 32 / 32) from the table, 2^(k/32)
// by exponent construction.  Error ~1 ulp.  x < -708 returns 0 (such terms
// are negligible next to the unit-scaled maximum), as exp_nonpos did.
__device__ __forceinline__ double exp_core(double x, const double* tab) {
  const double xc = dmax(x, -708.0);
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(xc, 46.16624130844683, magic);
  const int k = __double2loint(t);
  const double kd = t - magic;
  double r = fma(kd, -0.02166084939249829, xc);
  r = fma(kd, -7.247021293269686e-19, r);
  const double r2 = r * r;
  const double q45 = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  const double q23 = fma(r, 1.0 / 24.0, 1.0 / 6.0);
  const double q01 = fma(r, 0.5, 1.0);
  const double q25 = fma(r2, q45, q23);
  const double q = fma(r2, q25, q01);  // (e^r - 1) / r
  const double tj = tab[k & 31];
  const double y = fma(tj, r * q, tj);
  return y * __hiloint2double(((k >> 5) + 1023) << 20, 0);
}

// exp(x), clamped to [-708, 708] (finite for any input); 0 below -708.
__device__ __forceinline__ double exp_fast(double x, const double* tab) {
  return x < -708.0 ? 0.0 : exp_core(dmin(x, 708.0), tab);
}

// w * exp(x) for a weight w >= 0 whose exponent is shifted by an upper
// bound (x <= 0 up to rounding when w > 0); 0 for w == 0 whatever x is
// (zero-weight atoms carry unbounded potentials) and for x < -708.
__device__ __forceinline__ double wexp(double w, double x, const double* tab) {
  const double e = exp_core(x, tab);
  return (w > 0.0 && x >= -708.0) ? w * e : 0.0;
}


__device__ __forceinline__ double warp_dmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// Reduce-scatter butterfly: K values (K <= 16) summed over the warp with
// ~K shuffles instead of 5K.  Returns the sum of value (lane / (32 / P)),
// P = K rounded up to a power of two; lanes holding the same index hold
// bit-identical sums.
template <int K>
struct Pow2 {
  static constexpr int P = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16;
  static constexpr int G = 32 / P;  // lanes per value
};

template <int K>
__device__ __forceinline__ double warp_sum_scatter(const double (&v)[K]) {
  constexpr int P = Pow2<K>::P;
  static_assert(K <= 16, "warp_sum_scatter: K <= 16");
  const int lane = threadIdx.x & 31;
  double w[P];
#pragma unroll
  for (int k = 0; k < P; ++k) w[k] = k < K ? v[k] : 0.0;
#pragma unroll
  for (int lvl = 0; (P >> lvl) > 1; ++lvl) {
    const int o = 16 >> lvl;
    const int c = P >> lvl;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < c / 2; ++k) {
      const double send = up ? w[k] : w[k + c / 2];
      const double keep = up ? w[k + c / 2] : w[k];
      w[k] = keep + __shfl_xor_sync(FULL, send, o);
    }
  }
#pragma unroll
  for (int o = 16 / P; o >= 1; o >>= 1) w[0] += __shfl_xor_sync(FULL, w[0], o);
  return w[0];
}

// Block reductions, one sync: KS sums and KM maxima.  buf: (KS + KM) * NW
// doubles, 16-byte aligned; NW = blockDim.x / 32 (even).
template <int NW, int KS>
__device__ __forceinline__ void put_sums(const double (&sv)[KS], double* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double s = warp_sum_scatter<KS>(sv);
  constexpr int G = Pow2<KS>::G;
  if ((lane % G) == 0 && lane / G < KS) buf[(lane / G) * NW + warp] = s;
}

template <int NW>
__device__ __forceinline__ double get_sum(const double* buf) {
  const double2* q = reinterpret_cast<const double2*>(buf);
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < NW / 2; ++w) {
    const double2 u = q[w];
    t += u.x;
    t += u.y;
  }
  return t;
}

template <int NW>
__device__ __forceinline__ double get_max(const double* buf) {
  const double2* q = reinterpret_cast<const double2*>(buf);
  double t = -CUDART_INF;
#pragma unroll
  for (int w = 0; w < NW / 2; ++w) {
    const double2 u = q[w];
    t = dmax(t, dmax(u.x, u.y));
  }
  return t;
}

template <int NW, int KS, int KM>
__device__ __forceinline__ void block_red(double (&sv)[KS], double (&mv)[KM], double* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  put_sums<NW, KS>(sv, buf);
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const double mx = warp_dmax(mv[k]);
    if (lane == 0) buf[(KS + k) * NW + warp] = mx;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KS; ++k) sv[k] = get_sum<NW>(buf + k * NW);
#pragma unroll
  for (int k = 0; k < KM; ++k) mv[k] = get_max<NW>(buf + (KS + k) * NW);
}

template <int NW, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* buf) {
  put_sums<NW, K>(v, buf);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = get_sum<NW>(buf + k * NW);
}

template <int NW, int K>
__device__ __forceinline__ void block_max(double (&v)[K], double* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double mx = warp_dmax(v[k]);
    if (lane == 0) buf[k * NW + warp] = mx;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = get_max<NW>(buf + k * NW);
}

// Exclusive block scan (sum) of K per-thread totals, one sync.  On return
// v[k] = sum of the totals of all lower threads (formed as off + incl - v,
// the association the parity fixtures were produced with) and total[k] =
// the block sum.  buf: K * NW doubles.
template <int NW, int K>
__device__ __forceinline__ void block_scan_excl(double (&v)[K], double (&total)[K], double* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double incl[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = v[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += t;
    }
    incl[k] = s;
  }
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < K; ++k) buf[k * NW + warp] = incl[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double2* q = reinterpret_cast<const double2*>(buf + k * NW);
    double off = 0.0, tot = 0.0;
#pragma unroll
    for (int w = 0; w < NW / 2; ++w) {
      const double2 u = q[w];
      if (2 * w < warp) off += u.x;
      tot += u.x;
      if (2 * w + 1 < warp) off += u.y;
      tot += u.y;
    }
    total[k] = tot;
    v[k] = off + incl[k] - v[k];
  }
}

// Alternating scratch buffers for one-sync reductions.
template <int BUF>
struct Ping {
  double* base;
  int ph;
  __device__ double* next() {
    double* p = base + (ph & 1) * BUF;
    ++ph;
    return p;
  }
};

}  // namespace bops
}  // namespace uot
