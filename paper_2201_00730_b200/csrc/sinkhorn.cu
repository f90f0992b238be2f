// sinkhorn.cu -- F/H-Sinkhorn engine for sm_100a (see sinkhorn.cuh for the
// structure).  Reference: src/sinkhorn.py:93-163, src/entropies.py:67-92,
// :187-214, src/duality.py:175-178.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "../../include/uot_b200.h"
#include "sinkhorn.cuh"

#if defined(UOT_WITH_NCCL)
#include <nccl.h>
#endif

namespace uot {

// ---------------------------------------------------------------------------
// Exponent domains.  fp32 kernels work in log2 units so that each pair costs a
// single MUFU.EX2; fp64 kernels use natural units (libdevice exp/log).

template <typename T>
struct Dom;

template <>
struct Dom<float> {
  static constexpr double unit = LN2;  // natural = unit * domain
  static __device__ __forceinline__ float ex(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float lg(float x) { return __log2f(x); }
  static __device__ __forceinline__ double exd(double x) { return exp2(x); }
  static __device__ __forceinline__ double lgd(double x) { return log2(x); }
  static constexpr float HI = 24.0f, LO = -48.0f, TINY = 3.5527136788005009e-15f;  // 2^-48
};

template <>
struct Dom<double> {
  static constexpr double unit = 1.0;
  static __device__ __forceinline__ double ex(double x) { return exp(x); }
  static __device__ __forceinline__ double lg(double x) { return log(x); }
  static __device__ __forceinline__ double exd(double x) { return exp(x); }
  static __device__ __forceinline__ double lgd(double x) { return log(x); }
  static constexpr double HI = 64.0, LO = -256.0, TINY = 6.6e-112;  // ~e^-256
};

}  // namespace uot

#include "sinkhorn_tc.cuh"

namespace uot {

// ---------------------------------------------------------------------------
// Cost policies.  Each defines the packed record of a reduced-side index
// (written by the tail of the previous half-step), the per-output registers,
// and arg(r, o) = (pot_r - C(r,o))/eps + log w_r in domain units, split as
// arg_nov(rec, out) + bias(out) so the per-output bias folds into the shift.

// fp32 squared Euclidean, expanded form |x|^2 + |y|^2 - 2 x.y (d = D).
//   rec = [U, X_0..X_{D-1}, pad], U = (pot - |x|^2) L + log2 w, X = 2 L x
//   out: y[D], bias = -|y|^2 L
template <int D>
struct SqE32 {
  using T = float;
  static constexpr int RW = (D + 1 + 3) / 4 * 4;
  struct Out {
    float y[D];
    float bias;
  };
  static __device__ __forceinline__ void load(Out& o, const DirGeo<float>& g, int b, int idx) {
    const float* p = g.out_pts + b * g.out_pts_bstride + (long)idx * D;
    const float* c = g.ctr + b * g.ctr_bstride;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      o.y[k] = p[k] - c[k];
      s = fmaf(o.y[k], o.y[k], s);
    }
    o.bias = -s * g.L;
  }
  static __device__ __forceinline__ float arg(const float* rec, long, const Out& o,
                                              const DirGeo<float>&, int) {
    if constexpr (D == 2) {
      const float4 r = *reinterpret_cast<const float4*>(rec);
      return fmaf(r.z, o.y[1], fmaf(r.y, o.y[0], r.x));
    } else {
      float a = rec[0];
#pragma unroll
      for (int k = 0; k < D; ++k) a = fmaf(rec[1 + k], o.y[k], a);
      return a;
    }
  }
  static __device__ __forceinline__ void pack(float* rec, double hat, const float* pt, double w,
                                              double L, double, int, const float* ctr) {
    double s = 0.0;
    float xc[D];
    for (int k = 0; k < D; ++k) {
      xc[k] = pt[k] - ctr[k];
      s += (double)xc[k] * (double)xc[k];
    }
    rec[0] = (float)((hat - s) * L + log2(w));
    for (int k = 0; k < D; ++k) rec[1 + k] = (float)(2.0 * L * (double)xc[k]);
    for (int k = D + 1; k < RW; ++k) rec[k] = 0.f;
  }
  static int rw(int) { return RW; }
};

// fp32 squared Euclidean with runtime d (SIMT fallback for d > 3; the d >= 32
// tensor-core path replaces it for throughput).
struct SqE32N {
  using T = float;
  struct Out {
    const float* y;
    const float* c;
    float bias;
  };
  static __device__ __forceinline__ void load(Out& o, const DirGeo<float>& g, int b, int idx) {
    o.y = g.out_pts + b * g.out_pts_bstride + (long)idx * g.d;
    o.c = g.ctr + b * g.ctr_bstride;
    float s = 0.f;
    for (int k = 0; k < g.d; ++k) {
      const float yc = o.y[k] - o.c[k];
      s = fmaf(yc, yc, s);
    }
    o.bias = -s * g.L;
  }
  static __device__ __forceinline__ float arg(const float* rec, long, const Out& o,
                                              const DirGeo<float>& g, int) {
    float a = rec[0];
    for (int k = 0; k < g.d; ++k) a = fmaf(rec[1 + k], __ldg(o.y + k) - __ldg(o.c + k), a);
    return a;
  }
  static __device__ __forceinline__ void pack(float* rec, double hat, const float* pt, double w,
                                              double L, double, int d, const float* ctr) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const float xc = pt[k] - ctr[k];
      s += (double)xc * (double)xc;
    }
    rec[0] = (float)((hat - s) * L + log2(w));
    for (int k = 0; k < d; ++k) rec[1 + k] = (float)(2.0 * L * (double)(pt[k] - ctr[k]));
  }
  static int rw(int d) { return d + 1; }
};

// |x - y|^p on 1-D points (src/measures.py:228-234), any dtype.
//   rec = [P, x], P = pot * L + log w ; arg = P - L * |x - y|^p
template <typename TT>
struct Pow1D {
  using T = TT;
  struct Out {
    T y;
    T bias;
  };
  static __device__ __forceinline__ void load(Out& o, const DirGeo<T>& g, int b, int idx) {
    o.y = g.out_pts[b * g.out_pts_bstride + idx];
    o.bias = T(0);
  }
  static __device__ __forceinline__ T cost(T x, T y, T p) {
    T d = x - y;
    if (p == T(2)) return d * d;
    d = d < T(0) ? -d : d;
    if (p == T(1)) return d;
    return pow(d, p);
  }
  static __device__ __forceinline__ T arg(const T* rec, long, const Out& o, const DirGeo<T>& g,
                                          int) {
    return rec[0] - g.L * cost(rec[1], o.y, g.p);
  }
  static __device__ __forceinline__ void pack(T* rec, double hat, const T* pt, double w, double L,
                                              double, int, const T*) {
    rec[0] = (T)(hat * L + (Dom<T>::unit == 1.0 ? log(w) : log2(w)));
    rec[1] = pt[0];
  }
  static int rw(int) { return 2; }
};

// fp64 squared Euclidean, direct form sum_k (x_k - y_k)^2 (runtime d): the
// fp64 parity path for point clouds.  rec = [P, x_0..x_{d-1}].
struct SqE64 {
  using T = double;
  struct Out {
    const double* y;
    double bias;
  };
  static __device__ __forceinline__ void load(Out& o, const DirGeo<double>& g, int b, int idx) {
    o.y = g.out_pts + b * g.out_pts_bstride + (long)idx * g.d;
    o.bias = 0.0;
  }
  static __device__ __forceinline__ double arg(const double* rec, long, const Out& o,
                                               const DirGeo<double>& g, int) {
    double c = 0.0;
    for (int k = 0; k < g.d; ++k) {
      double t = rec[1 + k] - __ldg(o.y + k);
      c = fma(t, t, c);
    }
    return rec[0] - g.L * c;
  }
  static __device__ __forceinline__ void pack(double* rec, double hat, const double* pt, double w,
                                              double L, double, int d, const double*) {
    rec[0] = hat * L + log(w);
    for (int k = 0; k < d; ++k) rec[1 + k] = pt[k];
  }
  static int rw(int d) { return d + 1; }
};

// Dense explicit cost (src/measures.py:108-122).  rec = [P].
template <typename TT>
struct Explicit {
  using T = TT;
  struct Out {
    int o;
    T bias;
  };
  static __device__ __forceinline__ void load(Out& o, const DirGeo<T>&, int, int idx) {
    o.o = idx;
    o.bias = T(0);
  }
  static __device__ __forceinline__ T arg(const T* rec, long r, const Out& o, const DirGeo<T>& g,
                                          int b) {
    return rec[0] - g.L * __ldg(g.cmat + b * g.cm_bstride + r * g.ld_r + (long)o.o * g.ld_o);
  }
  static __device__ __forceinline__ void pack(T* rec, double hat, const T*, double w, double L,
                                              double, int, const T*) {
    rec[0] = (T)(hat * L + (Dom<T>::unit == 1.0 ? log(w) : log2(w)));
  }
  static int rw(int) { return 1; }
};

// fp32 squared Euclidean on d >= 32 features via tcgen05 (sinkhorn_tc.cuh).
// Records are written straight into the tile layout that the main kernel
// bulk-copies into shared memory.
struct SqE32TC {
  using T = float;
  struct Out {
    float bias;
  };
  static int rw(int d) { return tc_kp(d); }
  // Static part of a record, written once per solve (tc_init_static): the
  // fp16 split Xh, Xl of (2L / S) x', zero padding, the unit columns and
  // |x'|^2 (fp64) parked in float columns 8-9 (no MMA reads them).  x' = x - c
  // is the point relative to the problem's centre c (tc_center: |x - y|^2 =
  // |x'|^2 - 2 x'.y' + |y'|^2 for any c), so the fp16 operands and the fp32
  // accumulator scale with the clouds' extent, not their distance from the origin.
  static __device__ __forceinline__ void init_tile(float* base, long r, int KP, const float* pt,
                                                   const float* ctr, double L, double S, int d) {
    float* tile = base + (r / TC_TILE) * (long)TC_TILE * KP;
    __half* th = reinterpret_cast<__half*>(tile);
    const int rl = (int)(r % TC_TILE);
    const int dp = tc_dp(d), kh = tc_kh(d);
    const double sc = 2.0 * L / S;
    double s2 = 0.0;
    for (int k = 0; k < dp; ++k) {
      float xh = 0.f, xl = 0.f;
      if (k < d) {
        const float xc = pt[k] - ctr[k];
        const float x = (float)(sc * (double)xc);
        xh = __half2float(__float2half_rn(x));
        xl = x - xh;
        s2 += (double)xc * (double)xc;
      }
      th[tc_xidx(rl, k, d)] = __float2half_rn(xh);
      th[tc_xidx(rl, dp + k, d)] = __float2half_rn(xl);
    }
    for (int k = 2 * dp; k < kh; ++k) th[tc_xidx(rl, k, d)] = __float2half_rn(0.f);
    tile[tc_cidx(rl, 3, d)] = 1.f;
    tile[tc_cidx(rl, 4, d)] = 1.f;
    tile[tc_cidx(rl, 5, d)] = 1.f;
    tile[tc_cidx(rl, 6, d)] = 0.f;
    tile[tc_cidx(rl, 7, d)] = 0.f;
    tile[tc_cidx(rl, 10, d)] = 0.f;
    tile[tc_cidx(rl, 11, d)] = 0.f;
    *reinterpret_cast<double*>(tile + tc_cidx(rl, 8, d)) = s2;
  }
  // Per half-step: only U = (hat - |x|^2) L + log2 w changes -- one 16-byte
  // store [Uh, Um, Ul, 1] (tf32 splits) per record.
  static __device__ __forceinline__ void pack_tile(float* base, long r, int KP, double hat,
                                                   const float*, double w, double L, int d) {
    float* tile = base + (r / TC_TILE) * (long)TC_TILE * KP;
    const int rl = (int)(r % TC_TILE);
    const double s2 = *reinterpret_cast<const double*>(tile + tc_cidx(rl, 8, d));
    const double u = w > 0.0 ? (hat - s2) * L + log2(w) : -1e30;
    const float uh = tf32_hi((float)u);
    const double u1 = u - (double)uh;
    const float um = tf32_hi((float)u1);
    *reinterpret_cast<float4*>(tile + tc_cidx(rl, 0, d)) =
        make_float4(uh, um, (float)(u1 - (double)um), 1.f);
  }
};

__global__ void tc_init_static(float* rec, long rec_bstride, const float* pts, const float* ctr,
                               long ctr_bstride, int batch, int n, int d, int KP, double L,
                               double S) {
  const long total = (long)batch * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int b = (int)(i / n);
    const long r = i - (long)b * n;
    SqE32TC::init_tile(rec + (long)b * rec_bstride, r, KP, pts + i * d, ctr + b * ctr_bstride, L,
                       S, d);
  }
}

// Centre of problem b's fp32 point clouds (the expanded-form engines SqE32<D>,
// SqE32N and the tcgen05 path): the midpoint of the two clouds' centroids,
// c = (mean x + mean y) / 2, estimated on an evenly strided sample of at most
// CTR_SAMPLES points per side (one short kernel per solve; any c inside the
// clouds' hull does the job).  |x - y|^2 = |x'|^2 - 2 x'.y' + |y'|^2 for any c,
// and with x' = x - c, y' = y - c every term scales with the clouds' radii,
// not with their distance from the origin (no cancellation).  For d <= 256,
// thread t of the (R x d)-thread block owns coordinate t % d of samples t / d,
// t/d + R, ...; the R partials of a coordinate are added in a fixed order
// (deterministic); larger d loops over the coordinates.
constexpr int CTR_SAMPLES = 1024;

__global__ void __launch_bounds__(256) sk_center(const float* x, const float* y, int n, int m,
                                                 int d, float* ctr) {
  __shared__ double part[256];
  const int b = blockIdx.x;
  const float* xb = x + (long)b * n * d;
  const float* yb = y + (long)b * m * d;
  const int sn = min(n, CTR_SAMPLES), sm = min(m, CTR_SAMPLES);
  auto row_x = [&](int s) { return (long)s * n / sn; };
  auto row_y = [&](int s) { return (long)s * m / sm; };
  if (d > 256) {
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
      double sx = 0.0, sy = 0.0;
      for (int i = 0; i < sn; ++i) sx += (double)xb[row_x(i) * d + k];
      for (int j = 0; j < sm; ++j) sy += (double)yb[row_y(j) * d + k];
      ctr[(long)b * d + k] = (float)(0.5 * (sx / sn + sy / sm));
    }
    return;
  }
  const int R = blockDim.x / d;
  const int k = threadIdx.x % d, r0 = threadIdx.x / d;
  double sx = 0.0, sy = 0.0;
  if (r0 < R) {
    for (int i = r0; i < sn; i += R) sx += (double)xb[row_x(i) * d + k];
    for (int j = r0; j < sm; j += R) sy += (double)yb[row_y(j) * d + k];
  }
  part[threadIdx.x] = 0.5 * (sx / sn + sy / sm);
  __syncthreads();
  if (threadIdx.x < d) {
    double c = 0.0;
    for (int r = 0; r < R; ++r) c += part[r * d + threadIdx.x];
    ctr[(long)b * d + threadIdx.x] = (float)c;
  }
}

template <class P>
constexpr bool centred() {
  return std::is_same<P, SqE32TC>::value || std::is_same<P, SqE32N>::value ||
         std::is_same<P, SqE32<1>>::value || std::is_same<P, SqE32<2>>::value ||
         std::is_same<P, SqE32<3>>::value;
}

template <class P>
int launch_center(const uot_sinkhorn_desc& d, float* ctr, cudaStream_t st) {
  if constexpr (centred<P>()) {
    const int threads = d.d <= 256 ? d.d * (256 / d.d) : 256;
    sk_center<<<d.batch, threads, 0, st>>>((const float*)d.x, (const float*)d.y, d.n, d.m, d.d,
                                           ctr);
    UOT_CHECK_LAUNCH();
  }
  return UOT_OK;
}

// Power-of-two A-operand scale S of the tcgen05 path: the A rows carry S y'
// and the B records (2L / S) x', so S = sqrt(2L) balances their magnitudes
// (both ~ sqrt(2L) |x'|).  fp16 then overflows only when 2L R^2 > ~4e9
// (R = the largest distance to the centre), where the fp32 exponent
// arguments themselves (~2L R^2 in log2 units) carry no precision left.
inline double tc_ascale(double L) {
  const double s = std::ldexp(1.0, (int)std::lround(0.5 * std::log2(2.0 * L)));
  return std::min(std::max(s, std::ldexp(1.0, -24)), std::ldexp(1.0, 24));
}

// Record layout of a side: `rw` elements per index, or the tiled layout.
template <class P>
struct RecLayout {
  static long stride(int n, int d) { return (long)n * P::rw(d); }
  static __device__ __forceinline__ void pack(typename P::T* base, long o, int rw, double hat,
                                              const typename P::T* pt, double w, double L,
                                              double p, int d, const typename P::T* ctr) {
    P::pack(base + o * rw, hat, pt, w, L, p, d, ctr);
  }
};
template <>
struct RecLayout<SqE32TC> {
  static long stride(int n, int d) {
    return (long)((n + TC_TILE - 1) / TC_TILE) * TC_TILE * tc_kp(d);
  }
  static __device__ __forceinline__ void pack(float* base, long o, int rw, double hat,
                                              const float* pt, double w, double L, double,
                                              int d, const float*) {
    SqE32TC::pack_tile(base, o, rw, hat, pt, w, L, d);
  }
};

// One register tile: RT reduced records x COLS outputs.  Exponents are
// formed first, their max checked against the safe window of the current
// shift (conditional rescale, rarely taken), then exponentiated and summed.
template <class P, int COLS, int RT, bool CHECK>
__device__ __forceinline__ void tile(const typename P::T* srec, int rw, int rr, int clen, long rbase,
                                     const typename P::Out (&out)[COLS],
                                     const DirGeo<typename P::T>& g, int b,
                                     typename P::T (&cc)[COLS], typename P::T (&mm)[COLS],
                                     typename P::T (&acc)[COLS]) {
  using T = typename P::T;
  using D = Dom<T>;
  T t[RT][COLS];
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const bool ok = !CHECK || rr + i < clen;
    const T* rc = srec + (ok ? (rr + i) : 0) * rw;
#pragma unroll
    for (int c = 0; c < COLS; ++c) {
      const T v = P::arg(rc, rbase + rr + i, out[c], g, b) + cc[c];
      t[i][c] = ok ? v : T(-INFINITY);
    }
  }
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    T mx = t[0][c];
#pragma unroll
    for (int i = 1; i < RT; ++i) mx = fmax(mx, t[i][c]);
    if (mx > D::HI || (mx < D::LO && acc[c] < D::TINY)) {
      // Rare: the stale shift is off by more than the safe window.  Move the
      // shift to the current maximum (FA-style conditional rescale).
      T mn = mx;
      if (acc[c] > T(0)) mn = fmax(mn, D::lg(acc[c]));
      if (mn > T(-INFINITY) && mn < T(INFINITY)) {
        if (acc[c] > T(0)) acc[c] *= D::ex(-mn);
        mm[c] += mn;
        cc[c] -= mn;
#pragma unroll
        for (int i = 0; i < RT; ++i) t[i][c] -= mn;
      }
    }
    T s = D::ex(t[0][c]);
#pragma unroll
    for (int i = 1; i < RT; ++i) s += D::ex(t[i][c]);
    acc[c] += s;
  }
}

// ---------------------------------------------------------------------------
// Main kernel: partial online log-sum-exp over a split of the reduced index.

template <class P, int THREADS, int COLS, int RT>
__global__ void __launch_bounds__(THREADS) sk_main(MainArgs<typename P::T> A) {
  using T = typename P::T;
  using D = Dom<T>;
  const int b = blockIdx.z;
  if (A.done != nullptr && A.done[b]) return;
  const int split = blockIdx.y, S = gridDim.y;
  const long r0 = (long)A.nred * split / S;
  const long r1 = (long)A.nred * (split + 1) / S;
  const int rw = A.g.rw;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* srec = reinterpret_cast<T*>(smem_raw);

  typename P::Out out[COLS];
  T cc[COLS], mm[COLS], acc[COLS];
  const int ohi = A.out_hi > 0 ? A.out_hi : A.nout;
  const int obase = A.out_lo + blockIdx.x * THREADS * COLS + threadIdx.x;
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    const int o = obase + c * THREADS;
    const bool ok = o < ohi;
    P::load(out[c], A.g, b, ok ? o : 0);
    mm[c] = ok ? A.shift_in[(long)b * A.nout + o] : T(0);
    cc[c] = out[c].bias - mm[c];
    acc[c] = T(0);
  }

  const T* rec_g = A.g.red_rec + b * A.g.red_bstride;
  for (long cs = r0; cs < r1; cs += A.chunk) {
    const int clen = (int)min((long)A.chunk, r1 - cs);
    {
      const long base = (cs + A.red_offset) * rw;
      const int nel = clen * rw;
      for (int e = threadIdx.x; e < nel; e += THREADS) srec[e] = rec_g[base + e];
    }
    __syncthreads();
    // Full tiles run without bounds checks; the ragged tail of the chunk
    // takes the checked path.
    const int full = clen / RT * RT;
    for (int rr = 0; rr < full; rr += RT)
      tile<P, COLS, RT, false>(srec, rw, rr, clen, cs + A.red_offset, out, A.g, b, cc, mm, acc);
    if (full < clen)
      tile<P, COLS, RT, true>(srec, rw, full, clen, cs + A.red_offset, out, A.g, b, cc, mm, acc);
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    const int o = obase + c * THREADS;
    if (o < ohi) {
      const long idx = ((long)b * A.splits_total + A.split_base + split) * A.nout + o;
      A.part_m[idx] = mm[c];
      A.part_a[idx] = acc[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Packed fp32x2 main kernel for the 2-D squared-Euclidean cost (BASELINE
// cfg3).  Blackwell's FFMA2 / FADD2 process two output columns per
// instruction with the row record broadcast as a scalar operand, so a pair
// costs ~3.5 issued instructions (FADD2 + 2 FFMA2 per two pairs, FMNMX3 for
// the shift check, one MUFU.EX2, half an FADD2 for the sum) and the kernel is
// bound by the MUFU pipe (16 ex2 / clk / SM) rather than by issue.

typedef unsigned long long u64;

__device__ __forceinline__ u64 p2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void u2(u64 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for a packed pair on the FMA pipe (exp2 offload: the MUFU pipe, 16
// ex2/clk/SM, is the kernel's bound while issue slots are left over).
// x = n + f with n = rint(x) by the 1.5*2^23 trick, 2^f by a degree-4
// minimax polynomial on [-1/2, 1/2] (max rel. error 2.7e-6, vs ~2^-22 for
// ex2.approx), 2^n added into the exponent field with one IMAD.  Inputs are
// clamped below at -127 (the result is then ~2^-127, where MUFU flushes to
// 0: negligible next to the tile's unit-scale terms); the caller checks the
// running maximum `pmax` (FMNMX3) against 126 and falls back to MUFU.
__device__ __forceinline__ u64 ex2_poly2(u64 x, float& pmax) {
  float lo, hi;
  u2(x, lo, hi);
  asm("max.f32 %0, %0, %1, %2;" : "+f"(pmax) : "f"(lo), "f"(hi));
  const u64 xc = p2(fmaxf(lo, -127.f), fmaxf(hi, -127.f));
  const u64 MAG = p2(12582912.f, 12582912.f);
  const u64 tm = add2(xc, MAG);
  const u64 nf = add2(tm, p2(-12582912.f, -12582912.f));
  const u64 f = fma2(nf, p2(-1.f, -1.f), xc);
  u64 q = fma2(f, p2(0.009570101276040077f, 0.009570101276040077f),
               p2(0.05591786280274391f, 0.05591786280274391f));
  q = fma2(f, q, p2(0.240247443318367f, 0.240247443318367f));
  q = fma2(f, q, p2(0.6931217908859253f, 0.6931217908859253f));
  q = fma2(f, q, p2(0.9999992847442627f, 0.9999992847442627f));
  unsigned qlo, qhi, tlo, thi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(qlo), "=r"(qhi) : "l"(q));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(tlo), "=r"(thi) : "l"(tm));
  const unsigned rlo = tlo * 0x800000u + qlo, rhi = thi * 0x800000u + qhi;
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(rlo), "r"(rhi));
  return r;
}

#ifndef SQ2_NPOLY
#define SQ2_NPOLY 0  // rows per RT-row tile on the FMA-pipe exp2 (measured: no gain)
#endif

// Slow path of a packed tile (stale shift outside the safe window): redo
// the tile column by column with an explicit maximum and rescale.
template <int CP, int RT, bool CHECK>
__device__ __forceinline__ void tile_sq2_slow(const float* srec, int rr, int clen, const u64 (&y0)[CP],
                                           const u64 (&y1)[CP], u64 (&cc)[CP],
                                           float (&mm)[2 * CP], u64 (&acc)[CP]) {
  using D = Dom<float>;
#pragma unroll
  for (int j = 0; j < CP; ++j) {
    float yy0[2], yy1[2], c2[2], a2[2];
    u2(y0[j], yy0[0], yy0[1]);
    u2(y1[j], yy1[0], yy1[1]);
    u2(cc[j], c2[0], c2[1]);
    u2(acc[j], a2[0], a2[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float t[RT];
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const bool ok = !CHECK || rr + i < clen;
        const float4 r = *reinterpret_cast<const float4*>(srec + (ok ? (rr + i) : 0) * 4);
        t[i] = ok ? fmaf(r.z, yy1[h], fmaf(r.y, yy0[h], r.x + c2[h])) : -INFINITY;
        mx = fmaxf(mx, t[i]);
      }
      if (mx > D::HI || (mx < D::LO && a2[h] < D::TINY)) {
        float mn = mx;
        if (a2[h] > 0.f) mn = fmaxf(mn, D::lg(a2[h]));
        if (mn > -INFINITY && mn < INFINITY) {
          if (a2[h] > 0.f) a2[h] *= D::ex(-mn);
          mm[2 * j + h] += mn;
          c2[h] -= mn;
#pragma unroll
          for (int i = 0; i < RT; ++i) t[i] -= mn;
        }
      }
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < RT; ++i) sum += D::ex(t[i]);
      a2[h] += sum;
    }
    cc[j] = p2(c2[0], c2[1]);
    acc[j] = p2(a2[0], a2[1]);
  }
}

// Fast path: packed exponents, no per-pair maximum.  The accumulated sums are
// range-checked after the tile instead (overflow -> inf / > 2^100, or
// everything so far below 2^-100); a failing tile is redone by the slow path
// from the pre-tile state.  In steady state the stale shift (the previous
// iteration's log-sum-exp of the same output) keeps every tile in range.
template <int CP, int RT, bool CHECK>
__device__ __forceinline__ void tile_sq2(const float* srec, int rr, int clen, const u64 (&y0)[CP],
                                         const u64 (&y1)[CP], u64 (&cc)[CP], float (&mm)[2 * CP],
                                         u64 (&acc)[CP]) {
  u64 t[RT][CP];
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const bool ok = !CHECK || rr + i < clen;
    const float4 r = *reinterpret_cast<const float4*>(srec + (ok ? (rr + i) : 0) * 4);
    const float uu = ok ? r.x : -INFINITY;
    const u64 U = p2(uu, uu);
    const u64 X0 = p2(r.y, r.y), X1 = p2(r.z, r.z);
#pragma unroll
    for (int j = 0; j < CP; ++j) t[i][j] = fma2(X1, y1[j], fma2(X0, y0[j], add2(U, cc[j])));
  }
  u64 na[CP];
  bool bad = false;
  constexpr int NPOLY = CHECK ? 0 : (SQ2_NPOLY < RT ? SQ2_NPOLY : RT - 1);
  float pmax = -INFINITY;
#pragma unroll
  for (int j = 0; j < CP; ++j) {
    float lo, hi;
    u2(t[0][j], lo, hi);
    u64 s = p2(ex2f(lo), ex2f(hi));
#pragma unroll
    for (int i = 1; i < RT - NPOLY; ++i) {
      u2(t[i][j], lo, hi);
      s = add2(s, p2(ex2f(lo), ex2f(hi)));
    }
#pragma unroll
    for (int i = RT - NPOLY; i < RT; ++i) s = add2(s, ex2_poly2(t[i][j], pmax));
    na[j] = add2(acc[j], s);
    float alo, ahi;
    u2(na[j], alo, ahi);
    bad |= !(alo < 1.2676506e30f && ahi < 1.2676506e30f && alo > 7.8886091e-31f &&
             ahi > 7.8886091e-31f);  // (2^-100, 2^100)
  }
  bad |= pmax > 126.f;
  if (bad) {
    tile_sq2_slow<CP, RT, CHECK>(srec, rr, clen, y0, y1, cc, mm, acc);
  } else {
#pragma unroll
    for (int j = 0; j < CP; ++j) acc[j] = na[j];
  }
}

#ifndef SQ2_MINB
#define SQ2_MINB 8  // resident CTAs per SM asked of the compiler: 64 registers (44 B of spills) and 32
                    // warps per SM -- measured 7 / 8 / 9 / 10 CTAs: 488.0 / 496.8 / 492.0 / 488.5 iter/s at cfg3
#endif
template <int THREADS, int CP, int RT>
__global__ void __launch_bounds__(THREADS, SQ2_MINB) sk_main_sq2(MainArgs<float> A) {
  const int b = blockIdx.z;
  if (A.done != nullptr && A.done[b]) return;
  const int split = blockIdx.y, S = gridDim.y;
  const long r0 = (long)A.nred * split / S;
  const long r1 = (long)A.nred * (split + 1) / S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* srec = reinterpret_cast<float*>(smem_raw);
  constexpr int COLS = 2 * CP;
  u64 y0[CP], y1[CP], cc[CP], acc[CP];
  float mm[COLS];
  const int ohi = A.out_hi > 0 ? A.out_hi : A.nout;
  const int obase = A.out_lo + blockIdx.x * THREADS * COLS + threadIdx.x;
  const float L = A.g.L;
  const float* pts = A.g.out_pts + b * A.g.out_pts_bstride;
  const float cen0 = A.g.ctr[b * A.g.ctr_bstride], cen1 = A.g.ctr[b * A.g.ctr_bstride + 1];
#pragma unroll
  for (int j = 0; j < CP; ++j) {
    float ya0[2], ya1[2], c[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = obase + (2 * j + h) * THREADS;
      const bool ok = o < ohi;
      const float q0 = ok ? pts[(long)o * 2] - cen0 : 0.f;
      const float q1 = ok ? pts[(long)o * 2 + 1] - cen1 : 0.f;
      ya0[h] = q0;
      ya1[h] = q1;
      mm[2 * j + h] = ok ? A.shift_in[(long)b * A.nout + o] : 0.f;
      c[h] = -fmaf(q0, q0, q1 * q1) * L - mm[2 * j + h];
    }
    y0[j] = p2(ya0[0], ya0[1]);
    y1[j] = p2(ya1[0], ya1[1]);
    cc[j] = p2(c[0], c[1]);
    acc[j] = p2(0.f, 0.f);
  }
  const float* rec_g = A.g.red_rec + b * A.g.red_bstride;
  for (long cs = r0; cs < r1; cs += A.chunk) {
    const int clen = (int)min((long)A.chunk, r1 - cs);
    {
      const float4* src = reinterpret_cast<const float4*>(rec_g + (cs + A.red_offset) * 4);
      float4* dst = reinterpret_cast<float4*>(srec);
      for (int e = threadIdx.x; e < clen; e += THREADS) dst[e] = src[e];
    }
    __syncthreads();
    const int full = clen / RT * RT;
    for (int rr = 0; rr < full; rr += RT) tile_sq2<CP, RT, false>(srec, rr, clen, y0, y1, cc, mm, acc);
    if (full < clen) tile_sq2<CP, RT, true>(srec, full, clen, y0, y1, cc, mm, acc);
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < CP; ++j) {
    float a2[2];
    u2(acc[j], a2[0], a2[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = obase + (2 * j + h) * THREADS;
      if (o < ohi) {
        const long idx = ((long)b * A.splits_total + A.split_base + split) * A.nout + o;
        A.part_m[idx] = mm[2 * j + h];
        A.part_a[idx] = a2[h];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Entropy helpers (src/entropies.py:141-263) for the F / G steps.

// Berg aprox: the root of h(y) = y + eps log(rho / (rho - y)) - x on
// (-inf, rho), strictly increasing with range R (entropies.py:224-263):
// bracket (lo by doubling steps, hi towards rho by quartering gaps), then
// bisection-safeguarded Newton to |h| < 1e-12 or a bracket of 4 ulps.
__device__ double berg_aprox(double rho, double eps, double x) {
  auto h = [&](double y) { return y + eps * log(rho / (rho - y)) - x; };
  double lo = fmin(x, rho - 1.0);
  double step = fmax(1.0, eps);
  for (int it = 0; it < 200 && h(lo) > 0.0; ++it) {
    lo -= step;
    step *= 2.0;
  }
  const double top = nextafter(rho, -CUDART_INF);
  double gap = rho - fmin(x, rho - 1.0);
  double hi = fmin(rho - gap, top);
  for (int it = 0; it < 200 && h(hi) < 0.0 && hi < top; ++it) {
    gap *= 0.25;
    hi = fmin(rho - gap, top);
  }
  double y = fmin(fmax(fmin(x, rho - gap), lo), hi);
  const double em = 2.220446049250313e-16;
  for (int it = 0; it < 100; ++it) {
    const double res = h(y);
    if (fabs(res) < 1e-12 || (hi - lo) <= 4.0 * em * (1.0 + fabs(y))) break;
    if (res < 0.0) lo = y;
    if (res > 0.0) hi = y;
    const double nt = y - res / (1.0 + eps / (rho - y));
    y = (nt > lo && nt < hi) ? nt : 0.5 * (lo + hi);
  }
  return y;
}

// aprox(spec, eps, x) (entropies.py:203-221)
__device__ __forceinline__ double aprox_any(int ent, double rho, double eps, double x) {
  if (ent == UOT_ENT_KL) return (rho / (eps + rho)) * x;
  if (ent == UOT_ENT_BALANCED) return x;
  return berg_aprox(rho, eps, x);
}

// conj_grad / conj_hess (entropies.py:157-184) for KL and Berg
__device__ __forceinline__ double conj_grad_d(int ent, double rho, double x) {
  return ent == UOT_ENT_KL ? exp(x / rho) : rho / (rho - x);
}
__device__ __forceinline__ double conj_hess_d(int ent, double rho, double x) {
  return ent == UOT_ENT_KL ? exp(x / rho) / rho : rho / ((rho - x) * (rho - x));
}

// G variant with a Berg marginal: lambda* of the current pair by the
// reference's bracketed Newton (duality.py:182-247), one CTA per problem,
// starting from the incoming lam; the residual / slope are block reductions
// over both potentials (pot = hat + tau).
template <typename T>
__global__ void __launch_bounds__(256) sk_lambda_newton(int n, int m, const T* hatA,
                                                       const T* hatB, const T* wa, const T* wb,
                                                       int e1, int e2, double r1, double r2,
                                                       SkScalars* sc, int* status, int* done) {
  __shared__ double s_x[32];
  __shared__ double s_r[2];
  const int b = blockIdx.x;
  const double tf = sc[b].tau[0], tg = sc[b].tau[1];
  const T* f = hatA + (long)b * n;
  const T* g = hatB + (long)b * m;
  const T* a = wa + (long)b * n;
  const T* bw = wb + (long)b * m;
  double fmn = CUDART_INF, gmn = CUDART_INF;
  for (int i = threadIdx.x; i < n; i += blockDim.x) fmn = fmin(fmn, (double)f[i] + tf);
  for (int j = threadIdx.x; j < m; j += blockDim.x) gmn = fmin(gmn, (double)g[j] + tg);
  fmn = block_reduce(fmn, s_x, MinOp(), CUDART_INF);
  gmn = block_reduce(gmn, s_x, MinOp(), CUDART_INF);
  const double lo_dom = e1 == UOT_ENT_BERG ? -r1 - fmn : -CUDART_INF;
  const double hi_dom = e2 == UOT_ENT_BERG ? r2 + gmn : CUDART_INF;
  // NewtonError cases of src/duality.py:182-247 (codes as uot_translation):
  // the problem stops (done) and the status goes to the caller.
  auto fail = [&](int code) {
    if (threadIdx.x == 0) {
      if (status != nullptr) status[b] = code;
      done[b] = 1;
    }
  };
  if (!(lo_dom < hi_dom)) {  // :188-189 empty translation domain
    fail(1);
    return;
  }
  auto clamp = [&](double x) {
    if (lo_dom > -CUDART_INF) x = fmax(x, lo_dom + 1e-12 * fmax(1.0, fabs(lo_dom)));
    if (hi_dom < CUDART_INF) x = fmin(x, hi_dom - 1e-12 * fmax(1.0, fabs(hi_dom)));
    return x;
  };
  // residual and slope at lam (block-uniform results)
  auto eval = [&](double lam, double& res, double& slope) {
    double s1 = 0.0, s2 = 0.0, h1 = 0.0, h2 = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double w = (double)a[i];
      if (w > 0.0) {
        const double xv = -((double)f[i] + tf) - lam;
        s1 += w * conj_grad_d(e1, r1, xv);
        h1 += w * conj_hess_d(e1, r1, xv);
      }
    }
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      const double w = (double)bw[j];
      if (w > 0.0) {
        const double xv = -((double)g[j] + tg) + lam;
        s2 += w * conj_grad_d(e2, r2, xv);
        h2 += w * conj_hess_d(e2, r2, xv);
      }
    }
    s1 = block_reduce(s1, s_x, SumOp(), 0.0);
    s2 = block_reduce(s2, s_x, SumOp(), 0.0);
    h1 = block_reduce(h1, s_x, SumOp(), 0.0);
    h2 = block_reduce(h2, s_x, SumOp(), 0.0);
    res = s1 - s2;
    slope = -h1 - h2;
  };
  const double tol = 1e-11;
  double lam = clamp(sc[b].lam), r, ds;
  eval(lam, r, ds);
  if (fabs(r) >= tol) {
    double lo = lam, hi = lam, step = 1.0;
    bool bracketed = false;
    if (r > 0.0) {
      for (int it = 0; it < 200 && !bracketed; ++it) {
        hi = clamp(lam + step);
        double rh, dh;
        eval(hi, rh, dh);
        bracketed = rh <= 0.0;
        step *= 2.0;
      }
    } else {
      for (int it = 0; it < 200 && !bracketed; ++it) {
        lo = clamp(lam - step);
        double rl, dl;
        eval(lo, rl, dl);
        bracketed = rl >= 0.0;
        step *= 2.0;
      }
    }
    if (!bracketed) {  // :220-229 failed to bracket
      fail(2);
      return;
    }
    double x = 0.5 * (lo + hi);
    bool conv = false;
    for (int it = 0; it < 100; ++it) {
      eval(x, r, ds);
      if (fabs(r) < tol) {
        conv = true;
        break;
      }
      if (r > 0.0)
        lo = x;
      else
        hi = x;
      const double nt = (ds < 0.0 && isfinite(ds)) ? x - r / ds : CUDART_NAN;
      x = (nt > lo && nt < hi) ? nt : 0.5 * (lo + hi);
    }
    if (!conv) {  // :247 no convergence
      fail(3);
      return;
    }
    lam = x;
  }
  if (threadIdx.x == 0) sc[b].lam = lam;
  (void)s_r;
}

// ---------------------------------------------------------------------------
// Tail kernel.

constexpr int TAIL_THREADS = 256;

template <class P>
__global__ void __launch_bounds__(TAIL_THREADS) sk_tail(TailArgs<typename P::T> A) {
  using T = typename P::T;
  using D = Dom<T>;
  const int b = blockIdx.y;
  if (A.done != nullptr && A.done[b]) return;
  __shared__ double s_m[32], s_s[32], s_x[32];
  __shared__ int s_last;
  const int o = blockIdx.x * TAIL_THREADS + threadIdx.x;
  const bool ok = o < A.nout;
  const SkScalars sc = A.sc[b];
  double tau_red = sc.tau[A.red_side];
  double shat_red = sc.shat[A.red_side];
  double delta_red = 0.0;
  if (A.shard == 2) {
    // resolve the reduced side's scalars from every rank's published partials
    LsePair q{-CUDART_INF, 0.0};
    double qmax = -CUDART_INF, qmin = CUDART_INF;
    for (int r = 0; r < A.nranks; ++r) {
      const double* x = A.xs_in + (long)r * A.xs_stride + (long)b * 4;
      q = lse_merge(q, LsePair{x[0], x[1]});
      qmax = fmax(qmax, x[2]);
      qmin = fmin(qmin, x[3]);
    }
    shat_red = -A.rho_red * (q.m + log(q.s));
    tau_red = A.first ? 0.0 : A.tau_fac_red * shat_red;
    delta_red = fmax(qmax + tau_red, -(qmin + tau_red));
  }
  const double smin_red = shat_red + tau_red;
  const double tau_old = sc.tau[A.out_side];

  LsePair pr{-CUDART_INF, 0.0};
  double dmax = -CUDART_INF, dmin = CUDART_INF;
  if (ok) {
    double hat;
    if (A.mode == 1) {
      hat = (double)A.pot_in[(long)b * A.nout + o];
    } else {
      // fold the split partials (shift, sum): max, then the rescaled sum
      // (loads unrolled for memory-level parallelism; fp32 partials combine
      // with the fast exp2 -- they carry fp32 precision anyway)
      T M = (T)(-CUDART_INF);
      const long pbase = (long)b * A.pstride_b + o;
#pragma unroll 4
      for (int s = 0; s < A.nparts; ++s) {
        const T a = A.part_a[pbase + (long)s * A.pstride_s];
        const T mm = A.part_m[pbase + (long)s * A.pstride_s];
        if (a > (T)0) M = mm > M ? mm : M;
      }
      T acc = 0;
#pragma unroll 4
      for (int s = 0; s < A.nparts; ++s) {
        const T a = A.part_a[pbase + (long)s * A.pstride_s];
        const T mm = A.part_m[pbase + (long)s * A.pstride_s];
        if (a > (T)0) acc += a * D::ex(mm - M);
      }
      const double lse = (double)M + D::lgd((double)acc);  // domain units, excluding tau_red
      A.shift_out[(long)b * A.nout + o] = (T)lse;
      const double smin = -A.eps * A.unit * (lse + tau_red * A.inv_eu);
      if (A.gmode) {
        // G (src/sinkhorn.py:128-132) at the incoming lam, any aprox:
        // g' = lam - aprox(eps, lam - smin_cols(f)), f' = -lam - aprox(eps, -smin_rows(g) - lam)
        const double lm = sc.lam;
        hat = A.out_side == 1 ? lm - aprox_any(A.ent_out, A.rho_out, A.eps, lm - smin)
                              : -lm - aprox_any(A.ent_out, A.rho_out, A.eps, -smin - lm);
      } else if (A.ent_out == UOT_ENT_KL) {
        hat = A.a_coef * smin - A.k_coef * smin_red;
      } else {
        hat = -aprox_any(A.ent_out, A.rho_out, A.eps, -smin);  // F step, :111-113
      }
    }
    const T hat_t = (T)hat;
    hat = (double)hat_t;
    A.hat_out[(long)b * A.nout + o] = hat_t;
    const double w = (double)A.out_w[(long)b * A.nout + o];
    RecLayout<P>::pack(A.rec_out + (long)b * A.rec_bstride, o, A.rw, hat,
                       A.out_pts + ((long)b * A.nout + o) * A.d, w, (double)A.L, (double)A.p,
                       A.d, A.ctr != nullptr ? A.ctr + (long)b * A.d : nullptr);
    if (w > 0.0) pr = LsePair{-hat / A.rho_out, w};
    if (A.hat_old != nullptr) {
      const double dl = hat - ((double)A.hat_old[(long)b * A.nout + o] + tau_old);
      dmax = dl;
      dmin = dl;
    }
  }
  // Block partials: log-sum-exp of -hat/rho weighted by w, and delta bounds.
  pr = block_lse_ms(pr, s_x);
  dmax = block_reduce(dmax, s_x, MaxOp(), -CUDART_INF);
  dmin = block_reduce(dmin, s_x, MinOp(), CUDART_INF);
  double* blk = A.blk + (long)b * gridDim.x * 4;
  if (threadIdx.x == 0) {
    blk[blockIdx.x * 4 + 0] = pr.m;
    blk[blockIdx.x * 4 + 1] = pr.s;
    blk[blockIdx.x * 4 + 2] = dmax;
    blk[blockIdx.x * 4 + 3] = dmin;
  }
  if (!last_block_arrive(A.counter + b, gridDim.x, &s_last)) return;
  // Last block: fold the per-block partials (fixed order -> deterministic).
  LsePair q{-CUDART_INF, 0.0};
  double qmax = -CUDART_INF, qmin = CUDART_INF;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += TAIL_THREADS) {
    q = lse_merge(q, LsePair{blk[k * 4 + 0], blk[k * 4 + 1]});
    qmax = fmax(qmax, blk[k * 4 + 2]);
    qmin = fmin(qmin, blk[k * 4 + 3]);
  }
  q = block_lse_ms(q, s_x);
  qmax = block_reduce(qmax, s_x, MaxOp(), -CUDART_INF);
  qmin = block_reduce(qmin, s_x, MinOp(), CUDART_INF);
  if (threadIdx.x == 0 && A.shard == 1) {
    // publish this rank's partial scalars; resolved after the exchange
    A.xs_out[(long)b * 4 + 0] = q.m;
    A.xs_out[(long)b * 4 + 1] = q.s;
    A.xs_out[(long)b * 4 + 2] = qmax;
    A.xs_out[(long)b * 4 + 3] = qmin;
    A.counter[b] = 0u;
    return;
  }
  if (threadIdx.x == 0 && A.shard == 2) {
    A.sc[b].shat[A.red_side] = shat_red;
    A.sc[b].tau[A.red_side] = tau_red;
    if (!A.first && A.trace != nullptr) A.trace[(long)b * A.trace_len + A.t - 1] = delta_red;
  }
  if (threadIdx.x == 0) {
    const double shat = -A.rho_out * (q.m + log(q.s));
    const double tau = (A.mode == 1) ? 0.0 : A.tau_fac * shat;
    A.sc[b].shat[A.out_side] = shat;
    A.sc[b].tau[A.out_side] = tau;
    if (A.gmode && A.lam_closed && A.out_side == 0) {
      // lambda* of the new pair (duality.py:175-178) from the softmins
      // S = Smin(hat) + tau of both sides: (rho1 S_g - rho2 S_f) / (rho1 + rho2)
      const double Sf = shat + tau, Sg = A.sc[b].shat[1] + A.sc[b].tau[1];
      A.sc[b].lam = (A.rho1 * Sg - A.rho2 * Sf) / (A.rho1 + A.rho2);
    }
    if (A.hat_old != nullptr && A.trace != nullptr) {
      const double delta = fmax(qmax + tau, -(qmin + tau));
      const int tt = A.t_dev ? A.iters_done[b] : A.t;  // replayed graphs carry no t
      A.trace[(long)b * A.trace_len + tt] = delta;
      A.iters_done[b] = tt + 1;
      if (A.use_tol && delta < A.tol) A.done[b] = 1;
    }
    A.counter[b] = 0u;
  }
}

// ---------------------------------------------------------------------------
// Verification at scale (§8f row 3): one side of a given pair (f, g).  After
// a main pass that reduced the OTHER side's records over every output o,
// folds the split partials into smin_o (src/sinkhorn.py:93-100) and per
// problem reduces (one CTA per problem):
//   res = max_o |pot_o - a smin_o + sgn (eps/(eps+rho)) lam|   (:166-189)
//   L   = LSE_o(-smin_o/eps + pot_o/eps; w)  -- the log of <a x b, e^((f+g-C)/eps)>
//         (duality.py:124-132) when this is the target side.
// gridDim.x CTAs per problem (blockIdx.y) each fold a strided share of the
// outputs into (res, L.m, L.s) at blk[(b * gridDim.x + blockIdx.x) * 4]; then
// sk_verify_fold writes out[b*8 + base + 0..1] = (res, L).  (One CTA per
// problem took 2.7 ms of a 3.7 ms pass at N = M = 65536.)
template <typename T>
__global__ void __launch_bounds__(256) sk_verify_side(int nout, int nparts, const T* part_m,
                                                     const T* part_a, const T* pot, const T* w,
                                                     double eps, double unit, double a_coef,
                                                     double lam_coef, const double* lam,
                                                     double* blk) {
  using D = Dom<T>;
  __shared__ double s_m[32], s_s[32], s_x[32];
  const int b = blockIdx.y;
  const long pb = (long)b * nparts * nout;
  const double lm = lam[b];
  double res = 0.0;
  LsePair L{-CUDART_INF, 0.0};
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double M = -CUDART_INF;
    for (int s = 0; s < nparts; ++s) {
      const double a = (double)part_a[pb + (long)s * nout + o];
      if (a > 0.0) M = fmax(M, (double)part_m[pb + (long)s * nout + o]);
    }
    double acc = 0.0;
    for (int s = 0; s < nparts; ++s) {
      const double a = (double)part_a[pb + (long)s * nout + o];
      if (a > 0.0) acc += a * D::exd((double)part_m[pb + (long)s * nout + o] - M);
    }
    const double lse = M + D::lgd(acc);  // domain units
    const double smin = -eps * unit * lse;
    const double pv = (double)pot[(long)b * nout + o];
    res = fmax(res, fabs(pv - a_coef * smin + lam_coef * lm));
    const double wv = (double)w[(long)b * nout + o];
    if (wv > 0.0) L = lse_merge(L, LsePair{unit * lse + pv / eps, wv});
  }
  res = block_reduce(res, s_x, MaxOp(), 0.0);
  L = block_lse(L, s_m, s_s);
  if (threadIdx.x == 0) {
    double* p = blk + ((long)b * gridDim.x + blockIdx.x) * 4;
    p[0] = res;
    p[1] = L.m;
    p[2] = L.s;
  }
}

__global__ void __launch_bounds__(256) sk_verify_fold(int nb, const double* blk, double* out,
                                                     int base) {
  __shared__ double s_m[32], s_s[32], s_x[32];
  const int b = blockIdx.x;
  double res = 0.0;
  LsePair L{-CUDART_INF, 0.0};
  for (int k = threadIdx.x; k < nb; k += blockDim.x) {
    const double* p = blk + ((long)b * nb + k) * 4;
    res = fmax(res, p[0]);
    if (p[2] > 0.0) L = lse_merge(L, LsePair{p[1], p[2]});
  }
  res = block_reduce(res, s_x, MaxOp(), 0.0);
  L = block_lse(L, s_m, s_s);
  if (threadIdx.x == 0) {
    out[(long)b * 8 + base + 0] = res;
    out[(long)b * 8 + base + 1] = L.m + log(L.s);
  }
}

// KL parts of the objectives and lambda* from the init tails' softmins.
__global__ void sk_verify_kl(int batch, int n, int m, const SkScalars* sc, double rho1,
                             double rho2, double* lam) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  // Smin(f) = shat[0], Smin(g) = shat[1] (tau = 0 after init tails)
  lam[b] = (rho1 * sc[b].shat[1] - rho2 * sc[b].shat[0]) / (rho1 + rho2);
}

__global__ void sk_verify_pack(int batch, const SkScalars* sc, const double* lam, double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  out[(long)b * 8 + 4] = lam[b];
  out[(long)b * 8 + 5] = sc[b].shat[0];
  out[(long)b * 8 + 6] = sc[b].shat[1];
}

// Final pair: f = hat_f + tau_f, g = hat_g + tau_g (src/sinkhorn.py returns
// the plain potentials, :163).
template <typename T>
__global__ void sk_finalize(int n, int m, const T* hatA0, const T* hatA1, const T* hatB,
                            const SkScalars* sc, const int* iters_done, T* f, T* g) {
  const int b = blockIdx.y;
  const T* hatA = (iters_done[b] & 1) ? hatA1 : hatA0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max(n, m); i += gridDim.x * blockDim.x) {
    if (i < n) f[(long)b * n + i] = (T)((double)hatA[(long)b * n + i] + sc[b].tau[0]);
    if (i < m) g[(long)b * m + i] = (T)((double)hatB[(long)b * m + i] + sc[b].tau[1]);
  }
}

// Row sharding, phase 1: fold this rank's split partials into one
// (shift, sum) pair per output (the payload of the all-gather).
template <typename T>
__global__ void sk_combine(int nout, int S, const T* part_m, const T* part_a, T* out_m, T* out_a,
                           int o_lo, int o_hi) {
  using D = Dom<T>;
  const int b = blockIdx.y;
  const int o = o_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= o_hi) return;
  const long pb = (long)b * S * nout + o;
  double M = -CUDART_INF;
  for (int s = 0; s < S; ++s)
    if ((double)part_a[pb + (long)s * nout] > 0.0) M = fmax(M, (double)part_m[pb + (long)s * nout]);
  double acc = 0.0;
  for (int s = 0; s < S; ++s) {
    const double a = (double)part_a[pb + (long)s * nout];
    if (a > 0.0) acc += a * D::exd((double)part_m[pb + (long)s * nout] - M);
  }
  out_m[(long)b * nout + o] = (T)M;
  out_a[(long)b * nout + o] = (T)acc;
}

// Row sharding, end of run: resolve the last f-side scalars from the
// gathered slots (same arithmetic as the shard == 2 tail).
__global__ void sk_resolve_final(int batch, int nranks, const double* xs, long xs_stride,
                                 double rho1, double tau_fac, SkScalars* sc, double* trace,
                                 int trace_len, int t_last, int* iters_done) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  LsePair q{-CUDART_INF, 0.0};
  double qmax = -CUDART_INF, qmin = CUDART_INF;
  for (int r = 0; r < nranks; ++r) {
    const double* x = xs + (long)r * xs_stride + (long)b * 4;
    q = lse_merge(q, LsePair{x[0], x[1]});
    qmax = fmax(qmax, x[2]);
    qmin = fmin(qmin, x[3]);
  }
  const double shat = -rho1 * (q.m + log(q.s));
  const double tau = tau_fac * shat;
  sc[b].shat[0] = shat;
  sc[b].tau[0] = tau;
  if (trace != nullptr) trace[(long)b * trace_len + t_last] = fmax(qmax + tau, -(qmin + tau));
  iters_done[b] = t_last + 1;
}

__global__ void sk_reset(int batch, SkScalars* sc, unsigned int* counters, int* done,
                         int* iters_done) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) {
    sc[b] = SkScalars{{0.0, 0.0}, {0.0, 0.0}, 0.0};
    counters[b] = 0u;
    done[b] = 0;
    iters_done[b] = 0;
  }
}

__global__ void sk_set_lam(int batch, SkScalars* sc, double lam) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) sc[b].lam = lam;
}

template <typename T>
__global__ void sk_zero(long n, T* p) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[i] = T(0);
}

// Stale shifts of a verification pass from the pair being verified: at a KL
// fixed point g = a2 * smin_cols(f) (+ a constant for the H variant), so the
// column log-sum-exps are about -g / (a2 eps unit) -- close enough (the safe
// window is 2^+-100) for the main kernels' fast path; a pair far from any
// fixed point just sends the tiles down the checked path as a zero shift does.
template <typename T>
__global__ void sk_shift_guess(long n, const T* pot, double coef, T* shift) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double v = -(double)pot[i] * coef;
    shift[i] = (v == v && fabs(v) < 1e30) ? (T)v : T(0);
  }
}

// ---------------------------------------------------------------------------
// Host engine.

namespace {

struct WsLayout {
  size_t off[18];
  size_t total;
};

template <typename T>
struct Buffers {
  T* recA;
  T* recB;
  T* hatA0;
  T* hatA1;
  T* hatB;
  T* shiftA;
  T* shiftB;
  T* part_m;
  T* part_a;
  T* zeros;  // [B][max(n,m)] initial potential when none is given
  SkScalars* sc;
  double* blk;
  unsigned int* counter;
  int* done;
  int* iters_done;
  double* trace;  // scratch trace when the caller passes none
  T* ctr;         // [B][d] centre of the tcgen05 operands (tc_center)
  uint32_t* packA;  // tcgen05 path: precomputed A rows of the sources [B][n][W] (tc_pack_out)
  uint32_t* packB;  // ... of the targets [B][m][W]
};

struct Shape {
  int B, n, m, d, rwA, rwB, S, nblk;
  int total_n;  // all shards (emulation)
  long recA, recB;  // record elements per problem
  int pack_w = 0;   // tcgen05 path: words per precomputed A row (0: none)
};

template <typename T>
size_t layout(const Shape& s, int iters, WsLayout& L, Buffers<T>* buf, char* base) {
  size_t sizes[18];
  const long nm = std::max(s.total_n, s.m);
  sizes[0] = sizeof(T) * (size_t)s.B * s.recA;
  sizes[1] = sizeof(T) * (size_t)s.B * s.recB;
  sizes[2] = sizeof(T) * (size_t)s.B * s.total_n;
  sizes[3] = sizes[2];
  sizes[4] = sizeof(T) * (size_t)s.B * s.m;
  sizes[5] = sizes[2];
  sizes[6] = sizes[4];
  sizes[7] = sizeof(T) * (size_t)s.B * s.S * nm;
  sizes[8] = sizes[7];
  sizes[9] = sizeof(T) * (size_t)s.B * nm;
  sizes[10] = sizeof(SkScalars) * (size_t)s.B;
  sizes[11] = sizeof(double) * 4 * (size_t)s.B * s.nblk;
  sizes[12] = sizeof(unsigned int) * (size_t)s.B;
  sizes[13] = sizeof(int) * (size_t)s.B;
  sizes[14] = sizeof(int) * (size_t)s.B;
  sizes[15] = sizeof(double) * (size_t)s.B * std::max(iters, 1);
  sizes[16] = sizeof(T) * (size_t)s.B * std::max(s.d, 4);
  sizes[17] = sizeof(uint32_t) * (size_t)s.B * (s.total_n + s.m) * s.pack_w;
  size_t off = 0;
  for (int k = 0; k < 18; ++k) {
    L.off[k] = off;
    off += (sizes[k] + 255) / 256 * 256;
  }
  L.total = off;
  if (buf != nullptr) {
    buf->recA = (T*)(base + L.off[0]);
    buf->recB = (T*)(base + L.off[1]);
    buf->hatA0 = (T*)(base + L.off[2]);
    buf->hatA1 = (T*)(base + L.off[3]);
    buf->hatB = (T*)(base + L.off[4]);
    buf->shiftA = (T*)(base + L.off[5]);
    buf->shiftB = (T*)(base + L.off[6]);
    buf->part_m = (T*)(base + L.off[7]);
    buf->part_a = (T*)(base + L.off[8]);
    buf->zeros = (T*)(base + L.off[9]);
    buf->sc = (SkScalars*)(base + L.off[10]);
    buf->blk = (double*)(base + L.off[11]);
    buf->counter = (unsigned int*)(base + L.off[12]);
    buf->done = (int*)(base + L.off[13]);
    buf->iters_done = (int*)(base + L.off[14]);
    buf->trace = (double*)(base + L.off[15]);
    buf->ctr = (T*)(base + L.off[16]);
    buf->packA = s.pack_w > 0 ? (uint32_t*)(base + L.off[17]) : nullptr;
    buf->packB = s.pack_w > 0 ? buf->packA + (size_t)s.B * s.total_n * s.pack_w : nullptr;
  }
  return L.total;
}

template <class P>
struct Cfg;
#ifndef SQ2_THREADS
#define SQ2_THREADS 128
#endif
#ifndef SQ2_RT
#define SQ2_RT 8
#endif
template <int D>
struct Cfg<SqE32<D>> {
  static constexpr int THREADS = SQ2_THREADS, COLS = 4, RT = SQ2_RT;
};
template <>
struct Cfg<SqE32N> {
  static constexpr int THREADS = 128, COLS = 2, RT = 4;
};
template <>
struct Cfg<Pow1D<float>> {
  static constexpr int THREADS = 128, COLS = 4, RT = 8;
};
template <>
struct Cfg<Pow1D<double>> {
  static constexpr int THREADS = 128, COLS = 2, RT = 4;
};
template <>
struct Cfg<SqE64> {
  static constexpr int THREADS = 128, COLS = 2, RT = 4;
};
template <>
struct Cfg<SqE32TC> {
  static constexpr int THREADS = 128, COLS = 2, RT = 1;  // 256 outputs per CTA (two MMA blocks)
};
template <typename TT>
struct Cfg<Explicit<TT>> {
  static constexpr int THREADS = 128, COLS = 2, RT = 4;
};

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Splits of the reduced index: the main grid (out_blocks x splits x batch)
// should fill the chip about four times over with whole waves of
// (SMs x resident CTAs per SM), while keeping >= 16 reduced indices per split.
int choose_splits(int B, long nout, long nred, int out_per_block, int occ = 0) {
  const long out_blocks = (nout + out_per_block - 1) / out_per_block;
  static const long rows_min = [] {  // rows per split floor (UOT_SPLIT_ROWS: tuning only)
    const char* e = std::getenv("UOT_SPLIT_ROWS");
    return e ? std::max(1L, std::atol(e)) : 16L;
  }();
  const long s_max = std::min(4096L, std::max(1L, nred / rows_min));
  if (occ <= 0) {
    const long target = (long)num_sms() * 24;
    long s = (target + out_blocks * B - 1) / (out_blocks * B);
    return (int)std::max(1L, std::min(s, s_max));
  }
  const long wave = (long)num_sms() * occ;
  const long s0 = std::max(1L, (4 * wave + out_blocks * B - 1) / (out_blocks * B));
  long best_s = std::min(s0, s_max);
  double best_eff = -1.0;
  for (long sv = std::max(1L, s0 / 2); sv <= std::min(s_max, 2 * s0); ++sv) {
    const long total = out_blocks * sv * B;
    const long waves = (total + wave - 1) / wave;
    const double eff = (double)total / (double)(waves * wave);
    if (eff > best_eff + 0.005) {
      best_eff = eff;
      best_s = sv;
    }
  }
  return (int)best_s;
}

template <class P>
struct Engine {
  using T = typename P::T;
  using C = Cfg<P>;
  static constexpr int OUT_PER_BLOCK = C::THREADS * C::COLS;

  static int occupancy(int d) {
    // per host thread: concurrent callers with different d never share the pair
    static thread_local int cached = -1;
    static thread_local int cached_d = -1;
    if (cached >= 0 && cached_d == d) return cached;
    const int rw = P::rw(d);
    const size_t smem = (size_t)chunk_for(rw) * rw * sizeof(T);
    int occ = 0;
    cudaError_t e;
    if constexpr (std::is_same<P, SqE32TC>::value) {
      cached = 1;  // TMEM (512 columns) is allocated whole: one CTA per SM
      cached_d = d;
      return 1;
    } else if constexpr (std::is_same<P, SqE32<2>>::value)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &occ, sk_main_sq2<C::THREADS, C::COLS / 2, C::RT>, C::THREADS, smem);
    else
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sk_main<P, C::THREADS, C::COLS, C::RT>,
                                                        C::THREADS, smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      occ = 0;
    }
    cached = occ;
    cached_d = d;
    return occ;
  }

  static int splits(int B, long nout, long nred, int d) {
    return choose_splits(B, nout, nred, OUT_PER_BLOCK, occupancy(d));
  }

  static int chunk_for(int rw) {
    int ch = (int)(32768 / (rw * sizeof(T)));
    ch = std::max(16, std::min(1024, ch));
    return ch / 8 * 8;
  }

  static Shape shape(const uot_sinkhorn_desc& d) {
    Shape s;
    s.B = d.batch;
    s.n = d.n;
    s.m = d.m;
    s.d = d.d;
    s.rwA = P::rw(d.d);
    s.rwB = P::rw(d.d);
    s.total_n = d.n;
    s.recA = RecLayout<P>::stride(d.n, d.d);
    s.recB = RecLayout<P>::stride(d.m, d.d);
    const int sA = splits(d.batch, d.m, d.n, d.d);
    const int sB = splits(d.batch, d.n, d.m, d.d);
    s.S = std::max(sA, sB);
    if (d.nranks > 1 && d.nccl_comm == nullptr) s.S = std::max(s.S, d.nranks);
    s.nblk = (int)ceil_div(std::max(d.n, d.m), TAIL_THREADS);
    if constexpr (std::is_same<P, SqE32TC>::value)
      s.pack_w = std::getenv("UOT_TC_NOPACK") == nullptr ? tc_pack_words(d.d) : 0;
    return s;
  }

  static size_t ws_size(const uot_sinkhorn_desc& d) {
    if (d.nranks > 1 || d.nccl_comm != nullptr) return ws_size_sharded(d);
    WsLayout L;
    Shape s = shape(d);
    return layout<T>(s, d.iters, L, nullptr, nullptr);
  }

  static int launch_main(const uot_sinkhorn_desc& d, const Buffers<T>& bf, cudaStream_t st,
                         bool to_target, int splits, int red_offset, int nred, int split_base,
                         int splits_total, int out_lo = 0, int out_hi = 0) {
    MainArgs<T> a{};
    a.out_lo = out_lo;
    a.out_hi = out_hi;
    const double L = 1.0 / (d.eps * Dom<T>::unit);
    a.g.rw = P::rw(d.d);
    a.g.d = d.d;
    a.g.L = (T)L;
    a.g.p = (T)d.p;
    if (to_target) {  // g-update: reduce over the source side, outputs = targets
      a.g.red_rec = bf.recA;
      a.g.red_bstride = RecLayout<P>::stride(d.n, d.d);
      a.g.out_pts = (const T*)d.y;
      a.g.out_pts_bstride = (long)d.m * d.d;
      a.g.cmat = (const T*)d.c;
      a.g.cm_bstride = (long)d.n * d.m;
      a.g.ld_r = d.m;
      a.g.ld_o = 1;
      a.nout = d.m;
      a.shift_in = bf.shiftB;
    } else {  // f-update: reduce over the target side, outputs = sources
      a.g.red_rec = bf.recB;
      a.g.red_bstride = RecLayout<P>::stride(d.m, d.d);
      a.g.out_pts = (const T*)d.x;
      a.g.out_pts_bstride = (long)d.n * d.d;
      a.g.cmat = (const T*)d.ct;
      a.g.cm_bstride = (long)d.n * d.m;
      a.g.ld_r = d.n;
      a.g.ld_o = 1;
      a.nout = d.n;
      a.shift_in = bf.shiftA;
    }
    a.g.ctr = bf.ctr;
    a.g.ctr_bstride = d.d;
    a.g.ascale = (T)tc_ascale((double)(float)L);
    a.g.tc_full = 2.0 * (double)(float)L > 128.0 ? 1 : 0;
    a.g.tc_pack = to_target ? bf.packB : bf.packA;
    a.g.tc_pack_bstride = (long)(to_target ? d.m : d.n) * tc_pack_words(d.d);
    a.nred = nred;
    a.red_offset = red_offset;
    a.part_m = bf.part_m;
    a.part_a = bf.part_a;
    a.done = bf.done;
    a.chunk = chunk_for(a.g.rw);
    a.split_base = split_base;
    a.splits_total = splits_total;
    dim3 grid(ceil_div((out_hi > 0 ? out_hi : a.nout) - out_lo, OUT_PER_BLOCK), splits, d.batch);
    const size_t smem = (size_t)a.chunk * a.g.rw * sizeof(T);
    if constexpr (std::is_same<P, SqE32TC>::value) {
      const size_t tsm = tc_smem_bytes(d.d);
      auto go = [&](auto kern) -> int {
        UOT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)tsm));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((grid.x + 1) / 2 * 2, grid.y, grid.z);  // whole CTA pairs
        cfg.blockDim = dim3(TC_THREADS, 1, 1);
        cfg.dynamicSmemBytes = tsm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        UOT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, tc_kp(d.d)));
        return UOT_OK;
      };
      int rc;
      switch (d.d) {
        case 32: rc = go(sk_main_tc<32>); break;
        case 48: rc = go(sk_main_tc<48>); break;
        case 64: rc = go(sk_main_tc<64>); break;
        case 96: rc = go(sk_main_tc<96>); break;
        default: rc = go(sk_main_tc<0>); break;
      }
      if (rc != UOT_OK) return rc;
    } else if constexpr (std::is_same<P, SqE32<2>>::value) {
      static_assert(C::COLS % 2 == 0, "packed kernel needs an even column count");
      sk_main_sq2<C::THREADS, C::COLS / 2, C::RT><<<grid, C::THREADS, smem, st>>>(a);
    } else {
      sk_main<P, C::THREADS, C::COLS, C::RT><<<grid, C::THREADS, smem, st>>>(a);
    }
    UOT_CHECK_LAUNCH();
    return UOT_OK;
  }

  struct ShardOpt {
    int shard;
    const double* xs_in;
    long xs_stride;
    int nranks;
    int first;
    double* xs_out;
    const T* pm;
    const T* pa;
    long pstride_s, pstride_b;
  };

  static int launch_tail(const uot_sinkhorn_desc& d, const Buffers<T>& bf, cudaStream_t st,
                         bool to_target, int mode, int nparts, const T* hat_old, T* hat_out,
                         const T* pot_in, int t, double* trace, int trace_len,
                         const ShardOpt* so = nullptr, int t_dev = 0) {
    TailArgs<T> a{};
    a.t_dev = t_dev;
    const bool H = d.variant == UOT_SINKHORN_H;
    const double eps = d.eps, r1 = d.rho1, r2 = d.rho2;
    const double ro = to_target ? r2 : r1;        // own marginal strength
    const double rother = to_target ? r1 : r2;    // the other marginal
    a.nout = to_target ? d.m : d.n;
    a.nparts = nparts;
    a.mode = mode;
    a.out_side = to_target ? 1 : 0;
    a.red_side = to_target ? 0 : 1;
    a.part_m = bf.part_m;
    a.part_a = bf.part_a;
    a.pstride_s = a.nout;
    a.pstride_b = (long)nparts * a.nout;
    a.pot_in = pot_in;
    a.sc = bf.sc;
    a.eps = eps;
    a.unit = Dom<T>::unit;
    a.inv_eu = 1.0 / (eps * Dom<T>::unit);
    // src/sinkhorn.py:154-162: hat = rho/(rho+eps) smin - (eps/(eps+rho)) (rho/(r1+r2)) Smin_other
    a.a_coef = ro / (ro + eps);
    a.k_coef = H ? (eps / (eps + ro)) * (ro / (r1 + r2)) : 0.0;
    const double kk = (eps / (eps + ro)) * (rother / (r1 + r2));
    a.tau_fac = H ? kk / (1.0 - kk) : 0.0;
    a.gmode = d.variant == UOT_SINKHORN_G ? 1 : 0;
    a.rho1 = r1;
    a.rho2 = r2;
    a.ent_out = to_target ? d.ent2 : d.ent1;
    a.lam_closed = (d.ent1 == UOT_ENT_KL && d.ent2 == UOT_ENT_KL) ? 1 : 0;
    if (a.ent_out == UOT_ENT_BALANCED) a.a_coef = 1.0;
    a.rho_out = ro;
    a.hat_out = hat_out;
    a.hat_old = hat_old;
    a.shift_out = to_target ? bf.shiftB : bf.shiftA;
    a.rec_out = to_target ? bf.recB : bf.recA;
    a.rec_bstride = RecLayout<P>::stride(to_target ? d.m : d.n, d.d);
    a.rw = P::rw(d.d);
    a.out_pts = (const T*)(to_target ? d.y : d.x);
    a.ctr = centred<P>() ? bf.ctr : nullptr;
    a.d = d.d;
    a.out_w = (const T*)(to_target ? d.b : d.a);
    a.L = (T)(1.0 / (eps * Dom<T>::unit));
    a.p = (T)d.p;
    a.blk = bf.blk;
    a.counter = bf.counter;
    a.trace = trace;
    a.trace_len = trace_len;
    a.t = t;
    a.iters_done = bf.iters_done;
    a.done = bf.done;
    a.tol = d.tol;
    a.use_tol = d.use_tol;
    if (so != nullptr) {
      a.shard = so->shard;
      a.xs_in = so->xs_in;
      a.xs_stride = so->xs_stride;
      a.nranks = so->nranks;
      a.first = so->first;
      a.xs_out = so->xs_out;
      if (so->pm != nullptr) {
        a.part_m = so->pm;
        a.part_a = so->pa;
        a.pstride_s = so->pstride_s;
        a.pstride_b = so->pstride_b;
      }
      // reduced side of the g-update is the (sharded) source side
      a.rho_red = r1;
      const double kka = (eps / (eps + r1)) * (r2 / (r1 + r2));
      a.tau_fac_red = H ? kka / (1.0 - kka) : 0.0;
    }
    dim3 grid(ceil_div(a.nout, TAIL_THREADS), d.batch);
    sk_tail<P><<<grid, TAIL_THREADS, 0, st>>>(a);
    UOT_CHECK_LAUNCH();
    return UOT_OK;
  }

  static int run(const uot_sinkhorn_desc& d, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (d.nranks > 1 || d.nccl_comm != nullptr) return run_sharded(d, ws, ws_bytes, st);
    Shape s = shape(d);
    WsLayout L;
    Buffers<T> bf;
    const size_t need = layout<T>(s, d.iters, L, &bf, (char*)ws);
    if (ws_bytes < need) {
      set_error("sinkhorn workspace too small: %zu < %zu", ws_bytes, need);
      return UOT_INVALID;
    }
    sk_reset<<<ceil_div(d.batch, 128), 128, 0, st>>>(d.batch, bf.sc, bf.counter, bf.done,
                                                      bf.iters_done);
    UOT_CHECK_LAUNCH();
    UOT_TRY(launch_center<P>(d, reinterpret_cast<float*>(bf.ctr), st));
    if constexpr (std::is_same<P, SqE32TC>::value) {
      tc_fill_dead<<<1024, 256, 0, st>>>(bf.recA, (long)d.batch * s.recA / tc_kp(d.d), d.d,
                                         tc_kp(d.d));
      tc_fill_dead<<<1024, 256, 0, st>>>(bf.recB, (long)d.batch * s.recB / tc_kp(d.d), d.d,
                                         tc_kp(d.d));
      // same fp32-rounded L as the tails' record packing
      const double Lr = (double)(float)(1.0 / (d.eps * Dom<float>::unit));
      const double Sa = tc_ascale(Lr);
      tc_init_static<<<1024, 256, 0, st>>>(bf.recA, s.recA, (const float*)d.x,
                                           (const float*)bf.ctr, (long)d.d, d.batch, d.n,
                                           d.d, tc_kp(d.d), Lr, Sa);
      tc_init_static<<<1024, 256, 0, st>>>(bf.recB, s.recB, (const float*)d.y,
                                           (const float*)bf.ctr, (long)d.d, d.batch, d.m,
                                           d.d, tc_kp(d.d), Lr, Sa);
      if (bf.packA != nullptr) {
        tc_pack_out<<<1024, 256, 0, st>>>(bf.packA, (const float*)d.x, (const float*)bf.ctr,
                                          (long)d.d, d.batch, d.n, d.d, (float)Sa);
        tc_pack_out<<<1024, 256, 0, st>>>(bf.packB, (const float*)d.y, (const float*)bf.ctr,
                                          (long)d.d, d.batch, d.m, d.d, (float)Sa);
      }
      UOT_CHECK_LAUNCH();
    }
    const long nm = std::max(d.n, d.m);
    if (!d.warm_shifts) {  // else: the previous call's log-sum-exps (same problem, same ws)
      sk_zero<T><<<256, 256, 0, st>>>((long)d.batch * s.n, bf.shiftA);
      sk_zero<T><<<256, 256, 0, st>>>((long)d.batch * s.m, bf.shiftB);
      UOT_CHECK_LAUNCH();
    }
    const T* f0 = (const T*)d.f;
    if (!d.init_given) {
      sk_zero<T><<<256, 256, 0, st>>>((long)d.batch * nm, bf.zeros);
      UOT_CHECK_LAUNCH();
      f0 = bf.zeros;
    }
    double* trace = d.trace_delta != nullptr ? d.trace_delta : bf.trace;
    const int trace_len = std::max(d.iters, 1);
    if (d.variant == UOT_SINKHORN_G) {
      // G starts from lambda*(f0, g0) (src/sinkhorn.py:263-265): Smin_b(g0)
      // first, the f0 init tail then forms lambda.
      const T* g0 = d.init_given ? (const T*)d.g : bf.zeros;
      if (d.init_given) {
        UOT_CUDA_TRY(cudaMemcpyAsync(bf.hatB, g0, sizeof(T) * (size_t)d.batch * d.m,
                                     cudaMemcpyDeviceToDevice, st));
        g0 = bf.hatB;
      } else {
        sk_zero<T><<<256, 256, 0, st>>>((long)d.batch * nm, bf.zeros);
        UOT_CHECK_LAUNCH();
      }
      UOT_TRY(launch_tail(d, bf, st, true, 1, 0, nullptr, bf.hatB, g0, 0, nullptr, trace_len));
    }
    // init: hat_f = f0, Smin_a(f0), pack source records.
    UOT_TRY(launch_tail(d, bf, st, false, 1, 0, nullptr, bf.hatA0, f0, 0, nullptr, trace_len));
    const bool g_newton =
        d.variant == UOT_SINKHORN_G && !(d.ent1 == UOT_ENT_KL && d.ent2 == UOT_ENT_KL);
    if (d.status != nullptr)
      UOT_CUDA_TRY(cudaMemsetAsync(d.status, 0, sizeof(int32_t) * (size_t)d.batch, st));
    auto lam_newton = [&](const T* hatA) -> int {
      sk_lambda_newton<T><<<d.batch, 256, 0, st>>>(d.n, d.m, hatA, bf.hatB, (const T*)d.a,
                                                   (const T*)d.b, d.ent1, d.ent2, d.rho1, d.rho2,
                                                   bf.sc, d.status, bf.done);
      UOT_CHECK_LAUNCH();
      return UOT_OK;
    };
    if (d.variant == UOT_SINKHORN_G && d.lam_given) {  // g_sinkhorn_step(prob, d, lam)
      sk_set_lam<<<ceil_div(d.batch, 128), 128, 0, st>>>(d.batch, bf.sc, d.lam0);
      UOT_CHECK_LAUNCH();
    } else if (g_newton) {
      UOT_TRY(lam_newton(bf.hatA0));  // lambda*(f0, g0) (:263-265)
    }
    const int sB = splits(d.batch, d.m, d.n, d.d);  // g-update splits
    const int sA = splits(d.batch, d.n, d.m, d.d);  // f-update splits
    // one iteration: two half-steps (main + tail each), hat buffers by parity
    auto body = [&](int t, cudaStream_t s, int t_dev) -> int {
      T* hat_old = (t & 1) ? bf.hatA1 : bf.hatA0;
      T* hat_new = (t & 1) ? bf.hatA0 : bf.hatA1;
      UOT_TRY(launch_main(d, bf, s, true, sB, 0, d.n, 0, sB));
      UOT_TRY(launch_tail(d, bf, s, true, 0, sB, nullptr, bf.hatB, nullptr, t, nullptr,
                          trace_len, nullptr, t_dev));
      UOT_TRY(launch_main(d, bf, s, false, sA, 0, d.m, 0, sA));
      UOT_TRY(launch_tail(d, bf, s, false, 0, sA, hat_old, hat_new, nullptr, t, trace,
                          trace_len, nullptr, t_dev));
      if (g_newton) {  // lambda_star(pair, initial=lam) (:134)
        sk_lambda_newton<T><<<d.batch, 256, 0, s>>>(d.n, d.m, hat_new, bf.hatB, (const T*)d.a,
                                                    (const T*)d.b, d.ent1, d.ent2, d.rho1, d.rho2,
                                                    bf.sc, d.status, bf.done);
        UOT_CHECK_LAUNCH();
      }
      return UOT_OK;
    };
    // Long runs replay a captured two-iteration CUDA graph: the per-kernel
    // CPU launch cost otherwise bounds small problems (the kernels read the
    // iteration index from iters_done, so the graph carries no t).
    const int pairs = (d.iters >= 8 && !std::getenv("UOT_NO_GRAPH")) ? d.iters / 2 : 0;
    if (pairs > 0) {
      static thread_local cudaStream_t cap = nullptr;  // capture stream (per thread, per device)
      static thread_local int cap_dev = -1;
      int dev = 0;
      UOT_CUDA_TRY(cudaGetDevice(&dev));
      if (cap == nullptr || cap_dev != dev) {
        UOT_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cap_dev = dev;
      }
      cudaGraph_t graph = nullptr;
      UOT_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      int rc = body(0, cap, 1);
      if (rc == UOT_OK) rc = body(1, cap, 1);
      const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
      if (rc != UOT_OK) {
        if (graph != nullptr) cudaGraphDestroy(graph);
        return rc;
      }
      UOT_CUDA_TRY(ce);
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      UOT_CUDA_TRY(ie);
      for (int k = 0; k < pairs; ++k) {
        const cudaError_t le = cudaGraphLaunch(exec, st);
        if (le != cudaSuccess) {
          cudaGraphExecDestroy(exec);
          UOT_CUDA_TRY(le);
        }
      }
      UOT_CUDA_TRY(cudaGraphExecDestroy(exec));  // the launches stay enqueued
    }
    for (int t = 2 * pairs; t < d.iters; ++t) UOT_TRY(body(t, st, pairs > 0 ? 1 : 0));
    sk_finalize<T><<<dim3(ceil_div(nm, 256), d.batch), 256, 0, st>>>(
        d.n, d.m, bf.hatA0, bf.hatA1, bf.hatB, bf.sc, bf.iters_done, (T*)d.f, (T*)d.g);
    UOT_CHECK_LAUNCH();
    if (d.iterations != nullptr) {
      UOT_CUDA_TRY(cudaMemcpyAsync(d.iterations, bf.iters_done, sizeof(int) * d.batch,
                                   cudaMemcpyDeviceToDevice, st));
    }
    return UOT_OK;
  }

  // ---- Verification of a given pair (d.f, d.g as inputs; not modified).
  // out [batch][8]: res_g, log<a x b, e^((f+g-C)/eps)>, res_f, (unused),
  // lambda*, Smin_a(f), Smin_b(g), (unused).
  static int verify(const uot_sinkhorn_desc& d, void* ws, size_t ws_bytes, cudaStream_t st,
                    double* out) {
    Shape s = shape(d);
    WsLayout L;
    Buffers<T> bf;
    const size_t need = layout<T>(s, std::max(d.iters, 1), L, &bf, (char*)ws);
    if (ws_bytes < need) {
      set_error("sinkhorn workspace too small: %zu < %zu", ws_bytes, need);
      return UOT_INVALID;
    }
    sk_reset<<<ceil_div(d.batch, 128), 128, 0, st>>>(d.batch, bf.sc, bf.counter, bf.done,
                                                      bf.iters_done);
    UOT_CHECK_LAUNCH();
    UOT_TRY(launch_center<P>(d, reinterpret_cast<float*>(bf.ctr), st));
    if constexpr (std::is_same<P, SqE32TC>::value) {
      tc_fill_dead<<<1024, 256, 0, st>>>(bf.recA, (long)d.batch * s.recA / tc_kp(d.d), d.d,
                                         tc_kp(d.d));
      tc_fill_dead<<<1024, 256, 0, st>>>(bf.recB, (long)d.batch * s.recB / tc_kp(d.d), d.d,
                                         tc_kp(d.d));
      const double Lr = (double)(float)(1.0 / (d.eps * Dom<float>::unit));
      const double Sa = tc_ascale(Lr);
      tc_init_static<<<1024, 256, 0, st>>>(bf.recA, s.recA, (const float*)d.x,
                                           (const float*)bf.ctr, (long)d.d, d.batch, d.n,
                                           d.d, tc_kp(d.d), Lr, Sa);
      tc_init_static<<<1024, 256, 0, st>>>(bf.recB, s.recB, (const float*)d.y,
                                           (const float*)bf.ctr, (long)d.d, d.batch, d.m,
                                           d.d, tc_kp(d.d), Lr, Sa);
      if (bf.packA != nullptr) {
        tc_pack_out<<<1024, 256, 0, st>>>(bf.packA, (const float*)d.x, (const float*)bf.ctr,
                                          (long)d.d, d.batch, d.n, d.d, (float)Sa);
        tc_pack_out<<<1024, 256, 0, st>>>(bf.packB, (const float*)d.y, (const float*)bf.ctr,
                                          (long)d.d, d.batch, d.m, d.d, (float)Sa);
      }
      UOT_CHECK_LAUNCH();
    }
    {
      const double c1 = 1.0 / ((d.rho1 / (d.rho1 + d.eps)) * d.eps * Dom<T>::unit);
      const double c2 = 1.0 / ((d.rho2 / (d.rho2 + d.eps)) * d.eps * Dom<T>::unit);
      sk_shift_guess<T><<<256, 256, 0, st>>>((long)d.batch * s.n, (const T*)d.f, c1, bf.shiftA);
      sk_shift_guess<T><<<256, 256, 0, st>>>((long)d.batch * s.m, (const T*)d.g, c2, bf.shiftB);
    }
    UOT_CHECK_LAUNCH();
    const int tl = std::max(d.iters, 1);
    // records of both sides from the given pair (init tails: tau = 0)
    UOT_TRY(launch_tail(d, bf, st, false, 1, 0, nullptr, bf.hatA0, (const T*)d.f, 0, nullptr,
                        tl));
    UOT_TRY(launch_tail(d, bf, st, true, 1, 0, nullptr, bf.hatB, (const T*)d.g, 0, nullptr, tl));
    double* lam = bf.trace;  // [batch] scratch (>= batch doubles)
    sk_verify_kl<<<ceil_div(d.batch, 128), 128, 0, st>>>(d.batch, d.n, d.m, bf.sc, d.rho1,
                                                         d.rho2, lam);
    UOT_CHECK_LAUNCH();
    const double a2 = d.rho2 / (d.rho2 + d.eps), a1 = d.rho1 / (d.rho1 + d.eps);
    // g side: smin_cols(f) over all rows (:98) -> res_g, L
    const int sB = splits(d.batch, d.m, d.n, d.d);
    UOT_TRY(launch_main(d, bf, st, true, sB, 0, d.n, 0, sB));
    const int vb_g = std::max(1, std::min(s.nblk, (int)ceil_div(d.m, 256)));
    sk_verify_side<T><<<dim3(vb_g, d.batch), 256, 0, st>>>(
        d.m, sB, bf.part_m, bf.part_a, (const T*)d.g, (const T*)d.b, d.eps, Dom<T>::unit, a2,
        -(d.eps / (d.eps + d.rho2)), lam, bf.blk);
    sk_verify_fold<<<d.batch, 256, 0, st>>>(vb_g, bf.blk, out, 0);
    UOT_CHECK_LAUNCH();
    // f side: smin_rows(g) over all columns (:100) -> res_f
    const int sA = splits(d.batch, d.n, d.m, d.d);
    UOT_TRY(launch_main(d, bf, st, false, sA, 0, d.m, 0, sA));
    const int vb_f = std::max(1, std::min(s.nblk, (int)ceil_div(d.n, 256)));
    sk_verify_side<T><<<dim3(vb_f, d.batch), 256, 0, st>>>(
        d.n, sA, bf.part_m, bf.part_a, (const T*)d.f, (const T*)d.a, d.eps, Dom<T>::unit, a1,
        d.eps / (d.eps + d.rho1), lam, bf.blk);
    sk_verify_fold<<<d.batch, 256, 0, st>>>(vb_f, bf.blk, out, 2);
    UOT_CHECK_LAUNCH();
    sk_verify_pack<<<ceil_div(d.batch, 128), 128, 0, st>>>(d.batch, bf.sc, lam, out);
    UOT_CHECK_LAUNCH();
    return UOT_OK;
  }

  // ---- Row-sharded run (BASELINE cfg3 on P GPUs).  Every
  // rank owns a slice of the source rows and the whole target side.  Per
  // iteration: g-update partial LSEs over the local rows -> one (shift, sum)
  // pair per column -> ONE all-gather (which also carries the f-side
  // scalars of the previous f-tail) -> every rank folds the P pairs in rank
  // order, so the replicated g is bitwise identical on all ranks; the
  // f-update is local.  nccl_comm == NULL with nranks > 1 runs the same
  // protocol for all shards in this process (device copies replace NCCL).
  struct ShardLayout {
    int R;  // rank contexts held by this process
    std::vector<int> nl, off;
    std::vector<size_t> ctx_off;
    std::vector<Shape> shp;
    size_t stride;  // bytes per rank in the exchange buffer
    size_t xbuf_off, xall_off, xfin_off, total;
  };

  static int shard_layout(const uot_sinkhorn_desc& d, ShardLayout& L) {
    const bool real = d.nccl_comm != nullptr;
    const int NR = std::max(1, d.nranks);
    if (d.batch != 1) {
      set_error("row sharding runs a single problem (batch must be 1)");
      return UOT_INVALID;
    }
    L.R = real ? 1 : NR;
    L.nl.assign(L.R, 0);
    L.off.assign(L.R, 0);
    if (real) {
      L.nl[0] = d.n;
    } else {
      if (d.shard_rows == nullptr) {
        set_error("emulated sharding needs shard_rows");
        return UOT_INVALID;
      }
      int o = 0;
      for (int r = 0; r < NR; ++r) {
        L.nl[r] = d.shard_rows[r];
        L.off[r] = o;
        o += L.nl[r];
        if (L.nl[r] < 1) {
          set_error("every shard needs at least one row");
          return UOT_INVALID;
        }
      }
      if (o != d.n) {
        set_error("shard_rows must sum to n");
        return UOT_INVALID;
      }
    }
    L.stride = ((sizeof(double) * 4 * d.batch + 2 * sizeof(T) * (size_t)d.batch * d.m) + 255) /
               256 * 256;
    size_t off = 0;
    L.ctx_off.assign(L.R, 0);
    L.shp.assign(L.R, Shape{});
    for (int r = 0; r < L.R; ++r) {
      uot_sinkhorn_desc dr = d;
      dr.n = L.nl[r];
      Shape s = shape(dr);
      L.shp[r] = s;
      WsLayout wl;
      L.ctx_off[r] = off;
      off += layout<T>(s, d.iters, wl, nullptr, nullptr);
    }
    L.xbuf_off = off;
    off += L.stride * L.R;
    L.xall_off = off;
    off += L.stride * NR;
    L.xfin_off = off;
    off += (sizeof(double) * 4 * d.batch * NR + 255) / 256 * 256;
    L.total = off;
    return UOT_OK;
  }

  static size_t ws_size_sharded(const uot_sinkhorn_desc& d) {
    ShardLayout L;
    if (shard_layout(d, L) != UOT_OK) return 0;
    return L.total;
  }

  static int shard_chunks(int m, int nranks) {
    const char* e = std::getenv("UOT_SHARD_CHUNKS");
    int c = e ? std::atoi(e) : (nranks > 1 ? 4 : 1);
    c = std::max(1, std::min(c, 16));
    const int min_cols = e ? 1 : 1024;  // default: chunks of >= 1024 columns
    while (c > 1 && m / c < min_cols) --c;
    return c;
  }

  // Exchange of the g-update's pairs for columns [c0, c1) (and, with the
  // first chunk, the published scalars) into the same gathered layout as
  // exchange(): grouped NCCL sends / receives with every peer over
  // NVLink, or device copies between the emulated rank contexts.
  static int exchange_cols(const uot_sinkhorn_desc& d, const ShardLayout& L, char* base,
                           char* recv, int c0, int c1, bool scalars, cudaStream_t st) {
    const size_t scal_bytes = sizeof(double) * 4 * d.batch;
    const size_t arr = sizeof(T) * (size_t)d.batch * d.m;  // bytes of one pair array
    const size_t lo = sizeof(T) * (size_t)c0, len = sizeof(T) * (size_t)(c1 - c0);
    // pieces of a rank's slot: (offset, bytes); batch == 1 on the sharded path
    const size_t off[3] = {0, scal_bytes + lo, scal_bytes + arr + lo};
    const size_t sz[3] = {scalars ? scal_bytes : 0, len, len};
#if defined(UOT_WITH_NCCL)
    if (d.nccl_comm != nullptr) {
      ncclComm_t comm = (ncclComm_t)d.nccl_comm;
      const int me = d.rank, npeer = d.nranks;
      char* mine = base + L.xbuf_off;
      ncclResult_t rc = ncclGroupStart();
      for (int k = 0; k < 3 && rc == ncclSuccess; ++k) {
        if (sz[k] == 0) continue;
        for (int p = 0; p < npeer && rc == ncclSuccess; ++p) {
          if (p == me) continue;
          rc = ncclSend(mine + off[k], sz[k], ncclChar, p, comm, st);
          if (rc == ncclSuccess)
            rc = ncclRecv(recv + L.stride * p + off[k], sz[k], ncclChar, p, comm, st);
        }
      }
      const ncclResult_t re = ncclGroupEnd();
      if (rc != ncclSuccess || re != ncclSuccess) {
        set_error("chunked exchange failed: %s",
                  ncclGetErrorString(rc != ncclSuccess ? rc : re));
        return UOT_NCCL;
      }
      for (int k = 0; k < 3; ++k)
        if (sz[k] > 0)
          UOT_CUDA_TRY(cudaMemcpyAsync(recv + L.stride * me + off[k], mine + off[k], sz[k],
                                       cudaMemcpyDeviceToDevice, st));
      return UOT_OK;
    }
#endif
    if (d.nccl_comm != nullptr) {
      set_error("built without NCCL");
      return UOT_NCCL;
    }
    for (int r = 0; r < L.R; ++r)
      for (int k = 0; k < 3; ++k)
        if (sz[k] > 0)
          UOT_CUDA_TRY(cudaMemcpyAsync(recv + L.stride * r + off[k],
                                       base + L.xbuf_off + L.stride * r + off[k], sz[k],
                                       cudaMemcpyDeviceToDevice, st));
    return UOT_OK;
  }

  static int exchange(const uot_sinkhorn_desc& d, const ShardLayout& L, char* base, size_t bytes,
                      char* recv, size_t recv_stride, cudaStream_t st) {
#if defined(UOT_WITH_NCCL)
    if (d.nccl_comm != nullptr) {
      ncclResult_t r = ncclAllGather(base + L.xbuf_off, recv, bytes, ncclChar,
                                     (ncclComm_t)d.nccl_comm, st);
      if (r != ncclSuccess) {
        set_error("ncclAllGather failed: %s", ncclGetErrorString(r));
        return UOT_NCCL;
      }
      return UOT_OK;
    }
#endif
    if (d.nccl_comm != nullptr) {
      set_error("built without NCCL");
      return UOT_NCCL;
    }
    for (int r = 0; r < L.R; ++r)
      UOT_CUDA_TRY(cudaMemcpyAsync(recv + recv_stride * r, base + L.xbuf_off + L.stride * r,
                                   bytes, cudaMemcpyDeviceToDevice, st));
    return UOT_OK;
  }

  static int run_sharded(const uot_sinkhorn_desc& d, void* ws, size_t ws_bytes, cudaStream_t st) {
    ShardLayout L;
    UOT_TRY(shard_layout(d, L));
    if (ws_bytes < L.total) {
      set_error("sinkhorn workspace too small: %zu < %zu", ws_bytes, L.total);
      return UOT_INVALID;
    }
    const int NR = std::max(1, d.nranks);
    char* base = (char*)ws;
    const int trace_len = std::max(d.iters, 1);
    const bool H = d.variant == UOT_SINKHORN_H;
    const double kka = (d.eps / (d.eps + d.rho1)) * (d.rho2 / (d.rho1 + d.rho2));
    const double tau_fac_a = H ? kka / (1.0 - kka) : 0.0;
    std::vector<uot_sinkhorn_desc> dr(L.R, d);
    std::vector<Buffers<T>> bf(L.R);
    std::vector<int> sA(L.R), sB(L.R);
    char* xall = base + L.xall_off;
    double* xfin = (double*)(base + L.xfin_off);
    const long stride_d = (long)(L.stride / sizeof(double));
    const long stride_t = (long)(L.stride / sizeof(T));
    const size_t scal_bytes = sizeof(double) * 4 * d.batch;
    for (int r = 0; r < L.R; ++r) {
      WsLayout wl;
      layout<T>(L.shp[r], d.iters, wl, &bf[r], base + L.ctx_off[r]);
      dr[r].n = L.nl[r];
      dr[r].x = (const char*)d.x + sizeof(T) * (size_t)L.off[r] * d.d;
      dr[r].a = (const char*)d.a + sizeof(T) * (size_t)L.off[r];
      dr[r].f = (char*)d.f + sizeof(T) * (size_t)L.off[r];
      if (d.c != nullptr) {
        set_error("row sharding supports point-cloud and 1-D costs");
        return UOT_INVALID;
      }
      sB[r] = splits(d.batch, d.m, L.nl[r], d.d);
      sA[r] = splits(d.batch, L.nl[r], d.m, d.d);
      sk_reset<<<ceil_div(d.batch, 128), 128, 0, st>>>(d.batch, bf[r].sc, bf[r].counter,
                                                        bf[r].done, bf[r].iters_done);
      // each shard centres its own records (the cost, hence every partial, does not
      // depend on the centre)
      UOT_TRY(launch_center<P>(dr[r], reinterpret_cast<float*>(bf[r].ctr), st));
      sk_zero<T><<<256, 256, 0, st>>>((long)L.nl[r], bf[r].shiftA);
      sk_zero<T><<<256, 256, 0, st>>>((long)d.m, bf[r].shiftB);
      UOT_CHECK_LAUNCH();
      const T* f0 = (const T*)dr[r].f;
      if (!d.init_given) {
        sk_zero<T><<<256, 256, 0, st>>>((long)std::max(L.nl[r], d.m), bf[r].zeros);
        f0 = bf[r].zeros;
      }
      double* xb = (double*)(base + L.xbuf_off + L.stride * r);
      ShardOpt so{1, nullptr, 0, NR, 0, xb, nullptr, nullptr, 0, 0};
      UOT_TRY(launch_tail(dr[r], bf[r], st, false, 1, 0, nullptr, bf[r].hatA0, f0, 0, nullptr,
                          trace_len, &so));
    }
    double* trace = d.trace_delta != nullptr ? d.trace_delta : bf[0].trace;
    // The g-update's exchange runs in column chunks on a second stream: chunk
    // c's (shift, sum) pairs travel while the main kernel computes chunk c+1
    // (SURVEY.md §8e).  UOT_SHARD_CHUNKS overrides the count (1: no overlap).
    const int nchunk = shard_chunks(d.m, NR);
    cudaStream_t cs = st;
    std::vector<cudaEvent_t> ev;
    if (nchunk > 1) {
      UOT_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      ev.resize(nchunk + 1);
      for (auto& e : ev) UOT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    struct StreamGuard {
      cudaStream_t s, main;
      std::vector<cudaEvent_t>* ev;
      ~StreamGuard() {
        if (s != main) {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
          for (auto& e : *ev) cudaEventDestroy(e);
        }
      }
    } guard{cs, st, &ev};
    for (int t = 0; t < d.iters; ++t) {
      for (int c = 0; c < nchunk; ++c) {
        const int c0 = (int)((long)d.m * c / nchunk), c1 = (int)((long)d.m * (c + 1) / nchunk);
        for (int r = 0; r < L.R; ++r) {
          UOT_TRY(launch_main(dr[r], bf[r], st, true, sB[r], 0, L.nl[r], 0, sB[r], c0, c1));
          char* xb = base + L.xbuf_off + L.stride * r;
          T* pm = (T*)(xb + scal_bytes);
          T* pa = pm + (size_t)d.batch * d.m;
          sk_combine<T><<<dim3(ceil_div(c1 - c0, 256), d.batch), 256, 0, st>>>(
              d.m, sB[r], bf[r].part_m, bf[r].part_a, pm, pa, c0, c1);
          UOT_CHECK_LAUNCH();
        }
        if (nchunk == 1) {
          UOT_TRY(exchange(d, L, base, L.stride, xall, L.stride, st));
        } else {
          UOT_CUDA_TRY(cudaEventRecord(ev[c], st));
          UOT_CUDA_TRY(cudaStreamWaitEvent(cs, ev[c], 0));
          UOT_TRY(exchange_cols(d, L, base, xall, c0, c1, c == 0, cs));
        }
      }
      if (nchunk > 1) {  // the g-tail needs every chunk
        UOT_CUDA_TRY(cudaEventRecord(ev[nchunk], cs));
        UOT_CUDA_TRY(cudaStreamWaitEvent(st, ev[nchunk], 0));
      }
      for (int r = 0; r < L.R; ++r) {
        const T* pm = (const T*)(xall + scal_bytes);
        const T* pa = pm + (size_t)d.batch * d.m;
        ShardOpt so{2, (const double*)xall, stride_d, NR, t == 0 ? 1 : 0, nullptr, pm, pa,
                    stride_t, (long)d.m};
        UOT_TRY(launch_tail(dr[r], bf[r], st, true, 0, NR, nullptr, bf[r].hatB, nullptr, t,
                            r == 0 ? trace : nullptr, trace_len, &so));
      }
      for (int r = 0; r < L.R; ++r) {
        T* hat_old = (t & 1) ? bf[r].hatA1 : bf[r].hatA0;
        T* hat_new = (t & 1) ? bf[r].hatA0 : bf[r].hatA1;
        UOT_TRY(launch_main(dr[r], bf[r], st, false, sA[r], 0, d.m, 0, sA[r]));
        double* xb = (double*)(base + L.xbuf_off + L.stride * r);
        ShardOpt so{1, nullptr, 0, NR, 0, xb, nullptr, nullptr, 0, 0};
        UOT_TRY(launch_tail(dr[r], bf[r], st, false, 0, sA[r], hat_old, hat_new, nullptr, t,
                            nullptr, trace_len, &so));
      }
    }
    UOT_TRY(exchange(d, L, base, scal_bytes, (char*)xfin, scal_bytes, st));
    for (int r = 0; r < L.R; ++r) {
      sk_resolve_final<<<ceil_div(d.batch, 128), 128, 0, st>>>(
          d.batch, NR, xfin, (long)(scal_bytes / sizeof(double)), d.rho1, tau_fac_a, bf[r].sc,
          r == 0 ? trace : nullptr, trace_len, d.iters - 1, bf[r].iters_done);
      UOT_CHECK_LAUNCH();
      const long nm = std::max(L.nl[r], d.m);
      sk_finalize<T><<<dim3(ceil_div(nm, 256), d.batch), 256, 0, st>>>(
          L.nl[r], d.m, bf[r].hatA0, bf[r].hatA1, bf[r].hatB, bf[r].sc, bf[r].iters_done,
          (T*)dr[r].f, (T*)d.g);
      UOT_CHECK_LAUNCH();
    }
    if (d.iterations != nullptr) {
      UOT_CUDA_TRY(cudaMemcpyAsync(d.iterations, bf[0].iters_done, sizeof(int) * d.batch,
                                   cudaMemcpyDeviceToDevice, st));
    }
    return UOT_OK;
  }
};

// Bench hook: after a normal run (which leaves the workspace holding a valid
// state), time `reps` launches of each direction's main kernel with CUDA
// events on the caller's stream; returns the mean per-launch milliseconds of
// the g-direction and f-direction kernels.
template <class E>
int time_main(const uot_sinkhorn_desc& d, void* ws, size_t ws_bytes, cudaStream_t st, int reps,
              float* ms) {
  using T = typename E::T;
  UOT_TRY(E::run(d, ws, ws_bytes, st));
  Shape s = E::shape(d);
  WsLayout L;
  Buffers<T> bf;
  layout<T>(s, d.iters, L, &bf, (char*)ws);
  const int sB = E::splits(d.batch, d.m, d.n, d.d);
  const int sA = E::splits(d.batch, d.n, d.m, d.d);
  cudaEvent_t e0, e1;
  UOT_CUDA_TRY(cudaEventCreate(&e0));
  UOT_CUDA_TRY(cudaEventCreate(&e1));
  for (int dir = 0; dir < 2; ++dir) {
    UOT_TRY(E::launch_main(d, bf, st, dir == 0, dir == 0 ? sB : sA, 0, dir == 0 ? d.n : d.m, 0,
                           dir == 0 ? sB : sA));
    UOT_CUDA_TRY(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r)
      UOT_TRY(E::launch_main(d, bf, st, dir == 0, dir == 0 ? sB : sA, 0, dir == 0 ? d.n : d.m, 0,
                             dir == 0 ? sB : sA));
    UOT_CUDA_TRY(cudaEventRecord(e1, st));
    UOT_CUDA_TRY(cudaEventSynchronize(e1));
    float t = 0.f;
    UOT_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
    ms[dir] = t / (float)reps;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return UOT_OK;
}

template <class Fn>
int dispatch(const uot_sinkhorn_desc& d, Fn&& fn) {
  if (d.dtype == UOT_F32) {
    switch (d.cost) {
      case UOT_COST_SQEUCLID:
        if (d.d == 1) return fn(Engine<SqE32<1>>());
        if (d.d == 2) return fn(Engine<SqE32<2>>());
        if (d.d == 3) return fn(Engine<SqE32<3>>());
        // UOT_SINKHORN_SIMT=1 keeps d >= 32 on the SIMT engine (comparison runs)
        if (d.d >= 32 && d.d % 4 == 0 && 2 * tc_ka(d.d) <= 256 && d.nranks <= 1 &&
            d.nccl_comm == nullptr && std::getenv("UOT_SINKHORN_SIMT") == nullptr)
          return fn(Engine<SqE32TC>());
        return fn(Engine<SqE32N>());
      case UOT_COST_POWER:
        return fn(Engine<Pow1D<float>>());
      case UOT_COST_EXPLICIT:
        return fn(Engine<Explicit<float>>());
    }
  } else if (d.dtype == UOT_F64) {
    switch (d.cost) {
      case UOT_COST_SQEUCLID:
        return fn(Engine<SqE64>());
      case UOT_COST_POWER:
        return fn(Engine<Pow1D<double>>());
      case UOT_COST_EXPLICIT:
        return fn(Engine<Explicit<double>>());
    }
  }
  set_error("unsupported sinkhorn dtype/cost combination (%d, %d)", d.dtype, d.cost);
  return UOT_INVALID;
}

int validate(const uot_sinkhorn_desc* d) {
  if (d == nullptr) {
    set_error("null descriptor");
    return UOT_INVALID;
  }
  if (d->batch < 1 || d->n < 1 || d->m < 1 || d->d < 1 || d->iters < 1) {
    set_error("invalid sizes (batch=%d n=%d m=%d d=%d iters=%d)", d->batch, d->n, d->m, d->d,
              d->iters);
    return UOT_INVALID;
  }
  if (!(d->eps > 0.0) || !std::isfinite(d->eps)) {
    set_error("sinkhorn iterations need eps > 0");  // src/sinkhorn.py:192-194
    return UOT_INVALID;
  }
  if (!(d->rho1 > 0.0) || !(d->rho2 > 0.0) || !std::isfinite(d->rho1) || !std::isfinite(d->rho2)) {
    set_error("rho must be positive and finite");  // src/entropies.py:46-48
    return UOT_INVALID;
  }
  if (d->variant != UOT_SINKHORN_F && d->variant != UOT_SINKHORN_H &&
      d->variant != UOT_SINKHORN_G) {
    set_error("variant must be F (0), H (1) or G (2)");
    return UOT_INVALID;
  }
  if (d->ent1 < UOT_ENT_KL || d->ent1 > UOT_ENT_BALANCED || d->ent2 < UOT_ENT_KL ||
      d->ent2 > UOT_ENT_BALANCED) {
    set_error("ent1 / ent2 must be UOT_ENT_KL, UOT_ENT_BERG or UOT_ENT_BALANCED");
    return UOT_INVALID;
  }
  const bool klkl = d->ent1 == UOT_ENT_KL && d->ent2 == UOT_ENT_KL;
  if (d->variant == UOT_SINKHORN_H && !klkl) {
    set_error("h-sinkhorn requires kl penalties on both marginals");  // sinkhorn.py:151-152
    return UOT_UNSUPPORTED_ENTROPY;
  }
  if (d->variant == UOT_SINKHORN_G &&
      (d->ent1 == UOT_ENT_BALANCED || d->ent2 == UOT_ENT_BALANCED)) {
    set_error("optimal translation needs strictly convex conjugates (KL or Berg)");
    return UOT_UNSUPPORTED_ENTROPY;
  }
  if (!klkl && (d->nranks > 1 || d->nccl_comm != nullptr)) {
    set_error("row sharding runs KL marginals");
    return UOT_INVALID;
  }
  if (d->variant == UOT_SINKHORN_G && (d->nranks > 1 || d->nccl_comm != nullptr)) {
    set_error("the G variant runs unsharded");
    return UOT_INVALID;
  }
  if (d->cost == UOT_COST_POWER && (d->d != 1 || !(d->p >= 1.0))) {
    set_error("power cost needs d == 1 and p >= 1");  // src/measures.py:200-202
    return UOT_INVALID;
  }
  if (d->cost == UOT_COST_EXPLICIT && (d->c == nullptr || d->ct == nullptr)) {
    set_error("explicit cost needs c and its transpose ct");
    return UOT_INVALID;
  }
  return UOT_OK;
}

}  // namespace

}  // namespace uot

extern "C" int uot_sinkhorn_workspace_size(const uot_sinkhorn_desc* desc, size_t* bytes) {
  using namespace uot;
  UOT_TRY(validate(desc));
  return dispatch(*desc, [&](auto eng) {
    *bytes = decltype(eng)::ws_size(*desc);
    return (int)UOT_OK;
  });
}

extern "C" int uot_sinkhorn_run(const uot_sinkhorn_desc* desc, void* workspace,
                                size_t workspace_bytes, void* stream) {
  using namespace uot;
  UOT_TRY(validate(desc));
  return dispatch(*desc, [&](auto eng) {
    return decltype(eng)::run(*desc, workspace, workspace_bytes, (cudaStream_t)stream);
  });
}

extern "C" int uot_sinkhorn_verify(const uot_sinkhorn_desc* desc, void* workspace,
                                   size_t workspace_bytes, void* stream, double* out) {
  using namespace uot;
  UOT_TRY(validate(desc));
  if (desc->nranks > 1 || desc->nccl_comm != nullptr) {
    set_error("uot_sinkhorn_verify runs unsharded");
    return UOT_INVALID;
  }
  if (desc->ent1 != UOT_ENT_KL || desc->ent2 != UOT_ENT_KL) {
    set_error("uot_sinkhorn_verify evaluates KL objectives");
    return UOT_UNSUPPORTED_ENTROPY;
  }
  return dispatch(*desc, [&](auto eng) {
    return decltype(eng)::verify(*desc, workspace, workspace_bytes, (cudaStream_t)stream, out);
  });
}

extern "C" int uot_sinkhorn_time_main(const uot_sinkhorn_desc* desc, void* workspace,
                                      size_t workspace_bytes, void* stream, int reps,
                                      float* ms_out) {
  using namespace uot;
  UOT_TRY(validate(desc));
  return dispatch(*desc, [&](auto eng) {
    return time_main<decltype(eng)>(*desc, workspace, workspace_bytes, (cudaStream_t)stream,
                                    reps, ms_out);
  });
}


#ifdef UOT_TC_TIMING
// scripts/tc_timeline.py (timing build only)
extern "C" int uot_debug_tc_stamps(unsigned long long* out, int n) {
  cudaMemcpyFromSymbol(out, uot::g_tc_stamps, sizeof(unsigned long long) * 8 * (size_t)n);
  return 0;
}
#endif

// ---------------------------------------------------------------------------
// The entropy-family functions of the reference API on the device
// (src/entropies.py:67-263): weighted log-sum-exp (flat and along an axis),
// conjugates and their derivatives, aprox, and the divergences.

namespace uot {
namespace {

// op 0 conj, 1 conj_grad, 2 conj_hess, 3 aprox (entropies.py:142-221)
__global__ void entropy_map_kernel(int op, int ent, double rho, double eps, long n,
                                   const double* __restrict__ x, double* __restrict__ out,
                                   int* __restrict__ bad) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const double v = x[i];
    double r = 0.0;
    if (op == 3) {
      r = aprox_any(ent, rho, eps, v);
    } else if (ent == UOT_ENT_KL) {
      r = op == 0 ? rho * expm1(v / rho) : op == 1 ? exp(v / rho) : exp(v / rho) / rho;
    } else if (ent == UOT_ENT_BERG) {
      if (op != 2 && !(v < rho)) *bad = 1;  // the conjugate lives on x < rho
      r = op == 0 ? -rho * log1p(-v / rho) : op == 1 ? rho / (rho - v) : rho / ((rho - v) * (rho - v));
    } else {
      r = op == 0 ? v + 0.0 : op == 1 ? 1.0 : 0.0;
    }
    out[i] = r;
  }
}

// log sum_k w_k exp(scale v[o][k][i]) with zero-weight entries masked before
// the max shift (entropies.py:67-92); one thread per (o, i) output.
__global__ void lse_axis_kernel(long outer, long K, long inner, const double* __restrict__ v,
                                const double* __restrict__ w, double scale,
                                double* __restrict__ out) {
  const long total = outer * inner;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long o = t / inner, i = t - o * inner;
    const double* vo = v + o * K * inner + i;
    double mx = -CUDART_INF;
    for (long k = 0; k < K; ++k)
      if (w[k] > 0.0) mx = fmax(mx, scale * vo[k * inner]);
    const double sh = isfinite(mx) ? mx : 0.0;
    double s = 0.0;
    for (long k = 0; k < K; ++k)
      if (w[k] > 0.0) s += w[k] * exp(scale * vo[k * inner] - sh);
    out[t] = log(s) + sh;
  }
}

// inner == 1: one block per output (masked block max, then the sum).
__global__ void __launch_bounds__(256) lse_flat_kernel(long K, const double* __restrict__ v,
                                                       const double* __restrict__ w, double scale,
                                                       double* __restrict__ out) {
  __shared__ double scratch[32];
  const double* vo = v + blockIdx.x * K;
  double mx = -CUDART_INF;
  for (long k = threadIdx.x; k < K; k += blockDim.x)
    if (w[k] > 0.0) mx = fmax(mx, scale * vo[k]);
  mx = block_reduce(mx, scratch, MaxOp(), -CUDART_INF);
  const double sh = isfinite(mx) ? mx : 0.0;
  double s = 0.0;
  for (long k = threadIdx.x; k < K; k += blockDim.x)
    if (w[k] > 0.0) s += w[k] * exp(scale * vo[k] - sh);
  s = block_reduce(s, scratch, SumOp(), 0.0);
  if (threadIdx.x == 0) out[blockIdx.x] = log(s) + sh;
}

// Csiszar divergence (entropies.py:104-140), one block.
__global__ void __launch_bounds__(1024) divergence_kernel(int ent, double rho, long n,
                                                          const double* __restrict__ mu,
                                                          const double* __restrict__ nu,
                                                          double* __restrict__ out) {
  __shared__ double scratch[32];
  double terms = 0.0, sing = 0.0, zero_mu = 0.0, md = 0.0, mw = 0.0;
  for (long i = threadIdx.x; i < n; i += blockDim.x) {
    const double m = mu[i], w = nu[i];
    if (ent == UOT_ENT_BALANCED) {
      md = fmax(md, fabs(m - w));
      mw = fmax(mw, fabs(w));
    } else if (w > 0.0) {
      if (ent == UOT_ENT_KL) {
        terms += (m > 0.0 ? m * log(m / w) : 0.0) - m + w;
      } else {
        if (m == 0.0) zero_mu = 1.0;
        else terms += m - w - w * log(m / w);
      }
    } else {
      sing += m;
    }
  }
  terms = block_reduce(terms, scratch, SumOp(), 0.0);
  sing = block_reduce(sing, scratch, SumOp(), 0.0);
  zero_mu = block_reduce(zero_mu, scratch, MaxOp(), 0.0);
  md = block_reduce(md, scratch, MaxOp(), 0.0);
  mw = block_reduce(mw, scratch, MaxOp(), 0.0);
  if (threadIdx.x != 0) return;
  double r;
  if (ent == UOT_ENT_BALANCED) r = md <= 1e-9 * (1.0 + mw) ? 0.0 : CUDART_INF;
  else if (ent == UOT_ENT_KL) r = sing > 0.0 ? CUDART_INF : rho * terms;
  else r = zero_mu > 0.0 ? CUDART_INF : rho * (terms + sing);
  out[0] = r;
}

}  // namespace
}  // namespace uot

extern "C" int uot_entropy_map(int32_t op, int32_t ent, double rho, double eps, int64_t n,
                               const double* x, double* out, int32_t* bad, void* stream) {
  using namespace uot;
  if (op < 0 || op > 3 || ent < 0 || ent > 2 || n < 0 || (op == 3 && !(eps > 0.0))) {
    set_error("entropy_map: invalid arguments");
    return UOT_INVALID;
  }
  if (n == 0) return UOT_OK;
  const long blocks = std::min<long>(4096, (n + 255) / 256);
  entropy_map_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(op, ent, rho, eps, n, x,
                                                                         out, bad);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_logdotexp(int64_t outer, int64_t k, int64_t inner, const double* v,
                             const double* w, double scale, double* out, void* stream) {
  using namespace uot;
  if (outer < 1 || k < 0 || inner < 1 || out == nullptr) {
    set_error("logdotexp: invalid arguments");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (inner == 1 && outer <= 65535) {
    lse_flat_kernel<<<(unsigned)outer, 256, 0, st>>>(k, v, w, scale, out);
  } else {
    const long blocks = std::min<long>(4096, (outer * inner + 255) / 256);
    lse_axis_kernel<<<(unsigned)blocks, 256, 0, st>>>(outer, k, inner, v, w, scale, out);
  }
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_divergence(int32_t ent, double rho, int64_t n, const double* mu,
                              const double* nu, double* out, void* stream) {
  using namespace uot;
  if (ent < 0 || ent > 2 || n < 0 || out == nullptr) {
    set_error("divergence: invalid arguments");
    return UOT_INVALID;
  }
  divergence_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(ent, rho, n, mu, nu, out);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}
