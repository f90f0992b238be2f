/*
 * scale.c -- vectorised fp64 softmin for generating the BASELINE-scale
 * fixtures (tests/golden/make_scale.py).  TEST INFRASTRUCTURE ONLY: it is the
 * same restatement as oracle.c's oracle_smin (sinkhorn.py:93-100 on
 * entropies.py:84-92: zero weights masked, max shift, shift + log sum w
 * exp(v - shift)) with the reduction split into SIMD lanes and blocks of
 * output indices, so cfg3 (65536^2 x 400 half-steps) runs in minutes on the
 * container instead of hours (single thread: the container has about one core
 * of throughput; the omp parallel pragmas only take effect under -fopenmp).  Only the summation order differs from
 * oracle_smin (the reference itself reduces with numpy's pairwise sum); the
 * exp is glibc's libmvec (< 4 ulp).  Never shipped, never on the GPU box.
 *
 * Squared Euclidean cost between point clouds: C(i, j) = sum_k (xr_ik - xo_jk)^2
 * (measures.py:135-136 computes p = 2 as diff * diff), evaluated in fp64.
 */
#include <math.h>
#include <stdlib.h>

/* d = 2: four output indices per sweep over a chunk of the reduced side
 * (x0, x1, pot and w read once for four outputs), the cost recomputed in each
 * of the two passes.  pass 0 folds the masked maxima into m[4]; pass 1 adds
 * w exp(v - s) into acc[4]. */
static void sq2_chunk(int pass, int i0, int i1, const double* x0, const double* x1,
                      const double* pot, const double* w, double eps, const double* y0,
                      const double* y1, const double* s, double* m, double* acc) {
    const double ya0 = y0[0], ya1 = y0[1], ya2 = y0[2], ya3 = y0[3];
    const double yb0 = y1[0], yb1 = y1[1], yb2 = y1[2], yb3 = y1[3];
#define C(Q) ((a - ya##Q) * (a - ya##Q) + (b - yb##Q) * (b - yb##Q))
    if (pass == 0) {
        double m0 = m[0], m1 = m[1], m2 = m[2], m3 = m[3];
#pragma omp simd reduction(max : m0, m1, m2, m3)
        for (int i = i0; i < i1; ++i) {
            const double a = x0[i], b = x1[i], u = pot[i];
            const int live = w[i] > 0.0;
#define V(Q) (live ? (u - C(Q)) / eps : -INFINITY)
            double v0 = V(0), v1 = V(1), v2 = V(2), v3 = V(3);
#undef V
            m0 = v0 > m0 ? v0 : m0;
            m1 = v1 > m1 ? v1 : m1;
            m2 = v2 > m2 ? v2 : m2;
            m3 = v3 > m3 ? v3 : m3;
        }
        m[0] = m0, m[1] = m1, m[2] = m2, m[3] = m3;
        return;
    }
    const double s0 = s[0], s1 = s[1], s2 = s[2], s3 = s[3];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma omp simd reduction(+ : a0, a1, a2, a3)
    for (int i = i0; i < i1; ++i) {
        const double a = x0[i], b = x1[i], u = pot[i], ww = w[i] > 0.0 ? w[i] : 0.0;
#define E(Q, S) (ww * exp((u - C(Q)) / eps - S))
        a0 += E(0, s0);
        a1 += E(1, s1);
        a2 += E(2, s2);
        a3 += E(3, s3);
#undef E
    }
    acc[0] += a0, acc[1] += a1, acc[2] += a2, acc[3] += a3;
#undef C
}

/* One block of up to JB outputs: the reduced side is swept in L2-sized
 * chunks so it streams from DRAM once per block and pass (not once per
 * four outputs). */
#define JB 32
#define ICH 4096
static void smin_sq2_block(int nred, const double* x0, const double* x1, const double* pot,
                           const double* w, double eps, const double* yo, int nj, double* out) {
    double y0[JB], y1[JB], m[JB], s[JB], acc[JB];
    for (int q = 0; q < JB; ++q) {
        int qq = q < nj ? q : nj - 1;
        y0[q] = yo[2 * qq];
        y1[q] = yo[2 * qq + 1];
        m[q] = -INFINITY;
        acc[q] = 0.0;
    }
    for (int pass = 0; pass < 2; ++pass) {
        for (int i0 = 0; i0 < nred; i0 += ICH) {
            int i1 = nred - i0 < ICH ? nred : i0 + ICH;
            for (int q = 0; q < nj; q += 4)
                sq2_chunk(pass, i0, i1, x0, x1, pot, w, eps, y0 + q, y1 + q, s + q, m + q,
                          acc + q);
        }
        if (pass == 0)
            for (int q = 0; q < JB; ++q) s[q] = isfinite(m[q]) ? m[q] : 0.0;
    }
    for (int q = 0; q < nj; ++q) out[q] = -eps * (log(acc[q]) + s[q]);
}

/* xt is the reduced side transposed to [d][nred]; generic d builds the cost
 * row of one output index in d vectorised passes, then a max pass and an
 * exp-sum pass. */
void scale_smin_sq(int nred, int nout, int d, const double* xt, const double* xo,
                   const double* pot, const double* w, double eps, double* out) {
    if (d == 2) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int j = 0; j < nout; j += JB)
            smin_sq2_block(nred, xt, xt + nred, pot, w, eps, xo + 2L * j,
                           nout - j < JB ? nout - j : JB, out + j);
        return;
    }
#pragma omp parallel
    {
        double* c = (double*)malloc(sizeof(double) * (size_t)nred);
#pragma omp for schedule(dynamic, 4)
        for (int j = 0; j < nout; ++j) {
            for (int i = 0; i < nred; ++i) c[i] = 0.0;
            for (int k = 0; k < d; ++k) {
                const double yk = xo[(long)j * d + k];
                const double* xk = xt + (long)k * nred;
#pragma omp simd
                for (int i = 0; i < nred; ++i) {
                    double t = xk[i] - yk;
                    c[i] += t * t;
                }
            }
            double mx = -INFINITY;
#pragma omp simd reduction(max : mx)
            for (int i = 0; i < nred; ++i) {
                double v = w[i] > 0.0 ? (pot[i] - c[i]) / eps : -INFINITY;
                mx = v > mx ? v : mx;
            }
            const double s = isfinite(mx) ? mx : 0.0;
            double acc = 0.0;
#pragma omp simd reduction(+ : acc)
            for (int i = 0; i < nred; ++i) {
                double e = exp((pot[i] - c[i]) / eps - s);
                acc += w[i] > 0.0 ? w[i] * e : 0.0;
            }
            out[j] = -eps * (log(acc) + s);
        }
        free(c);
    }
}
