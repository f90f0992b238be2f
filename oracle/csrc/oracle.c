/*
 * oracle.c -- CPU restatement (fp64) of the reference's sequential sweeps and
 * of the dense softmin reduction, for the parity tests and the CPU baseline.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2201_00730_b200/ links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load it, as the checker.
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/pkg/src/uotkit/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* Cost kinds shared with oracle/__init__.py. */
enum { COST_SQEUCLID = 0, COST_POWER1D = 1, COST_EXPLICIT = 2 };

/* measures.py:228-234 (build_cost_matrix) and ot1d.py:466-472 (_cost_fn):
 * |x-y|^p with p==1 -> |d|, p==2 -> d*d (both exact-rounded like the
 * reference's numpy / CPython pow). */
static inline double pow_cost(double xi, double yj, double p) {
    double d = fabs(xi - yj);
    if (p == 1.0) return d;
    if (p == 2.0) return d * d;
    return pow(d, p);
}

/*
 * Softmin of the cost slack along the reduced index, for every output index:
 *   out[j] = -eps * logdotexp((pot_i - C(i, j)) / eps, w)      (over i)
 * sinkhorn.py:93-100 (_smin_cols/_smin_rows) on top of entropies.py:84-92
 * (axis form of logdotexp: zero weights masked to -inf before the max shift,
 * non-finite shift replaced by 0, then shift + log(sum w * exp(v - shift))).
 *
 * Geometry: kind COST_SQEUCLID: xr[nred*d], xo[nout*d], C = sum_k (xr-xo)^2
 *           kind COST_POWER1D : xr[nred], xo[nout], C = |xr - xo|^p
 *           kind COST_EXPLICIT: cm is the dense matrix; C(i, j) =
 *                               cm[i*ldi_stride + j*ldj_stride]
 * Parallelised over output indices with pthreads (the reduction order per
 * output index is the reference's sequential order).
 */
typedef struct {
    int kind, nred, nout, d;
    const double *xr, *xo, *cm, *pot, *w;
    double p, eps;
    long ldi, ldj;
    double* out;
    int j0, j1;
} smin_job;

static void* smin_worker(void* arg) {
    const smin_job* s = (const smin_job*)arg;
    for (int j = s->j0; j < s->j1; ++j) {
        double shift = -INFINITY;
        for (int pass = 0; pass < 2; ++pass) {
            double acc = 0.0;
            for (int i = 0; i < s->nred; ++i) {
                if (!(s->w[i] > 0.0)) continue;
                double c;
                if (s->kind == COST_SQEUCLID) {
                    c = 0.0;
                    for (int k = 0; k < s->d; ++k) {
                        double t = s->xr[(long)i * s->d + k] - s->xo[(long)j * s->d + k];
                        c += t * t;
                    }
                } else if (s->kind == COST_POWER1D) {
                    c = pow_cost(s->xr[i], s->xo[j], s->p);
                } else {
                    c = s->cm[(long)i * s->ldi + (long)j * s->ldj];
                }
                double v = (s->pot[i] - c) / s->eps;
                if (pass == 0) {
                    if (v > shift) shift = v;
                } else {
                    acc += s->w[i] * exp(v - shift);
                }
            }
            if (pass == 0) {
                if (!isfinite(shift)) shift = 0.0;
            } else {
                s->out[j] = -s->eps * (log(acc) + shift);
            }
        }
    }
    return NULL;
}

/* Worker count: ORACLE_THREADS, else the online CPU count. */
static int oracle_threads(void) {
    const char* env = getenv("ORACLE_THREADS");
    int t = env ? atoi(env) : (int)sysconf(_SC_NPROCESSORS_ONLN);
    return t < 1 ? 1 : (t > 256 ? 256 : t);
}

void oracle_smin(int kind, int nred, int nout, int d, const double* xr, const double* xo,
                 double p, const double* cm, long ldi, long ldj, const double* pot,
                 const double* w, double eps, double* out) {
    int nt = oracle_threads();
    if ((long)nred * nout < 65536) nt = 1;
    if (nt > nout) nt = nout;
    pthread_t th[256];
    smin_job jobs[256];
    for (int t = 0; t < nt; ++t) {
        smin_job s = {kind, nred, nout, d, xr, xo, cm, pot, w, p, eps, ldi, ldj, out,
                      (int)((long)nout * t / nt), (int)((long)nout * (t + 1) / nt)};
        jobs[t] = s;
    }
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, smin_worker, &jobs[t]);
    smin_worker(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

/*
 * Balanced 1-D OT by the monotone north-west sweep: ot1d.py:112-172
 * (Algorithm 1).  Entries with step > 0 are emitted;
 * f_0 = 0, g_0 = C(0,0); a source advance sets f_i = C(i,j) - g_j, a target
 * advance sets g_j = C(i,j) - f_i; ties advance the source unless it sits at
 * its last atom (ot1d.py:158).  Mass validation is done by the caller
 * (ot1d.py:133-136).  Returns the number of entries written (<= n+m-1).
 */
long oracle_ot1d(int n, int m, const double* x, const double* y, const double* wa,
                 const double* wb, int kind, double p, const double* cm, int64_t* ei,
                 int64_t* ej, double* em, double* f, double* g) {
#define COST(I, J) (kind == COST_EXPLICIT ? cm[(long)(I) * m + (J)] : pow_cost(x[I], y[J], p))
    for (int i = 0; i < n; ++i) f[i] = 0.0;
    for (int j = 0; j < m; ++j) g[j] = 0.0;
    g[0] = COST(0, 0);
    long e = 0;
    int i = 0, j = 0;
    double rem_a = wa[0], rem_b = wb[0];
    for (;;) {
        double step = rem_a < rem_b ? rem_a : rem_b;
        if (step > 0) {
            ei[e] = i;
            ej[e] = j;
            em[e] = step;
            ++e;
        }
        rem_a -= step;
        rem_b -= step;
        if (i == n - 1 && j == m - 1) break;
        if ((rem_a <= rem_b && i < n - 1) || j == m - 1) {
            ++i;
            rem_a = wa[i];
            f[i] = COST(i, j) - g[j];
        } else {
            ++j;
            rem_b = wb[j];
            g[j] = COST(i, j) - f[i];
        }
    }
    return e;
#undef COST
}

/* barycenter.py:148-156 (multimarginal_cost): sum_k w_k (x_k - B)^2, B = <w, x>. */
static double bary_cost(int k, const double* w, const double* pts) {
    double b = 0.0;
    for (int q = 0; q < k; ++q) b += w[q] * pts[q];
    double c = 0.0;
    for (int q = 0; q < k; ++q) {
        double t = pts[q] - b;
        c += w[q] * (t * t);
    }
    return c;
}

/*
 * Balanced K-marginal sweep: barycenter.py:169-233 (Algorithm 3,
 * PAPER.md:707-726).  Lists are concatenated: list q occupies
 * [off[q], off[q] + len[q]) of xs / ws / pots.  At each step the coordinate
 * with the least remaining mass among those that can still advance is
 * exhausted (ties -> lowest q, the first argmin, barycenter.py:218); rem is
 * clamped at 0 (:223); the advanced coordinate's potential is set through
 * sum_k f_k = cost on the new tuple (:225-229).  Entry tuples go to
 * idx[e*k + q].  Returns the entry count.
 */
long oracle_mot1d(int k, const int* len, const long* off, const double* xs, const double* ws,
                  const double* w, int64_t* idx, double* mass, double* pots) {
    int64_t* cur = (int64_t*)calloc((size_t)k, sizeof(int64_t));
    double* rem = (double*)malloc(sizeof(double) * k);
    double* pts = (double*)malloc(sizeof(double) * k);
    long total = 0;
    for (int q = 0; q < k; ++q) total += len[q];
    for (long t = 0; t < total; ++t) pots[t] = 0.0;
    for (int q = 0; q < k; ++q) {
        rem[q] = ws[off[q]];
        pts[q] = xs[off[q]];
    }
    pots[off[0]] = bary_cost(k, w, pts);
    double pot_sum = pots[off[0]];
    long e = 0;
    for (;;) {
        int p = -1;
        double best = INFINITY;
        for (int q = 0; q < k; ++q) {
            if (cur[q] < len[q] - 1 && rem[q] < best) {
                best = rem[q];
                p = q;
            }
        }
        if (p < 0) {
            double step = rem[0];
            for (int q = 1; q < k; ++q) step = rem[q] < step ? rem[q] : step;
            if (step > 0) {
                for (int q = 0; q < k; ++q) idx[e * k + q] = cur[q];
                mass[e++] = step;
            }
            break;
        }
        double step = rem[p];
        if (step > 0) {
            for (int q = 0; q < k; ++q) idx[e * k + q] = cur[q];
            mass[e++] = step;
        }
        for (int q = 0; q < k; ++q) {
            double r = rem[q] - step;
            rem[q] = r > 0.0 ? r : 0.0;
        }
        cur[p] += 1;
        pts[p] = xs[off[p] + cur[p]];
        double old = pots[off[p] + cur[p] - 1];
        double nw = bary_cost(k, w, pts) - (pot_sum - old);
        pots[off[p] + cur[p]] = nw;
        pot_sum += nw - old;
        rem[p] = ws[off[p] + cur[p]];
    }
    free(cur);
    free(rem);
    free(pts);
    return e;
}
