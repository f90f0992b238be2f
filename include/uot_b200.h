/*
 * uot_b200.h -- C-ABI of the B200 (sm_100a) implementation of the two hot
 * paths of arXiv 2201.00730: translation-invariant (H-) Sinkhorn for entropic
 * unbalanced OT, and 1-D Frank-Wolfe UOT with its multimarginal barycenter.
 *
 * The reference (uotkit, /root/reference/pkg/src/uotkit) is pure Python; its
 * "plugin boundary" is the public solver API re-exported by
 * src/__init__.py:10-70.  Each entry point below names the reference
 * interface it replaces (file:line, relative to that package).
 *
 * Conventions:
 *  - Plain pointers and sizes.  Array arguments are DEVICE pointers unless
 *    stated; dtype is given per call (fp32 or fp64).  Batched arrays are
 *    dense row-major with the batch index outermost.
 *  - No allocation inside: the caller provides a device workspace whose size
 *    is returned by the matching *_workspace_size query.
 *  - Work is enqueued on the caller's cudaStream_t (passed as void*); calls
 *    are reentrant per stream.
 *  - Every call returns a status.  Codes map onto the reference exceptions
 *    (src/exceptions.py:4-25): 1 MassBalanceError, 2 UnsupportedEntropyError,
 *    3 ValueError, 6 InfeasibleDualError; 4/5 are CUDA / NCCL failures.
 *    uot_last_error() returns a thread-local message for the last failure.
 */
#ifndef UOT_B200_H
#define UOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  UOT_OK = 0,
  UOT_ERR_MASS_BALANCE = 1,
  UOT_ERR_UNSUPPORTED_ENTROPY = 2,
  UOT_ERR_INVALID = 3,
  UOT_ERR_CUDA = 4,
  UOT_ERR_NCCL = 5,
  UOT_ERR_INFEASIBLE = 6
};

enum { UOT_F32 = 0, UOT_F64 = 1 };
enum { UOT_SINKHORN_F = 0, UOT_SINKHORN_H = 1, UOT_SINKHORN_G = 2 };
/* marginal penalties (src/entropies.py): KL(rho), Berg(rho), Balanced */
enum { UOT_ENT_KL = 0, UOT_ENT_BERG = 1, UOT_ENT_BALANCED = 2 };
/* Ground costs: squared Euclidean between d-dim point clouds; |x-y|^p on 1-D
 * points (src/measures.py:93-105 PowerDistance); dense explicit matrix
 * (src/measures.py:108-122 ExplicitMatrix). */
enum { UOT_COST_SQEUCLID = 0, UOT_COST_POWER = 1, UOT_COST_EXPLICIT = 2 };
enum { UOT_STEP_HARMONIC = 0, UOT_STEP_LINESEARCH = 1, UOT_STEP_PAIRWISE = 2 };

/* Library identity / diagnostics. */
const char* uot_version(void);
const char* uot_last_error(void);
int uot_device_arch(int device, int* sm_major, int* sm_minor);

/* ------------------------------------------------------------------------
 * Sinkhorn: replaces src/sinkhorn.py:246-315 `run(prob, config, init)` for
 * variants "f" (f_sinkhorn_step, :103-114), "h" (h_sinkhorn_step,
 * :137-163) and "g" (g_sinkhorn_step, :117-134: translated steps at the
 * incoming lambda, then lambda* of the new pair; unsharded), with the
 * marginal penalties ent1 / ent2 (KL, Berg, Balanced; "h" is KL/KL), for a
 * batch of independent problems, with a fixed iteration budget and the
 * reference's optional `delta_f < tol` stop (:304-306) evaluated per problem.
 * fp32 squared-Euclidean costs with d >= 32 (d % 4 == 0) run on the tensor
 * cores (tcgen05: fp16 hi/lo split cost tiles + a tf32 constants MMA, points
 * taken relative to the midpoint of the two clouds' centroids, operands balanced by a
 * power-of-two scale; the fp16 range holds while 2 R^2 / (eps ln 2) < ~4e9,
 * R = the largest distance to that point -- beyond it the fp32 log-domain
 * exponents themselves carry no precision).
 *
 * Inputs (dtype elements): x [batch][n][d], y [batch][m][d] (d = 1 for
 * UOT_COST_POWER); explicit costs c [batch][n][m] and its transpose
 * ct [batch][m][n]; weights a [batch][n], b [batch][m].  f [batch][n] holds
 * the initial f when init_given (the g input is unused by "f" and "h", as in
 * the reference; "g" starts from lambda*(f, g) of the given pair, :263-265)
 * and receives the final pair with g.
 * trace_delta [batch][iters] (fp64) receives ||f_t - f_{t-1}||_inf,
 * iterations [batch] the number of steps taken.
 *
 * Row sharding (BASELINE cfg3): with nccl_comm != NULL the n rows given are
 * this rank's slice of a problem whose target side (y, b, g) is replicated;
 * column partial log-sum-exps are exchanged with one ncclAllGather per
 * iteration.  nranks > 1 with nccl_comm == NULL emulates the same protocol
 * in one process on one GPU (x, a, f then hold all shards back to back and
 * shard_rows[nranks] gives the row count of each shard).
 * ------------------------------------------------------------------------ */
typedef struct uot_sinkhorn_desc {
  int32_t variant, dtype, cost;
  int32_t batch, n, m, d;
  double p;
  double eps, rho1, rho2;
  const void* x;
  const void* y;
  const void* c;
  const void* ct;
  const void* a;
  const void* b;
  void* f;
  void* g;
  int32_t init_given;
  int32_t iters;
  double tol;
  int32_t use_tol;
  double* trace_delta;
  int32_t* iterations;
  void* nccl_comm;
  int32_t nranks, rank;
  const int32_t* shard_rows; /* host array [nranks] (emulation only) */
  int32_t ent1, ent2;        /* UOT_ENT_*: "h" needs KL/KL, "g" KL or Berg, "f" any */
  int32_t lam_given;         /* "g", single device: start from lam0 instead of lambda*(f0, g0) */
  double lam0;               /* (g_sinkhorn_step's incoming lam, src/sinkhorn.py:117-134) */
  int32_t* status;           /* optional [batch]: 0, or the NewtonError of the G variant's
                                lambda* with a Berg marginal (src/duality.py:182-247):
                                1 empty domain, 2 no bracket, 3 no convergence; the problem
                                stops at that iteration */
  int32_t warm_shifts;       /* nonzero: the workspace still holds a previous call's state
                                for the same problem (a continued run): its per-output
                                log-sum-exp shifts seed this call's tiles */
} uot_sinkhorn_desc;

int uot_sinkhorn_workspace_size(const uot_sinkhorn_desc* desc, size_t* bytes);

/* Verification of a given pair at scale: f, g of the
 * descriptor are INPUTS (not modified; iters / init_given ignored).  Two
 * on-the-fly cost passes, no N x M matrix.  out [batch][8] (fp64):
 *   [0] res_g = max_j |g - a2 smin_cols(f) - eps/(eps+rho2) lam|  (src/sinkhorn.py:166-189)
 *   [1] log <alpha x beta, exp((f + g - C)/eps)>                 (src/duality.py:124-132)
 *   [2] res_f = max_i |f - a1 smin_rows(g) + eps/(eps+rho1) lam|
 *   [4] lam = lambda*(f, g) (KL, duality.py:175-178)
 *   [5] Smin_alpha^rho1(f), [6] Smin_beta^rho2(g)  (entropies.py:187-200)
 * from which eval_F / eval_G / eval_H follow in closed form (KL).
 * Workspace: uot_sinkhorn_workspace_size of the same descriptor. */
int uot_sinkhorn_verify(const uot_sinkhorn_desc* desc, void* workspace, size_t workspace_bytes,
                        void* stream, double* out);
int uot_sinkhorn_run(const uot_sinkhorn_desc* desc, void* workspace, size_t workspace_bytes,
                     void* stream);

/* Softmin / log-sum-exp reductions used by the API mirror:
 * replaces src/duality.py:160-178 `lambda_star` (KL closed form),
 * src/entropies.py:187-200 `softmin` and src/duality.py:279-290 `_eval_h_kl`
 * for a batch: out[b*3 + 0] = lambda*, out[b*3 + 1] = H_0 (no eps term),
 * out[b*3 + 2] = Smin_a^{rho1}(f).  fp64, device pointers, out [batch][3]. */
int uot_kl_scalars(int32_t batch, int32_t n, int32_t m, const double* a, const double* b,
                   const double* f, const double* g, double rho1, double rho2, double* out,
                   void* stream);

/* ------------------------------------------------------------------------
 * Anderson extrapolation of the Sinkhorn map: replaces the window state of
 * src/sinkhorn.py:215-243 (`_AndersonState.push` / `extrapolate`) and
 * src/sinkhorn.py:197-212 `anderson_weights`, as used by run() with
 * `config.anderson` (:281-292).  fp64, device pointers, `batch` independent
 * windows over vectors of length len = n + m (the concatenated (f, g)).
 * uot_anderson_step pushes (tz, tz - z) -- restarting the window when the new
 * residual's sup norm exceeds the previous one's, keeping the last `depth`
 * entries -- then writes the extrapolation to znew (may alias z) and
 * delta_f[b] = max_{i < nf} |znew - z|.  status[b] = 1 when the window
 * system is singular / degenerate (the reference raises LinAlgError).
 * Device limit: depth <= 32.  The workspace is persistent state: call
 * uot_anderson_reset once before the first step.
 * ------------------------------------------------------------------------ */
int uot_anderson_workspace_size(int32_t batch, int64_t len, int32_t depth, size_t* bytes);
int uot_anderson_reset(int32_t batch, int64_t len, int32_t depth, void* workspace,
                       size_t workspace_bytes, void* stream);
int uot_anderson_step(int32_t batch, int64_t len, int64_t nf, int32_t depth, double reg,
                      const double* z, const double* tz, double* znew, double* delta_f,
                      int32_t* status, void* workspace, size_t workspace_bytes, void* stream);
/* anderson_weights(U, r) for one window U [rows][k] (row-major): c [k],
 * status (device int32) 1 on a singular system.  k <= 32. */
int uot_anderson_weights(int32_t rows, int32_t k, const double* U, double reg, double* c,
                         int32_t* status, void* stream);

/* ------------------------------------------------------------------------
 * Entropy family (src/entropies.py), fp64, device pointers:
 *  uot_logdotexp: out[o*inner + i] = log sum_k w[k] exp(scale v[o][k][i]) with
 *    zero-weight entries masked before the max shift -- :67-92 `logdotexp`
 *    (flat: outer = inner = 1; `softmin` :187-200 is scale = -1/eps).
 *  uot_entropy_map: op 0 conj, 1 conj_grad, 2 conj_hess, 3 aprox of entropy
 *    `ent` (UOT_ENT_*) elementwise -- :142-221; *bad (device int32) = 1 when a
 *    Berg argument leaves x < rho (the reference raises ValueError).
 *  uot_divergence: out[0] = D(mu | nu) -- :104-140 (+inf where the reference
 *    returns +inf).
 * ------------------------------------------------------------------------ */
int uot_logdotexp(int64_t outer, int64_t k, int64_t inner, const double* v, const double* w,
                  double scale, double* out, void* stream);
int uot_entropy_map(int32_t op, int32_t ent, double rho, double eps, int64_t n, const double* x,
                    double* out, int32_t* bad, void* stream);
int uot_divergence(int32_t ent, double rho, int64_t n, const double* mu, const double* nu,
                   double* out, void* stream);

/* ------------------------------------------------------------------------
 * Dense and plan-level helpers of the reference API (fp64, device pointers):
 *  uot_cost_matrix: C[i*m + j] = |x_i - y_j|^p -- src/measures.py:125-145
 *    `build_cost_matrix` (p = 1: |d|, p = 2: d*d as the reference).
 *  uot_cost_quadruple_diameter: out[0] = max_{k,l} range_j (C[j,k] - C[j,l])
 *    -- src/measures.py:168-184 (used by birkhoff_rate_bound,
 *    src/sinkhorn.py:338-346).
 *  uot_updated_marginals: ta = a exp((-f - lam)/rho1), tb = b exp((-g + lam)/rho2)
 *    -- src/duality.py:293-303 for KL/KL (lam = lambda*(f, g)).
 *  uot_eval_primal: out[0] = <plan, C> + eps KL(plan | a x b) + D1 + D2 over
 *    the plan entries (ii, jj, mass)[E] -- src/duality.py:306-344; cost from
 *    x, y, p (1-D power) or the dense C when non-NULL; KL / Berg / Balanced
 *    divergences (UOT_ENT_*), +inf where the reference returns +inf.
 * ------------------------------------------------------------------------ */
int uot_cost_matrix(int32_t n, int32_t m, const double* x, const double* y, double p, double* C,
                    void* stream);
int uot_cost_quadruple_diameter(int32_t n, int32_t m, const double* C, double* out, void* stream);
int uot_updated_marginals(int32_t n, int32_t m, const double* a, const double* b, const double* f,
                          const double* g, double rho1, double rho2, double lam, double* ta,
                          double* tb, void* stream);
int uot_eval_primal(int32_t n, int32_t m, const double* x, const double* y, double p,
                    const double* C, const double* a, const double* b, int32_t E,
                    const int64_t* ii, const int64_t* jj, const double* mass, int32_t ent1,
                    int32_t ent2, double rho1, double rho2, double eps, double* out, void* stream);

/* ------------------------------------------------------------------------
 * Balanced 1-D OT (Algorithm 1): replaces src/ot1d.py:112-172
 * `solve_ot_1d(a, b, cost)` for a batch of problems with sorted supports.
 * fp64.  Costs: UOT_COST_POWER with exponent p, or UOT_COST_EXPLICIT with
 * c [batch][n][m].  Outputs: f [batch][n], g [batch][m]; plan entries
 * (ei, ej int32, em fp64) [batch][n+m-1] with count [batch]; entries are in
 * sweep order.  status [batch] gets 1 for a mass mismatch above 1e-9
 * relative (src/ot1d.py:133-136).  An ExplicitMatrix cost (device c,
 * row-major per problem) is looked up at C(i, j) along the staircase
 * exactly as src/ot1d.py:100-107 does; the caller validates it (Monge check,
 * src/measures.py:148-165); p is ignored then.  n, m <= 4096 per problem.
 * ------------------------------------------------------------------------ */
int uot_ot1d_workspace_size(int32_t batch, int32_t n, int32_t m, size_t* bytes);
int uot_ot1d_batched(int32_t batch, int32_t n, int32_t m, const double* x, const double* y,
                     const double* a, const double* b, int32_t cost, double p, const double* c,
                     double* f, double* g, int32_t* ei, int32_t* ej, double* em, int32_t* count,
                     int32_t* status, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Batched 1-D Frank-Wolfe UOT at eps = 0: replaces src/fw.py:176-232
 * `fw_solve(prob, FwConfig(step, max_iters, gap_tol))` (+ `_lmo` :159-173,
 * `_h0` :106-115, `eval_primal` src/duality.py:320-344, line search
 * :131-148, `_finalize` :235-252) for KL(rho1)/KL(rho2) marginals and
 * |x-y|^p costs on sorted supports, or an explicit (Monge) cost matrix c
 * [batch][n][m] when c != NULL (ExplicitMatrix, src/fw.py:168-172).  fp64.
 *
 * f, g [batch][n|m]: in = initial pair (must be dual feasible), out = the
 * final iterate TRANSLATED by lambda* (report.final).  Traces
 * [batch][max_iters] h0, fw_gap, pd_gap; iterations [batch]; the last
 * oracle plan (ei, ej, em, count) as for uot_ot1d_batched; final primal /
 * dual / lambda* in summary [batch][3]; status [batch] (1 = reweighted
 * masses disagree, fw.py:161-166).  With early_exit != 0 a problem stops at
 * the first pd_gap < gap_tol (fw.py:220-222).
 * step = UOT_STEP_PAIRWISE runs pairwise FW (src/fw.py:255-357): an atom
 * store of up to max_iters + 1 dual-pair atoms per problem lives in the
 * workspace; natoms (optional [batch][max_iters]) receives the active atom
 * count after each iteration and step_size the weight transferred.
 * n, m <= 4096 per problem (one CTA per problem, state resident on chip).
 * A Berg penalty on either side (ent1 / ent2 = UOT_ENT_BERG, src/fw.py:98-103)
 * runs the generic path (csrc/fw1d_generic.cu): per iteration the bracketed
 * Newton translation (src/duality.py:182-247), the oracle and a ternary line
 * search whose every value solves its own translation (fw.py:106-148);
 * harmonic / line search steps; the call synchronises the stream every 16
 * iterations to test the early exit.  status 3 = NewtonError.
 * ------------------------------------------------------------------------ */
typedef struct uot_fw_desc {
  int32_t batch, n, m;
  double p;
  double rho1, rho2;
  int32_t step;       /* UOT_STEP_* */
  int32_t max_iters;
  double gap_tol;
  int32_t early_exit;
  const double* x;
  const double* y;
  const double* a;
  const double* b;
  double* f;
  double* g;
  double* h0;
  double* fw_gap;
  double* pd_gap;
  int32_t* iterations;
  int32_t* ei;
  int32_t* ej;
  double* em;
  int32_t* count;
  double* summary;
  int32_t* status;
  double* step_size; /* optional [batch][max_iters]: gamma of each iteration */
  int32_t* natoms;   /* optional [batch][max_iters]: active atoms (pairwise) */
  const double* ref_f; /* optional [batch][n]: reference potential (src/fw.py:217-219) */
  double* err_f;       /* optional [batch][max_iters]: ||f_t + lambda*_t - ref_f||_inf */
  const double* c;     /* optional [batch][n][m]: explicit cost (else |x - y|^p) */
  int32_t ent1, ent2;  /* UOT_ENT_KL (0, default) or UOT_ENT_BERG per marginal */
  /* Parity / trace mode (all optional, NULL = off; KL path):
   * step_in [batch][max_iters]: replay these step sizes instead of the step
   *   rule (the reference's gamma_t, src/fw.py:223-230 / :295-297);
   * away_in [batch][max_iters]: pairwise only, the away position in the
   *   active list (insertion order, fw.py:287), -1 = no step that iteration;
   * supp_hash / supp_nnz [batch][max_iters]: hash and entry count of every
   *   iteration's oracle plan support (plan-hash definition below). */
  const double* step_in;
  const int32_t* away_in;
  uint64_t* supp_hash;
  int32_t* supp_nnz;
} uot_fw_desc;

int uot_fw1d_workspace_size(const uot_fw_desc* desc, size_t* bytes);
int uot_fw1d_run(const uot_fw_desc* desc, void* workspace, size_t workspace_bytes, void* stream);

/* Dense feasibility check max(0, max_ij f_i + g_j - C_ij) for 1-D power
 * costs: replaces src/duality.py:117-121 `dual_feasibility_violation`.
 * out [batch] fp64. */
int uot_feasibility_1d(int32_t batch, int32_t n, int32_t m, const double* x, const double* y,
                       double p, const double* f, const double* g, double* out, void* stream);
/* Optimal translation lambda* of (f, g) for KL / Berg penalties by the
 * bracketed Newton of src/duality.py:182-247 started at lam0 (solve != 0; stop at
 * |residual| < tol within max_iters Newton steps -- the reference's 1e-11 / 100), or
 * lambda = lam0 given (solve == 0, e.g. eval_G / eval_F).  Optional outputs:
 * lam [batch]; ta, tb [batch][n|m] = weights * conj_grad(-f - lam | -g + lam)
 * (updated_marginals, :293-303); h [batch] = <a, -phi1*(-(f + lam))> +
 * <b, -phi2*(-(g - lam))> (_h0, src/fw.py:111-115; src/duality.py:102-114,
 * Balanced allowed when solve == 0); status [batch]: 0, 1 = empty Berg
 * domain, 2 = no bracket, 3 = no convergence (NewtonError). */
int uot_translation(int32_t batch, int32_t n, int32_t m, const double* a, const double* b,
                    const double* f, const double* g, int32_t ent1, int32_t ent2, double rho1,
                    double rho2, int32_t solve, double lam0, double tol, int32_t max_iters,
                    double* lam, double* ta, double* tb, double* h, int32_t* status, void* stream);
/* The same for explicit costs C [batch][n][m] (ExplicitMatrix). */
int uot_feasibility_explicit(int32_t batch, int32_t n, int32_t m, const double* C,
                             const double* f, const double* g, double* out, void* stream);

/* ------------------------------------------------------------------------
 * Balanced K-marginal sweep (Algorithm 3) and the KL barycenter FW:
 * replace src/barycenter.py:169-233 `solve_mot_1d(inputs, w)` and
 * :330-430 `fw_barycenter(problem, config)` (with _h_value :320-327,
 * multimarginal_lambda :298-317, plan_cost :236-240, the final translation
 * :413-414) for a batch of problems with K (2..16) sorted inputs, fp64.
 * x, a, f [batch][K][n] (row stride n; list q holds lens[q] <= n atoms when
 * the optional host array lens is given); omega [K] barycentric weights
 * (host); rho_k = omega_k * rho (barycenter.py:81-84).  Plans come back as
 * tuple indices [batch][K*(n-1)+1][K] int32 and masses [batch][K*(n-1)+1]
 * with count [batch], positive-mass states only, in sweep order.
 * ------------------------------------------------------------------------ */
typedef struct uot_bary_desc {
  int32_t batch, k, n;
  const double* omega;  /* host array [k] */
  const int32_t* lens;  /* host array [k] or NULL (all lists have n atoms) */
  double rho;
  int32_t step;
  int32_t max_iters;
  double gap_tol;
  int32_t early_exit;
  const double* x;
  const double* a;
  double* f;           /* in: initial potentials; out: translated final potentials */
  double* h0;
  double* fw_gap;
  double* pd_gap;
  int32_t* iterations;
  int32_t* idx;        /* [batch][k*(n-1)+1][k] */
  double* mass;        /* [batch][k*(n-1)+1] */
  int32_t* count;
  double* summary;     /* [batch][2]: primal, dual of the last iteration */
  int32_t* status;
  /* Parity / trace mode (optional, NULL = off): step_in [batch][max_iters]
   * replays the reference's gamma_t (barycenter.py:397-411); supp_hash /
   * supp_nnz [batch][max_iters] receive every iteration's plan support hash
   * and entry count. */
  const double* step_in;
  uint64_t* supp_hash;
  int32_t* supp_nnz;
} uot_bary_desc;

/* Plan-support hash of the trace mode (supp_hash above):
 *   mix64(z): z += 0x9e3779b97f4a7c15; z = (z ^ z>>30) * 0xbf58476d1ce4e5b9;
 *             z = (z ^ z>>27) * 0x94d049bb133111eb; return z ^ z>>31
 *   entry with index tuple (i_0 .. i_{K-1}) (K = 2 for the 1-D OT plan):
 *             mix64(sum_q mix64(((q + 1) << 40) | i_q))   (mod 2^64)
 *   plan:     sum of the entry hashes over the positive-mass entries (mod 2^64)
 * Equal supports give equal hashes; the tests compare them with the hash of
 * the reference's SparsePlan / MultiPlan indices at every iteration. */

int uot_mot1d_workspace_size(int32_t batch, int32_t k, int32_t n, size_t* bytes);
/* f receives the sweep's dual potentials (barycenter.py:206-229). */
int uot_mot1d_batched(int32_t batch, int32_t k, int32_t n, const int32_t* lens, const double* x,
                      const double* a, const double* omega_host, double* f, int32_t* idx,
                      double* mass, int32_t* count, int32_t* status, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Certificate of a balanced multi-marginal solution (replaces
 * src/barycenter.py:261-295 `mot_certificate` + :236-240 `plan_cost` +
 * :243-258 `dual_feasibility_exhaustive` for the barycentric cost).  Inputs
 * as uot_mot1d_batched's outputs: f [batch][k][n], idx [batch][k*(n-1)+1][k],
 * mass, count.  out [batch][6]: primal (plan cost), dual sum_k <a_k, f_k>,
 * support violation max_e |sum_k f_k - Cc|, marginal violation, exhaustive
 * feasibility violation (only when the grid has <= 1e5 tuples), and 1.0 if
 * that sweep ran.  workspace >= 32 k + 256 bytes (device). */
int uot_mot_certify(int32_t batch, int32_t k, int32_t n, const int32_t* lens, const double* x,
                    const double* a, const double* omega_host, const double* f,
                    const int32_t* idx, const double* mass, const int32_t* count, double* out,
                    void* workspace, size_t workspace_bytes, void* stream);

/* Custom tuple costs: `solve_mot_1d(inputs, costfn=...)`, `plan_cost`,
 * `dual_feasibility_exhaustive`, `mot_certificate(..., costfn)`
 * (src/barycenter.py:169-233, 236-295).  The sweep order depends only on the
 * weights, so a caller-supplied costfn (a host callable) is evaluated by the
 * caller on the tuples the device returns:
 *   1. uot_mot1d_states: every state the sweep visits, zero-mass ones
 *      included, idx [batch][K*(n-1)+1][K], mass, count = 1 + sum_q (len_q-1)
 *      (barycenter.py:209-229: the initial tuple, then one per advance);
 *      status as uot_mot1d_batched (1 = unequal masses).  Workspace of
 *      uot_mot1d_workspace_size.
 *   2. the caller evaluates cost[b][t] = costfn(points of state t);
 *   3. uot_mot1d_cost_duals: f [batch][K][n] with f_1[0] = cost[0], f_k[0] = 0
 *      and f_p[i] = f_p[i-1] + cost[t] - cost[t-1] for the state t advancing
 *      list p to i (:224-228).
 * uot_mot_certify_costs: uot_mot_certify with ecost [batch][K*(n-1)+1] =
 * costfn at the plan entries and, for grids of at most 1e5 tuples, gcost
 * [batch][grid] = costfn over the index grid in C order (NULL skips the
 * exhaustive sweep). */
int uot_mot1d_states(int32_t batch, int32_t k, int32_t n, const int32_t* lens, const double* a,
                     int32_t* idx, double* mass, int32_t* count, int32_t* status,
                     void* workspace, size_t workspace_bytes, void* stream);
int uot_mot1d_cost_duals(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                         const int32_t* idx, const int32_t* count, const double* cost, double* f,
                         void* workspace, size_t workspace_bytes, void* stream);
int uot_mot_certify_costs(int32_t batch, int32_t k, int32_t n, const int32_t* lens,
                          const double* a, const double* f, const int32_t* idx,
                          const double* mass, const int32_t* count, const double* ecost,
                          const double* gcost, double* out, void* workspace,
                          size_t workspace_bytes, void* stream);
int uot_bary_workspace_size(const uot_bary_desc* desc, size_t* bytes);
int uot_bary_run(const uot_bary_desc* desc, void* workspace, size_t workspace_bytes,
                 void* stream);

/* ------------------------------------------------------------------------
 * NCCL plumbing for the row-sharded Sinkhorn (one process per GPU).  The
 * unique id is 128 opaque bytes broadcast by the host (torch.distributed).
 * ------------------------------------------------------------------------ */
int uot_nccl_unique_id(char out[128]);
int uot_nccl_comm_init(const char id[128], int32_t nranks, int32_t rank, void** comm);
int uot_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* UOT_B200_H */
