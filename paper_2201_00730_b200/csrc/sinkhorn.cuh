// sinkhorn.cuh -- fused F/H-Sinkhorn half-steps (K1 of SURVEY.md §2.2).
//
// Reference: src/sinkhorn.py:93-163 (_smin_cols/_smin_rows, f_sinkhorn_step,
// h_sinkhorn_step) on top of src/entropies.py:67-92 (logdotexp) and
// :187-214 (softmin, KL aprox), src/duality.py:175-178 (lambda_star).
//
// One half-step = two launches:
//   sk_main  : for every output index o, a register-resident online
//              log-sum-exp over a split of the reduced index r of
//              arg(r, o) = (pot_r - C(r,o))/eps + log w_r, with C computed on
//              the fly from the point coordinates (staged through shared
//              memory).  Emits one (shift, sum) partial per (split, o).
//   sk_tail  : combines the partials, applies the KL aprox scale and the
//              translation-invariant correction, packs the reduced-side
//              records for the next half-step, and reduces the closed-form
//              translation scalars (softmin over the output side) with a
//              last-block-done grid reduction.  The scalar shift
//              k/(1-k) * Smin is kept separate ("hat" vectors + tau scalars)
//              and folded into the next half-step lazily, so no extra pass
//              over the vectors is ever needed.
#pragma once

#include "common.cuh"

namespace uot {

// Per-problem scalar state of the engine (double precision always).
struct SkScalars {
  double shat[2];  // Smin^{rho_s}_{w_s}(hat_s) of side s (0 = source/f, 1 = target/g)
  double tau[2];   // lazy translation of side s: potential_s = hat_s + tau[s]
  double lam;      // G variant: translation of the current pair (lambda*)
};

template <typename T>
struct DirGeo {
  const T* red_rec;     // packed records of the reduced side [B][nred][rw]
  long red_bstride;     // elements per problem
  int rw;               // record width (elements)
  const T* out_pts;     // points of the output side [B][nout][d]
  long out_pts_bstride;
  int d;
  T L;                  // exponent scale 1/(eps*unit)
  T p;                  // power exponent (power-1D cost)
  const T* cmat;        // explicit cost: C(r,o) = cmat[b*cm_bstride + r*ld_r + o*ld_o]
  long cm_bstride, ld_r, ld_o;
  const T* ctr;         // tcgen05 path: per-problem centre [B][d] (tc_center)
  long ctr_bstride;
  T ascale;             // tcgen05 path: power-of-two scale of the A operand (B gets 2L/ascale)
  int tc_full;          // tcgen05 path: also the Yl*Xl product (2L > 128, i.e. eps < ~0.0225)
  const uint32_t* tc_pack;  // tcgen05 path: precomputed A rows of the output side (tc_pack_out)
  long tc_pack_bstride;     // words per problem
};

template <typename T>
struct MainArgs {
  DirGeo<T> g;
  int nred, nout;
  const T* shift_in;  // [B][nout] stale log-sum-exp estimate (domain units)
  T* part_m;          // [B][S][nout]
  T* part_a;          // [B][S][nout]
  const int* done;    // [B] or nullptr
  int chunk;          // records staged per shared-memory chunk
  int red_offset;     // reduced range handled by this launch: [red_offset, red_offset+nred)
  int split_base;     // first split index written by this launch
  int splits_total;   // S of the partial buffer layout
  int out_lo, out_hi; // output range of this launch (out_hi == 0: all nout outputs)
};

template <typename T>
struct TailArgs {
  int nout, nparts;   // partials per output to combine
  int mode;           // 0 = combine partials, 1 = init from pot_in
  int out_side, red_side;
  const T* part_m;    // part (b, s) of output o at b*pstride_b + s*pstride_s + o
  const T* part_a;
  long pstride_b, pstride_s;
  const T* pot_in;    // [B][nout] (init mode)
  SkScalars* sc;      // [B]
  double eps, unit, inv_eu;    // unit = ln2 (log2 domain) or 1; inv_eu = 1/(eps*unit)
  double a_coef, k_coef;       // hat = a*smin - k*(shat_red + tau_red)
  double tau_fac;              // tau_out = tau_fac * shat_out
  int gmode;                   // G variant: hat includes lam, then lam = lambda* (KL/KL)
  double rho1, rho2;
  int ent_out;                 // UOT_ENT_* of the output side's marginal
  int lam_closed;              // G: lambda* in closed form (KL/KL) in the f-tail
  double rho_out;
  T* hat_out;                  // [B][nout]
  const T* hat_old;            // [B][nout] or nullptr (delta tracking)
  T* shift_out;                // [B][nout]
  T* rec_out;                  // [B] x rec_bstride records of the output side
  long rec_bstride;
  int rw;
  const T* out_pts;            // [B][nout][d]
  const T* ctr;                // [B][d] centre of the fp32 expanded-form records, or nullptr
  int d;
  const T* out_w;              // [B][nout]
  T L, p;
  double* blk;                 // [B][nblocks][4]
  unsigned int* counter;       // [B]
  double* trace;               // [B][trace_len] or nullptr
  int trace_len, t;
  int t_dev;                   // 1: t = iters_done[b] (graph-replayed iterations)
  int* iters_done;             // [B]
  int* done;                   // [B]
  double tol;
  int use_tol;
  // Row sharding (sinkhorn.cu run_sharded): shard = 1 makes the tail publish
  // its partial output-side scalars (LSE pair of -hat/rho, delta bounds) to
  // xs_out[b*4..] instead of finalising them; shard = 2 resolves the reduced
  // side's scalars from the ranks' gathered slots xs_in[r*xs_stride + b*4..].
  int shard;
  const double* xs_in;
  long xs_stride;
  int nranks;
  int first;
  double rho_red, tau_fac_red;
  double* xs_out;
};

}  // namespace uot
