// sinkhorn_tc.cuh -- tensor-core half-step for squared-Euclidean costs on
// d >= 32 feature vectors (BASELINE cfg4), sm_100a tcgen05, CTA pairs.
//
// The exponent of every pair, t_or = z_or - m_o (log2 units), is produced by
// kind::tf32 MMAs with split-precision compensation and the row / column
// constants folded into extra K columns:
//   A row o (output, in TMEM):  [Yh(d), Yl(d), 1, 1, 1, ch, cm, cl, 0..]
//   B row r (reduced, smem):    [Xh(d), Xl(d), Uh, Um, Ul, 1, 1, 1, 0..]
// with X = 2L x_r, U_r = (pot_r - |x_r|^2) L + log2 w_r, c_o = -|y_o|^2 L -
// m_o, every value split into TF32 hi/lo (3 parts for U and c).  Per 8-wide
// K slice the issuer runs Yh.Xh, Yl.Xh (same B data, two A offsets) and
// Yh.Xl, so the 3xTF32 product Yh.Xh + Yl.Xh + Yh.Xl + U + c reproduces the
// fp32 exponent to ~2^-21 while B carries each X value only twice
// (TF32 alone would miss the 1e-4 eps tolerance).
//
// CTA pairs (cta_group::2, M = 256): a cluster of two CTAs covers 256 output
// rows; each CTA keeps its 128 A rows in its own TMEM and streams only HALF
// of every B tile (64 of the 128 reduced rows) into its shared memory -- the
// leader's MMA reads both halves, so each SM ingests half the B bytes (the
// single-CTA version was bound by ~28 B/clk/SM of bulk-copy ingestion).
// Warp roles: warp 0 streams this CTA's B halves with 1-D bulk copies; in the
// leader, warp 1 issues tcgen05.mma.cta_group::2 from one thread into a
// double-buffered TMEM accumulator (commits multicast to both CTAs); in the
// peer, warp 1 relays "my half landed" to the leader's barrier; warps 2-5 of
// both CTAs read their 128 accumulator rows with tcgen05.ld and run the
// exp2 / sum epilogue on the MUFU pipe while the next tile is multiplied.
#pragma once

#include "sinkhorn.cuh"
#include "tcgen05.cuh"

namespace uot {

constexpr int TC_TILE = 128;        // outputs per CTA and reduced rows per B tile
constexpr int TC_HALF = 64;         // reduced rows per CTA per B tile
#ifndef UOT_TC_STAGE_K
#define UOT_TC_STAGE_K 16
#endif
constexpr int TC_STAGE_K = UOT_TC_STAGE_K;  // K elements per shared-memory stage
#ifndef UOT_TC_STAGES
#define UOT_TC_STAGES 24
#endif
constexpr int TC_STAGES = UOT_TC_STAGES;  // B-operand ring depth
constexpr int TC_THREADS = 192;
constexpr int TC_STAGE_BYTES = TC_HALF * TC_STAGE_K * 4;  // 4 KiB: one CTA's half stage

// Output-side point tile staged in shared memory for the A prologue: 128
// rows of d floats, row stride d + 4 (conflict-free float4 row reads).
__host__ __device__ __forceinline__ int tc_ystride(int d) { return d + 4; }
__host__ __device__ __forceinline__ size_t tc_smem_bytes(int d) {
  return (size_t)TC_STAGES * TC_STAGE_BYTES + sizeof(float) * 128 * (size_t)tc_ystride(d);
}

// K extent of a reduced-side record (B) and of an output-side row (A).
__host__ __device__ constexpr int tc_kp(int d) {
  return (2 * d + 6 + TC_STAGE_K - 1) / TC_STAGE_K * TC_STAGE_K;
}
__host__ __device__ constexpr int tc_ka(int d) { return 2 * d + 8; }

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(tc::tf32_rna(x)); }

// Index of element (row rl, column k) inside one 128-row record tile: two
// 64-row halves, each in the canonical K-major no-swizzle core-matrix layout
// ([k/4][row/8][row%8][k%4]; LBO = 1024 B between K groups, SBO = 128 B
// between 8-row groups), so a CTA's half of a stage is one contiguous copy.
__device__ __forceinline__ long tc_tile_index(int rl, int k, int KP) {
  return (long)(rl >> 6) * (TC_HALF * KP) + (long)(k >> 2) * (8 * 32) + ((rl >> 3) & 7) * 32 +
         (rl & 7) * 4 + (k & 3);
}

// One K-slice (8 columns of B) of a column tile: the MMAs it feeds.  Xh
// slices meet Yh and Yl, Xl slices meet Yh, the last slice meets the
// constants (3xTF32 split of 2L x.y + U + c).
__device__ __forceinline__ void tc_slice_mmas(int kb, int d, uint32_t dcol, uint32_t tbase,
                                              uint64_t bd, uint32_t idesc, bool& first) {
  if (kb < d) {
    tc::mma2_tf32_ts(dcol, tbase + kb, bd, idesc, first ? 0u : 1u);
    tc::mma2_tf32_ts(dcol, tbase + d + kb, bd, idesc, 1u);
    first = false;
  } else if (kb < 2 * d) {
    tc::mma2_tf32_ts(dcol, tbase + (kb - d), bd, idesc, first ? 0u : 1u);
    first = false;
  } else if (kb < 2 * d + 8) {
    tc::mma2_tf32_ts(dcol, tbase + 2 * d, bd, idesc, first ? 0u : 1u);
    first = false;
  }
}

// DT > 0: the feature dimension is a compile-time constant, so the MMA issue
// sequence of a column tile is fully unrolled and branch-free (a tight
// tcgen05.mma stream runs at its floor; a generic loop issue-bound).
// DT = 0: runtime d.  Launched with cluster dims (2, 1, 1) over row tiles.
template <int DT>
__global__ void __launch_bounds__(TC_THREADS, 1) sk_main_tc(MainArgs<float> A, int KP) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_b[TC_STAGES], empty_b[TC_STAGES], peer_b[TC_STAGES], dfull[2], dempty[2];
  __shared__ uint32_t tbase_s;
  const int b = blockIdx.z;
  if (A.done != nullptr && A.done[b]) return;  // uniform over the pair (same b)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const int split = blockIdx.y, S = gridDim.y;
  const int ntiles = (A.nred + TC_TILE - 1) / TC_TILE;
  const int t0 = (int)((long)ntiles * split / S), t1 = (int)((long)ntiles * (split + 1) / S);
  const int nst = DT > 0 ? tc_kp(DT) / TC_STAGE_K : KP / TC_STAGE_K;
  const int d = DT > 0 ? DT : A.g.d;

  if (warp == 1) tc::tmem_alloc2(&tbase_s, 512);
  if (tid == 0) {
    for (int i = 0; i < TC_STAGES; ++i) {
      tc::mbar_init(&full_b[i], 1);
      tc::mbar_init(&empty_b[i], 1);  // one multicast commit per use
      tc::mbar_init(&peer_b[i], 1);   // leader: the peer's half landed
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&dfull[i], 1);
      tc::mbar_init(&dempty[i], 8);  // leader: one arrive per epilogue warp of the pair
    }
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tbase_s;

  // Epilogue threads own one output row each (TMEM lane restriction: warp w
  // reaches lanes 32*(w%4) .. +31).
  const int lane_base = 32 * (warp & 3);
  const int row = lane_base + lane;
  const int o = blockIdx.x * TC_TILE + row;
  float m_o = 0.f;
  // Prologue: the CTA's 128 output points -> shared memory (all threads,
  // coalesced float4 loads), then each epilogue thread builds its A row
  // [Yh, Yl, 1, 1, 1, ch, cm, cl] (tf32 splits) and stores it into TMEM.
  float* ys = reinterpret_cast<float*>(smem + (size_t)TC_STAGES * TC_STAGE_BYTES);
  const int YS = tc_ystride(d);
  {
    const int row0 = blockIdx.x * TC_TILE;
    const int nrows = min(TC_TILE, A.nout - row0);
    const float4* src =
        reinterpret_cast<const float4*>(A.g.out_pts + b * A.g.out_pts_bstride + (long)row0 * d);
    const int q4 = d / 4;
    for (int idx = tid; idx < nrows * q4; idx += TC_THREADS) {
      const int r = idx / q4, c = idx - r * q4;
      *reinterpret_cast<float4*>(ys + r * YS + 4 * c) = src[idx];
    }
  }
  __syncthreads();
  if (warp >= 2) {
    const float* y = ys + row * YS;
    double s2 = 0.0;
    if (o < A.nout) {
      for (int k = 0; k < d; k += 4) {
        const float4 v = *reinterpret_cast<const float4*>(y + k);
        s2 = fma((double)v.x, (double)v.x, s2);
        s2 = fma((double)v.y, (double)v.y, s2);
        s2 = fma((double)v.z, (double)v.z, s2);
        s2 = fma((double)v.w, (double)v.w, s2);
      }
    }
    m_o = o < A.nout ? A.shift_in[(long)b * A.nout + o] : 0.f;
    const double c = -s2 * (double)A.g.L - (double)m_o;
    const float ch = tf32_hi((float)c);
    const double c1 = c - (double)ch;
    const float cm = tf32_hi((float)c1);
    const float cl = (float)(c1 - (double)cm);
    const uint32_t ta = tbase + ((uint32_t)lane_base << 16);
    // Yh at columns [0, d), Yl at [d, 2d): 8 columns per store
    for (int k0 = 0; k0 < d; k0 += 8) {
      float yv[8];
      if (o < A.nout) {
        const float4 u0 = *reinterpret_cast<const float4*>(y + k0);
        const float4 u1 = *reinterpret_cast<const float4*>(y + k0 + 4);
        yv[0] = u0.x, yv[1] = u0.y, yv[2] = u0.z, yv[3] = u0.w;
        yv[4] = u1.x, yv[5] = u1.y, yv[6] = u1.z, yv[7] = u1.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) yv[e] = 0.f;
      }
      uint32_t vh[8], vl[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float yh = tf32_hi(yv[e]);
        vh[e] = __float_as_uint(yh);
        vl[e] = __float_as_uint(yv[e] - yh);
      }
      tc::tmem_st8(ta + k0, vh);
      tc::tmem_st8(ta + d + k0, vl);
    }
    {
      const uint32_t vt[8] = {__float_as_uint(1.f), __float_as_uint(1.f), __float_as_uint(1.f),
                              __float_as_uint(ch),  __float_as_uint(cm),  __float_as_uint(cl),
                              0u,                   0u};
      tc::tmem_st8(ta + 2 * d, vt);
    }
    tc::wait_st();
  }
  // both CTAs' A rows and barriers ready before any MMA / remote arrive
  tc::fence_before();
  tc::cluster_sync_all();
  tc::fence_after();

  const float* recb = A.g.red_rec + b * A.g.red_bstride;
  if (warp == 0) {
    if (tc::elect_one()) {  // producer: this CTA's halves of the B stages
      int slot = 0;
      uint32_t phase = 0;
      for (int tile = t0; tile < t1; ++tile) {
        const float* src = recb + (long)tile * TC_TILE * KP + (long)rank * TC_HALF * KP;
        for (int st = 0; st < nst; ++st) {
          tc::mbar_wait(&empty_b[slot], phase ^ 1);
          tc::mbar_expect_tx(&full_b[slot], TC_STAGE_BYTES);
          tc::bulk_g2s(smem + slot * TC_STAGE_BYTES, src + (long)st * TC_HALF * TC_STAGE_K,
                       TC_STAGE_BYTES, &full_b[slot]);
          if (++slot == TC_STAGES) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      const int nstage = (t1 - t0) * nst;
      if (!leader) {
        // relay: my half of stage s landed -> the leader's peer barrier
        int slot = 0;
        uint32_t phase = 0;
        for (int s = 0; s < nstage; ++s) {
          tc::mbar_wait(&full_b[slot], phase);
          tc::mbar_arrive_remote_relaxed(tc::mapa(&peer_b[slot], 0));
          if (++slot == TC_STAGES) {
            slot = 0;
            phase ^= 1;
          }
        }
      } else {  // MMA issuer for the pair
        const uint32_t idesc = tc::idesc_tf32(2 * TC_TILE, TC_TILE);
        int slot = 0;
        uint32_t phase = 0;
        // descriptor of slot 0; other slots / slices add byte offset >> 4
        const uint64_t bd0 = tc::sdesc(smem, (TC_HALF / 8) * 128, 128);
        for (int i = 0; i < t1 - t0; ++i) {
          const int buf = i & 1;
          const uint32_t dph = (i >> 1) & 1;
          tc::mbar_wait(&dempty[buf], dph ^ 1);
          tc::fence_after();
          const uint32_t dcol = tbase + 256 + buf * TC_TILE;
          bool first = true;
          constexpr int NST = DT > 0 ? tc_kp(DT) / TC_STAGE_K : 1;
#pragma unroll
          for (int stu = 0; stu < (DT > 0 ? NST : 1); ++stu) {
            for (int str = 0; str < (DT > 0 ? 1 : nst); ++str) {
              const int st = DT > 0 ? stu : str;
              tc::mbar_wait(&full_b[slot], phase);
              tc::mbar_wait(&peer_b[slot], phase);
              tc::fence_after();
              const uint64_t bds = bd0 + (uint64_t)((slot * TC_STAGE_BYTES) >> 4);
#pragma unroll
              for (int ks = 0; ks < TC_STAGE_K / 8; ++ks) {
                const int kb = st * TC_STAGE_K + ks * 8;  // K offset of this slice in B
                tc_slice_mmas(kb, d, dcol, tbase,
                              bds + (uint64_t)((ks * 2 * (TC_HALF / 8) * 128) >> 4), idesc, first);
              }
              tc::mma2_commit_mc(&empty_b[slot], 3);
              if (++slot == TC_STAGES) {
                slot = 0;
                phase ^= 1;
              }
            }
          }
          tc::mma2_commit_mc(&dfull[buf], 3);
        }
      }
    }
    __syncwarp();
  } else {
    // Epilogue: exp2 + sum of each accumulator row, range-checked per tile.
    float acc = 0.f, corr = 0.f;
    const uint32_t tl = tbase + ((uint32_t)lane_base << 16);
    const uint32_t dempty_leader0 = tc::mapa(&dempty[0], 0);
    const uint32_t dempty_leader1 = tc::mapa(&dempty[1], 0);
    for (int i = 0; i < t1 - t0; ++i) {
      const int buf = i & 1;
      const uint32_t dph = (i >> 1) & 1;
      tc::mbar_wait(&dfull[buf], dph);
      tc::fence_after();
      const uint32_t dcol = tl + 256 + buf * TC_TILE;
      uint32_t v0[32], v1[32], v2[32], v3[32];
      tc::tmem_ld32(dcol, v0);
      tc::tmem_ld32(dcol + 32, v1);
      tc::tmem_ld32(dcol + 64, v2);
      tc::tmem_ld32(dcol + 96, v3);
      tc::wait_ld();
      // The accumulator is in registers (wait::ld completed): hand the buffer
      // back to the MMA issuer.  No TMEM read is outstanding, so a relaxed
      // arrive suffices (a release.cluster arrive per warp and tile costs
      // ~1.5x the kernel time).
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote_relaxed(buf ? dempty_leader1 : dempty_leader0);
      float s;
      {
        float sa = 0.f, sb = 0.f, sc = 0.f, sd = 0.f;
        if (__all_sync(0xffffffffu, corr == 0.f)) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            sa += Dom<float>::ex(__uint_as_float(v0[e]));
            sb += Dom<float>::ex(__uint_as_float(v1[e]));
            sc += Dom<float>::ex(__uint_as_float(v2[e]));
            sd += Dom<float>::ex(__uint_as_float(v3[e]));
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            sa += Dom<float>::ex(__uint_as_float(v0[e]) + corr);
            sb += Dom<float>::ex(__uint_as_float(v1[e]) + corr);
            sc += Dom<float>::ex(__uint_as_float(v2[e]) + corr);
            sd += Dom<float>::ex(__uint_as_float(v3[e]) + corr);
          }
        }
        s = (sa + sb) + (sc + sd);
      }
      float na = acc + s;
      if (!(na < 1.2676506e30f && na > 7.8886091e-31f)) {
        // Rare: the stale shift is off by > 2^100 -- rescale from this tile's max.
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          mx = fmaxf(mx, __uint_as_float(v0[e]) + corr);
          mx = fmaxf(mx, __uint_as_float(v1[e]) + corr);
          mx = fmaxf(mx, __uint_as_float(v2[e]) + corr);
          mx = fmaxf(mx, __uint_as_float(v3[e]) + corr);
        }
        float mn = mx;
        if (acc > 0.f) mn = fmaxf(mn, Dom<float>::lg(acc));
        if (mn > -INFINITY && mn < INFINITY) {
          if (acc > 0.f) acc *= Dom<float>::ex(-mn);
          corr -= mn;
        }
        s = 0.f;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          s += Dom<float>::ex(__uint_as_float(v0[e]) + corr);
          s += Dom<float>::ex(__uint_as_float(v1[e]) + corr);
          s += Dom<float>::ex(__uint_as_float(v2[e]) + corr);
          s += Dom<float>::ex(__uint_as_float(v3[e]) + corr);
        }
        na = acc + s;
      }
      acc = na;
    }
    if (o < A.nout) {
      const long idx = ((long)b * A.splits_total + A.split_base + split) * A.nout + o;
      A.part_m[idx] = m_o - corr;
      A.part_a[idx] = acc;
    }
  }
  tc::fence_before();
  tc::cluster_sync_all();  // both CTAs done with TMEM and remote barriers
  if (warp == 1) tc::tmem_free2(tbase, 512);
}

// Dead-row fill of a canonical record buffer: every row gets U = -1e30
// (exp2 -> 0) and the unit columns, so padded rows of the last tile never
// contribute; live rows are overwritten by the tails.
__global__ void tc_fill_dead(float* buf, long nrows_padded, int d, int KP) {
  const long total = nrows_padded * KP;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const long tile = idx / ((long)TC_TILE * KP);
    const long rem = idx % ((long)TC_TILE * KP);
    const long r2 = rem % ((long)TC_HALF * KP);  // within a 64-row half
    const int k = (int)(r2 / (8 * 32)) * 4 + (int)(r2 % 4);
    float v = 0.f;
    if (k == 2 * d) v = -1e30f;
    else if (k >= 2 * d + 3 && k < 2 * d + 6) v = 1.f;
    buf[tile * TC_TILE * KP + rem] = v;
  }
}

}  // namespace uot
