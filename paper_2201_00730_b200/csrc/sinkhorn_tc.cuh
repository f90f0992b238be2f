// sinkhorn_tc.cuh -- tensor-core half-step for squared-Euclidean costs on
// d >= 32 feature vectors (BASELINE cfg4), sm_100a tcgen05, CTA pairs.
//
// The exponent of every pair, t_or = z_or - m_o (log2 units), comes out of
// the tensor pipe complete:
//   2L x.y     by kind::f16 MMAs on fp16 hi/lo splits (3 products, fp32
//              accumulate): A row o = [Yh, Yl] of 8 y_o, B row r = [Xh, Xl]
//              of (2L / 8) x_r; per 16-wide K slice of Xh the issuer runs
//              Yh.Xh and Yl.Xh (same B data), per slice of Xl it runs Yh.Xl.
//              The power-of-two scale 8 balances the operands so the lo parts
//              stay clear of the fp16 subnormal range; the dropped Yl.Xl term
//              is ~2^-22 relative (|error| <~ 2^-22 2L in log2 units).
//   U_r + c_o  by one kind::tf32 MMA into the same accumulator:
//              A = [1, 1, 1, ch, cm, cl, 0, 0], B = [Uh, Um, Ul, 1, 1, 1, 0, 0]
//              (3-way tf32 splits: fp32 range and precision for
//              U_r = (pot_r - |x_r|^2) L + log2 w_r and c_o = -|y_o|^2 L - m_o).
// fp16 operands halve the MMA count of the former 3xTF32 split (12 + 1 per
// 256x128 tile at d = 64 instead of 25) and the B bytes per tile.
//
// CTA pairs (cta_group::2, M = 256): a cluster of two CTAs covers 256 output
// rows; each CTA keeps its 128 A rows in its own TMEM and streams only HALF
// of every B tile (64 of the 128 reduced rows) into its shared memory -- the
// leader's MMA reads both halves, so each SM ingests half the B bytes.
// Warp roles: warp 0 streams this CTA's B halves with 1-D bulk copies; in the
// leader, warp 1 issues tcgen05.mma.cta_group::2 from one thread into a
// double-buffered TMEM accumulator (commits multicast to both CTAs); in the
// peer, warp 1 relays "my half landed" to the leader's barrier; warps 2-5 of
// both CTAs read their 128 accumulator rows with tcgen05.ld and run the
// exp2 / sum epilogue on the MUFU pipe while the next tile is multiplied.
#pragma once

#include <cuda_fp16.h>

#include "sinkhorn.cuh"
#include "tcgen05.cuh"

namespace uot {

constexpr int TC_TILE = 128;        // outputs per CTA and reduced rows per B tile
constexpr int TC_HALF = 64;         // reduced rows per CTA per B tile
#ifndef UOT_TC_STAGES
#define UOT_TC_STAGES 24
#endif
constexpr int TC_STAGES = UOT_TC_STAGES;  // B-operand ring depth
// warps 0 (B producer), 1 (MMA issuer / relay), 2-5 and 6-9 (epilogue of
// output blocks 0 and 1: two warps per SM sub-partition keep the MUFU fed)
constexpr int TC_THREADS = 320;
constexpr int TC_NB = 2;  // output blocks of 128 rows per CTA
constexpr int TC_STAGE_BYTES = 4096;  // one CTA's half of a stage: 32 fp16 K columns
constexpr int TC_CBYTES = 2048;       // the constants' stage: 8 tf32 K columns
// A = S y', B = (2L / S) x' with the power-of-two S = tc_ascale(L) (sinkhorn.cu)

// Output-side points staged in shared memory for the A prologue: 256 rows
// of d floats, row stride d + 4 (conflict-free float4 row reads).
__host__ __device__ __forceinline__ int tc_ystride(int d) { return d + 4; }
__host__ __device__ __forceinline__ size_t tc_smem_bytes(int d) {
  return (size_t)TC_STAGES * TC_STAGE_BYTES +
         sizeof(float) * TC_NB * 128 * (size_t)tc_ystride(d);
}

// Record of a reduced row: an fp16 section [Xh(dp), Xl(dp), 0..] of KH
// halves (dp = d rounded up to 16, KH = 2 dp rounded up to 32) and a float
// section of 12 columns [Uh, Um, Ul, 1, 1, 1, 0, 0, |x|^2 (fp64), 0, 0].
__host__ __device__ constexpr int tc_dp(int d) { return (d + 15) / 16 * 16; }
__host__ __device__ constexpr int tc_kh(int d) { return (2 * tc_dp(d) + 31) / 32 * 32; }
// floats per record (size bookkeeping: KH halves + 12 floats)
__host__ __device__ constexpr int tc_kp(int d) { return tc_kh(d) / 2 + 12; }
// TMEM columns of an A row: dp packed fp16 pairs' worth (Yh, Yl) + 8 tf32
__host__ __device__ constexpr int tc_ka(int d) { return tc_dp(d) + 8; }

// A 128-row tile is two 64-row halves [X section | float section], each in
// the canonical K-major no-swizzle core-matrix layout (8 rows x 16 bytes per
// core matrix; LBO = 1024 B between K groups, SBO = 128 B between 8-row
// groups), so a CTA's half of a tile is one contiguous run of stages.
__host__ __device__ __forceinline__ long tc_half_floats(int d) { return (long)TC_HALF * tc_kp(d); }
// fp16 element (rl, k) of a tile, as an index in halves from the tile base
__device__ __forceinline__ long tc_xidx(int rl, int k, int d) {
  return (long)(rl >> 6) * 2 * tc_half_floats(d) + (long)(k >> 3) * 512 + ((rl >> 3) & 7) * 64 +
         (rl & 7) * 8 + (k & 7);
}
// float-section element (rl, c), c < 12, as an index in floats from the tile base
__device__ __forceinline__ long tc_cidx(int rl, int c, int d) {
  return (long)(rl >> 6) * tc_half_floats(d) + 32L * tc_kh(d) + (c >> 2) * 256 +
         ((rl >> 3) & 7) * 32 + (rl & 7) * 4 + (c & 3);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(tc::tf32_rna(x)); }

// Precomputed A row of an output point (tc_pack_out, once per solve: the
// points do not change across iterations): [Yh pairs (dp/2 words) | Yl pairs
// (dp/2 words) | |y'|^2 as an fp64 (2 words) | 2 pad words], 16-byte rows.
__host__ __device__ constexpr int tc_pack_words(int d) { return tc_dp(d) + 4; }

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);  // .x (low 16 bits) = a
  return *reinterpret_cast<const uint32_t*>(&h);
}

// The MMAs one 16-wide fp16 K slice of B feeds (kh = its K offset in halves):
// Xh slices meet Yh and Yl, Xl slices meet Yh -- and Yl too when `full` (the
// Yl Xl term is <= 2^-22 2L |x'||y'| in log2 units: dropped at moderate L,
// kept for small eps, see DirGeo::tc_full).
__device__ __forceinline__ void tc_slice_mmas(int kh, int dp, uint32_t dcol, uint32_t tbase,
                                              uint64_t bd, uint32_t idesc, bool& first,
                                              bool full) {
  if (kh < dp) {
    tc::mma2_f16_ts(dcol, tbase + (kh >> 1), bd, idesc, first ? 0u : 1u);
    tc::mma2_f16_ts(dcol, tbase + ((dp + kh) >> 1), bd, idesc, 1u);
    first = false;
  } else if (kh < 2 * dp) {
    tc::mma2_f16_ts(dcol, tbase + ((kh - dp) >> 1), bd, idesc, first ? 0u : 1u);
    if (full) tc::mma2_f16_ts(dcol, tbase + (kh >> 1), bd, idesc, 1u);
    first = false;
  }
}

// DT > 0: the feature dimension is a compile-time constant, so the MMA issue
// sequence of a column tile is fully unrolled and branch-free (a tight
// tcgen05.mma stream runs at its floor; a generic loop issue-bound).
// DT = 0: runtime d.  Launched with cluster dims (2, 1, 1); CTA c owns the
// output blocks 2c and 2c + 1 (128 rows each, A_0 / A_1 in its TMEM), so
// every B tile that lands feeds both blocks' MMAs (the pair's M = 256 rows
// of block j are CTA 2p's and CTA 2p+1's block j).
#ifdef UOT_TC_TIMING
// timing build only (scripts/tc_timeline.py): per-CTA %globaltimer stamps
// (start, A ready, first tile, last tile, end)
__device__ unsigned long long g_tc_stamps[1 << 16][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TC_STAMP(k) \
  if (threadIdx.x == 64) g_tc_stamps[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x][k] = gtimer()
#else
#define TC_STAMP(k)
#endif

template <int DT>
__global__ void __launch_bounds__(TC_THREADS, 1) sk_main_tc(MainArgs<float> A, int KP) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_b[TC_STAGES], empty_b[TC_STAGES], peer_b[TC_STAGES], dfull[TC_NB],
      dempty[TC_NB];
  __shared__ uint32_t tbase_s;
  const int b = blockIdx.z;
  if (A.done != nullptr && A.done[b]) return;  // uniform over the pair (same b)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const int split = blockIdx.y, S = gridDim.y;
  const int ntiles = (A.nred + TC_TILE - 1) / TC_TILE;
  const int t0 = (int)((long)ntiles * split / S), t1 = (int)((long)ntiles * (split + 1) / S);
  TC_STAMP(0);
  const int d = DT > 0 ? DT : A.g.d;
  const int dp = tc_dp(d);
  const int ka = tc_ka(d);        // TMEM columns of one A block
  const int nxs = tc_kh(d) / 32;  // fp16 stages per tile half; then one constants stage
  const int nst = nxs + 1;
  const bool full4 = A.g.tc_full != 0;
  (void)KP;
  // Precomputed A row of this epilogue thread (compile-time d): its loads are
  // issued before the TMEM allocation and barrier set-up, so their latency
  // overlaps the prologue.
  constexpr int PG = DT > 0 ? tc_dp(DT) / 16 : 1;  // 16-wide K groups
  uint4 pre[DT > 0 ? 4 * PG + 1 : 1];
  const bool packed = A.g.tc_pack != nullptr;
  const int row0 = blockIdx.x * (TC_NB * TC_TILE);
  const int blk = warp >= 2 ? (warp - 2) >> 2 : 0;
  const int lane_base = 32 * (warp & 3);
  const int row = lane_base + lane;
  const int o = row0 + blk * TC_TILE + row;
  // the stale shift of this output, also loaded up front
  const float m_pre = (warp >= 2 && o < A.nout) ? __ldg(A.shift_in + (long)b * A.nout + o) : 0.f;
  if constexpr (DT > 0) {
    if (packed && warp >= 2) {
      const uint4 zz = make_uint4(0u, 0u, 0u, 0u);
      const bool live = o < A.nout;
      const uint4* pr = reinterpret_cast<const uint4*>(A.g.tc_pack + b * A.g.tc_pack_bstride +
                                                       (long)(live ? o : 0) * tc_pack_words(DT));
#pragma unroll
      for (int i = 0; i < 4 * PG + 1; ++i) pre[i] = live ? __ldg(pr + i) : zz;
    }
  }

  if (warp == 1) tc::tmem_alloc2(&tbase_s, 512);
  if (tid == 0) {
    for (int i = 0; i < TC_STAGES; ++i) {
      tc::mbar_init(&full_b[i], 1);
      tc::mbar_init(&empty_b[i], 1);  // one multicast commit per use
      tc::mbar_init(&peer_b[i], 1);   // leader: the peer's half landed
    }
    for (int j = 0; j < TC_NB; ++j) {
      tc::mbar_init(&dfull[j], 1);
      tc::mbar_init(&dempty[j], 8);  // leader: one arrive per epilogue warp of the block, both CTAs
    }
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  TC_STAMP(5);
  const uint32_t tbase = tbase_s;

  // Epilogue threads own one output row of one block each (TMEM lane
  // restriction: warp w reaches lanes 32*(w%4) .. +31): blk, row, o above.
  float m_o = 0.f;
  // Prologue: the producer warp arrives at the cluster barrier and starts
  // streaming B stages at once (they depend on nothing else); the other
  // warps stage the CTA's 256 output points in shared memory (coalesced
  // float4 loads), then each epilogue thread builds its A row (fp16 splits of
  // 8 y + the tf32 constants) in its block's TMEM columns.
  float* ys = reinterpret_cast<float*>(smem + (size_t)TC_STAGES * TC_STAGE_BYTES);
  const int YS = tc_ystride(d);
  if (warp == 0) {
    tc::cluster_arrive();
  } else if (!packed) {
    const int nrows = max(0, min(TC_NB * TC_TILE, A.nout - row0));
    const float4* src =
        reinterpret_cast<const float4*>(A.g.out_pts + b * A.g.out_pts_bstride + (long)row0 * d);
    const float4* cen = reinterpret_cast<const float4*>(A.g.ctr + b * A.g.ctr_bstride);
    const int q4 = d / 4;
    for (int idx = tid - 32; idx < nrows * q4; idx += TC_THREADS - 32) {
      const int r = idx / q4, c = idx - r * q4;
      const float4 v = src[idx], cv = __ldg(cen + c);  // y' = y - centre (see init_tile)
      *reinterpret_cast<float4*>(ys + r * YS + 4 * c) =
          make_float4(v.x - cv.x, v.y - cv.y, v.z - cv.z, v.w - cv.w);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TC_THREADS - 32) : "memory");
    TC_STAMP(6);
  }
  if (warp >= 2 && packed) {
    // the precomputed row: 16-byte loads, no staging, no fp64 / fp16 work
    const uint32_t ta = tbase + ((uint32_t)lane_base << 16) + blk * ka;
    const int W = tc_pack_words(d);
    // (tcgen05.st is warp-collective: every lane stores, rows past nout zeros)
    const bool live = o < A.nout;
    const uint4* pr = reinterpret_cast<const uint4*>(A.g.tc_pack + b * A.g.tc_pack_bstride +
                                                     (long)(live ? o : 0) * W);
    const uint4 zz = make_uint4(0u, 0u, 0u, 0u);
    double s2 = 0.0;
    if constexpr (DT > 0) {  // rows preloaded at kernel entry
#pragma unroll
      for (int g = 0; g < PG; ++g) {
        const uint4 h0 = pre[2 * g], h1 = pre[2 * g + 1];
        const uint4 l0 = pre[2 * PG + 2 * g], l1 = pre[2 * PG + 2 * g + 1];
        const uint32_t vh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const uint32_t vl[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        tc::tmem_st8(ta + 8 * g, vh);
        tc::tmem_st8(ta + dp / 2 + 8 * g, vl);
      }
      if (live) s2 = __hiloint2double((int)pre[4 * PG].y, (int)pre[4 * PG].x);
    } else {
      for (int g = 0; g < dp / 16; ++g) {
        const uint4 h0 = live ? __ldg(pr + 2 * g) : zz, h1 = live ? __ldg(pr + 2 * g + 1) : zz;
        const uint4 l0 = live ? __ldg(pr + dp / 8 + 2 * g) : zz;
        const uint4 l1 = live ? __ldg(pr + dp / 8 + 2 * g + 1) : zz;
        const uint32_t vh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const uint32_t vl[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        tc::tmem_st8(ta + 8 * g, vh);
        tc::tmem_st8(ta + dp / 2 + 8 * g, vl);
      }
      if (live) {
        const uint4 q = __ldg(pr + dp / 4);
        s2 = __hiloint2double((int)q.y, (int)q.x);
      }
    }
    m_o = m_pre;
    const double c = -s2 * (double)A.g.L - (double)m_o;
    const float ch = tf32_hi((float)c);
    const double c1 = c - (double)ch;
    const float cm = tf32_hi((float)c1);
    const float cl = (float)(c1 - (double)cm);
    {
      const uint32_t vt[8] = {__float_as_uint(1.f), __float_as_uint(1.f), __float_as_uint(1.f),
                              __float_as_uint(ch),  __float_as_uint(cm),  __float_as_uint(cl),
                              0u,                   0u};
      tc::tmem_st8(ta + dp, vt);
    }
    tc::wait_st();
    TC_STAMP(7);
  } else if (warp >= 2) {
    const float* y = ys + (blk * TC_TILE + row) * YS;
    double s2 = 0.0;
    if (o < A.nout) {
      double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;  // four independent fp64 chains
      for (int k = 0; k < d; k += 4) {
        const float4 v = *reinterpret_cast<const float4*>(y + k);
        q0 = fma((double)v.x, (double)v.x, q0);
        q1 = fma((double)v.y, (double)v.y, q1);
        q2 = fma((double)v.z, (double)v.z, q2);
        q3 = fma((double)v.w, (double)v.w, q3);
      }
      s2 = (q0 + q1) + (q2 + q3);
    }
    m_o = o < A.nout ? A.shift_in[(long)b * A.nout + o] : 0.f;
    const double c = -s2 * (double)A.g.L - (double)m_o;
    const float ch = tf32_hi((float)c);
    const double c1 = c - (double)ch;
    const float cm = tf32_hi((float)c1);
    const float cl = (float)(c1 - (double)cm);
    const uint32_t ta = tbase + ((uint32_t)lane_base << 16) + blk * ka;
    // fp16 splits of 8 y: Yh at columns [0, dp/2), Yl at [dp/2, dp) (two
    // halves per column, the even K index in the low half); 16 K per store
    for (int k0 = 0; k0 < dp; k0 += 16) {
      float yv[16];
#pragma unroll
      for (int e = 0; e < 16; e += 4) {
        if (o < A.nout && k0 + e < d) {
          const float4 u = *reinterpret_cast<const float4*>(y + k0 + e);
          yv[e] = u.x, yv[e + 1] = u.y, yv[e + 2] = u.z, yv[e + 3] = u.w;
        } else {
          yv[e] = yv[e + 1] = yv[e + 2] = yv[e + 3] = 0.f;
        }
      }
      uint32_t vh[8], vl[8];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const float a0 = A.g.ascale * yv[2 * cc], a1 = A.g.ascale * yv[2 * cc + 1];
        const float h0 = __half2float(__float2half_rn(a0)), h1 = __half2float(__float2half_rn(a1));
        vh[cc] = pack_h2(h0, h1);
        vl[cc] = pack_h2(a0 - h0, a1 - h1);
      }
      tc::tmem_st8(ta + (k0 >> 1), vh);
      tc::tmem_st8(ta + ((dp + k0) >> 1), vl);
    }
    {
      const uint32_t vt[8] = {__float_as_uint(1.f), __float_as_uint(1.f), __float_as_uint(1.f),
                              __float_as_uint(ch),  __float_as_uint(cm),  __float_as_uint(cl),
                              0u,                   0u};
      tc::tmem_st8(ta + dp, vt);
    }
    tc::wait_st();
    TC_STAMP(7);
  }
  // both CTAs' A rows and barriers ready before any MMA / remote arrive
  if (warp != 0) {
    tc::fence_before();
    tc::cluster_arrive();
    tc::cluster_wait();
    tc::fence_after();
  }
  TC_STAMP(1);

  const float* recb = A.g.red_rec + b * A.g.red_bstride;
  if (warp == 0) {
    if (tc::elect_one()) {  // producer: this CTA's halves of the B stages
      int slot = 0;
      uint32_t phase = 0;
      const long hf = tc_half_floats(d);
      for (int tile = t0; tile < t1; ++tile) {
        const float* src = recb + (long)tile * 2 * hf + (long)rank * hf;
        for (int st = 0; st < nst; ++st) {
          const uint32_t bytes = st < nxs ? TC_STAGE_BYTES : TC_CBYTES;
          tc::mbar_wait(&empty_b[slot], phase ^ 1);
          tc::mbar_expect_tx(&full_b[slot], bytes);
          tc::bulk_g2s(smem + slot * TC_STAGE_BYTES, src + (long)st * (TC_STAGE_BYTES / 4), bytes,
                       &full_b[slot]);
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
        const uint32_t idesc = tc::idesc_f16(2 * TC_TILE, TC_TILE);
        const uint32_t idesc32 = tc::idesc_tf32(2 * TC_TILE, TC_TILE);
        // descriptor of slot 0; other slots / slices add byte offset >> 4
        const uint64_t bd0 = tc::sdesc(smem, (TC_HALF / 8) * 128, 128);
        constexpr int NXS = DT > 0 ? tc_kh(DT) / 32 : 1;
        int slot0 = 0;
        uint32_t phase0 = 0;
        for (int i = 0; i < t1 - t0; ++i) {
          const uint32_t ph = i & 1;
#pragma unroll 1
          for (int j = 0; j < TC_NB; ++j) {  // block 0, then block 1 on the same stages
            tc::mbar_wait(&dempty[j], ph ^ 1);
            tc::fence_after();
            const uint32_t dcol = tbase + 256 + j * TC_TILE;
            const uint32_t abase = tbase + j * ka;
            bool first = true;
            int slot = slot0;
            uint32_t phase = phase0;
#pragma unroll
            for (int stu = 0; stu < (DT > 0 ? NXS : 1); ++stu) {
              for (int str = 0; str < (DT > 0 ? 1 : nxs); ++str) {
                const int st = DT > 0 ? stu : str;
                if (j == 0) {
                  tc::mbar_wait(&full_b[slot], phase);
                  tc::mbar_wait(&peer_b[slot], phase);
                  tc::fence_after();
                }
                const uint64_t bds = bd0 + (uint64_t)((slot * TC_STAGE_BYTES) >> 4);
#pragma unroll
                for (int ks = 0; ks < 2; ++ks)  // two 16-wide K slices (2 KB each) per stage
                  tc_slice_mmas(st * 32 + ks * 16, dp, dcol, abase,
                                bds + (uint64_t)((ks * 2048) >> 4), idesc, first, full4);
                if (j == TC_NB - 1) tc::mma2_commit_mc(&empty_b[slot], 3);
                if (++slot == TC_STAGES) {
                  slot = 0;
                  phase ^= 1;
                }
              }
            }
            {  // the constants: U_r + c_o by one tf32 MMA into the same accumulator
              if (j == 0) {
                tc::mbar_wait(&full_b[slot], phase);
                tc::mbar_wait(&peer_b[slot], phase);
                tc::fence_after();
              }
              const uint64_t bds = bd0 + (uint64_t)((slot * TC_STAGE_BYTES) >> 4);
              tc::mma2_tf32_ts(dcol, abase + dp, bds, idesc32, first ? 0u : 1u);
              if (j == TC_NB - 1) tc::mma2_commit_mc(&empty_b[slot], 3);
              if (++slot == TC_STAGES) {
                slot = 0;
                phase ^= 1;
              }
            }
            tc::mma2_commit_mc(&dfull[j], 3);
            if (j == TC_NB - 1) {
              slot0 = slot;
              phase0 = phase;
            }
          }
        }
      }
    }
    __syncwarp();
  } else {
    // Epilogue: exp2 + sum of each accumulator row in two 64-column chunks,
    // range-checked per chunk; the block's accumulator is handed back as soon
    // as its second chunk is in registers.
    float acc = 0.f, corr = 0.f;
    const uint32_t tl = tbase + ((uint32_t)lane_base << 16) + 256 + blk * TC_TILE;
    const uint32_t dempty_leader = tc::mapa(&dempty[blk], 0);
    auto chunk = [&](const uint32_t (&v0)[32], const uint32_t (&v1)[32]) {
      float s;
      {
        float sa = 0.f, sb = 0.f, sc = 0.f, sd = 0.f;
        if (__all_sync(0xffffffffu, corr == 0.f)) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            sa += Dom<float>::ex(__uint_as_float(v0[e]));
            sb += Dom<float>::ex(__uint_as_float(v0[e + 16]));
            sc += Dom<float>::ex(__uint_as_float(v1[e]));
            sd += Dom<float>::ex(__uint_as_float(v1[e + 16]));
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            sa += Dom<float>::ex(__uint_as_float(v0[e]) + corr);
            sb += Dom<float>::ex(__uint_as_float(v0[e + 16]) + corr);
            sc += Dom<float>::ex(__uint_as_float(v1[e]) + corr);
            sd += Dom<float>::ex(__uint_as_float(v1[e + 16]) + corr);
          }
        }
        s = (sa + sb) + (sc + sd);
      }
      float na = acc + s;
      if (!(na < 1.2676506e30f && na > 7.8886091e-31f)) {
        // Rare: the stale shift is off by > 2^100 -- rescale from this chunk's max.
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          mx = fmaxf(mx, __uint_as_float(v0[e]) + corr);
          mx = fmaxf(mx, __uint_as_float(v1[e]) + corr);
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
        }
        na = acc + s;
      }
      acc = na;
    };
    for (int i = 0; i < t1 - t0; ++i) {
      tc::mbar_wait(&dfull[blk], i & 1);
      if (i == 0) TC_STAMP(2);
      tc::fence_after();
      uint32_t v0[32], v1[32], w0[32], w1[32];
      tc::tmem_ld32(tl, v0);
      tc::tmem_ld32(tl + 32, v1);
      tc::wait_ld();
      // the second half is read while the first half's exponentials run
      tc::tmem_ld32(tl + 64, w0);
      tc::tmem_ld32(tl + 96, w1);
      chunk(v0, v1);
      tc::wait_ld();
      // No TMEM read is outstanding, so a relaxed arrive suffices (a
      // release.cluster arrive per warp and tile costs ~1.5x the kernel time).
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote_relaxed(dempty_leader);
      chunk(w0, w1);
    }
    TC_STAMP(3);
    if (o < A.nout) {
      const long idx = ((long)b * A.splits_total + A.split_base + split) * A.nout + o;
      A.part_m[idx] = m_o - corr;
      A.part_a[idx] = acc;
    }
  }
  if (warp == 0) {
    __syncwarp();
    tc::cluster_wait();  // the producer warp's early arrive (phase 0)
  }
  tc::fence_before();
  tc::cluster_sync_all();  // both CTAs done with TMEM and remote barriers
  TC_STAMP(4);
  if (warp == 1) tc::tmem_free2(tbase, 512);
}

// A rows of the output side, once per solve: y' = y - centre, |y'|^2 by the
// prologue's four fp64 chains, and the fp16 hi/lo splits of ascale y' --
// bit for bit what sk_main_tc's unpacked prologue builds.
__global__ void tc_pack_out(uint32_t* out, const float* pts, const float* ctr, long ctr_bstride,
                            int batch, int nrows, int d, float ascale) {
  const int dp = tc_dp(d), W = tc_pack_words(d);
  const long total = (long)batch * nrows;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int b = (int)(i / nrows);
    const float* y = pts + i * d;
    const float* c = ctr + b * ctr_bstride;
    uint32_t* row = out + i * W;
    double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
    for (int k = 0; k < d; k += 4) {
      const float v0 = y[k] - c[k], v1 = y[k + 1] - c[k + 1], v2 = y[k + 2] - c[k + 2],
                  v3 = y[k + 3] - c[k + 3];
      q0 = fma((double)v0, (double)v0, q0);
      q1 = fma((double)v1, (double)v1, q1);
      q2 = fma((double)v2, (double)v2, q2);
      q3 = fma((double)v3, (double)v3, q3);
    }
    const double s2 = (q0 + q1) + (q2 + q3);
    for (int cc = 0; cc < dp / 2; ++cc) {
      const int k = 2 * cc;
      const float y0 = k < d ? y[k] - c[k] : 0.f, y1 = k + 1 < d ? y[k + 1] - c[k + 1] : 0.f;
      const float a0 = ascale * y0, a1 = ascale * y1;
      const float h0 = __half2float(__float2half_rn(a0)), h1 = __half2float(__float2half_rn(a1));
      row[cc] = pack_h2(h0, h1);
      row[dp / 2 + cc] = pack_h2(a0 - h0, a1 - h1);
    }
    row[dp] = (uint32_t)__double2loint(s2);
    row[dp + 1] = (uint32_t)__double2hiint(s2);
    row[dp + 2] = 0u;
    row[dp + 3] = 0u;
  }
}

// Dead-row fill of a record buffer: X = 0 and U = -1e30 (exp2 -> 0) with
// the unit columns, so padded rows of the last tile never contribute; live
// rows are overwritten by tc_init_static and the tails.
__global__ void tc_fill_dead(float* buf, long nrows_padded, int d, int) {
  const long hf = tc_half_floats(d);
  const long total = nrows_padded / TC_TILE * 2 * hf;  // floats
  const long xf = 32L * tc_kh(d);                       // floats of a half's X section
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const long r = idx % hf;  // within a 64-row half
    float v = 0.f;
    if (r >= xf) {
      const long cc = r - xf;
      const int c = (int)(cc / 256) * 4 + (int)(cc % 4);
      if (c == 0) v = -1e30f;
      else if (c >= 3 && c < 6) v = 1.f;
    }
    buf[idx] = v;
  }
}

}  // namespace uot
