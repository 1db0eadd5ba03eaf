// k_lmhead.cu — NEXT-1, forward half: the LM-head GEMM fused with the vocab-wide
// log-softmax + gather + entropy of north_star (3), so the [N, V] logits never reach HBM. PAPER.md:188:
// the "forward inference (fwd)" pool computes the log-probs of every trajectory token under the current /
// old / reference policy; with the LM head fused, its input is the final hidden state h [N, d] and the
// head weight W [V, d] (logits z = s * h W^T).
//
// tcgen05 GEMM on CTA pairs (cta_group::2, a 2-CTA cluster on the two SMs of a TPC), persistent:
//   the pair computes a 256-row x 256-column tile per MMA (M = 256, N = 256, K = 16): each CTA stages its
//   own 128 rows of h and half (128 columns) of the W tile per 64-wide k-block (6 stages x 32 KB), and
//   holds its 128 rows x 256 fp32 accumulators in TMEM — twice (512 columns), so the epilogue of tile t
//   overlaps the MMAs of tile t + 1.
//   warp 0      TMA producer (both CTAs): 2-D tensor-map loads, 128-byte swizzle, completion counted on
//               the leader CTA's stage barrier;
//   warp 1      MMA issuer (leader CTA, one thread): tcgen05.mma.cta_group::2; tcgen05.commit multicast
//               frees the stage in both CTAs and, after the last k-block, signals both epilogues;
//   warps 2-5   epilogue (both CTAs): warp w reads TMEM lane quadrant w % 4 with tcgen05.ld.32x32b.x32 —
//               one thread per row, 256 logits per vocab tile — and folds them into the row's online
//               (reference m, sum 2^{y-m}, sum 2^{y-m}(y-m)) in the log2 domain (y = s log2(e) z) plus the
//               target logit; then arrives on the leader's accumulator-empty barrier (DSMEM for the peer).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

#include "otk_internal.h"
#include "otk_ptx.cuh"
#include "otk_umma.cuh"

namespace otk {

using namespace ptx;
using namespace umma;

constexpr int kLmRows = 256;   // rows per pair tile (128 per CTA)
constexpr int kLmCols = 256;   // vocab columns per tile (MMA N; 128 staged per CTA)
constexpr int kLmK = 64;       // hidden elements per k-block (128 bytes of bf16: one swizzle atom row)
constexpr int kLmStages = 6;
constexpr int kLmABytes = 128 * kLmK * 2;  // 16 KB: this CTA's rows
constexpr int kLmBBytes = 128 * kLmK * 2;  // 16 KB: this CTA's half of the columns
constexpr int kLmStageBytes = kLmABytes + kLmBBytes;
constexpr int kLmEpiWarps = 4;  // one per TMEM lane quadrant (8, two per quadrant over half tiles: no faster)
constexpr int kLmThreads = 32 * (2 + kLmEpiWarps);
constexpr int kLmSmemBytes = kLmStages * kLmStageBytes + 1024 /* 1 KB alignment slack */ + 256 /* barriers */;

struct LmParams {
  int64_t num_rows, vocab;
  int64_t vocab_start, vocab_total;  // this rank's columns of a vocab-sharded head (0, vocab unsharded)
  int d;                 // hidden size (multiple of 64)
  int n_rowtiles;        // ceil(num_rows / 256)
  int n_chunks;          // vocab chunks
  int n_coltiles;        // ceil(vocab / 256)
  const int32_t* targets;
  const uint8_t* row_mask;  // NULL = all rows
  float k2;              // logit_scale * log2(e)
  float4* partials;      // [n_chunks][num_rows]
  int* err;
  // optional: the logits rounded to bf16 (the row statistics are then taken over the rounded values, so the
  // backward's p = 2^(s log2(e) x - L2) from these logits sums to 1 — k_lmhead_bwd.cu), stored in 64 x 64 tiles:
  // [rows_pad / 64][cols_pad / 64][64][64] with rows_pad / cols_pad the 256-padded sizes, every tile element
  // written (rows >= num_rows and columns >= vocab hold 0: their h / W operands were zero-filled)
  uint32_t* logits_out;
  int64_t ld_out;        // tiles per tile row = cols_pad / 64
};

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N = 256, M = 256 (CTA pair).
constexpr uint32_t kLmIdesc = umma::idesc_bf16(kLmRows, kLmCols, false, false);

__device__ __forceinline__ int chunk_tile0(int c, int n_chunks, int n_coltiles) {
  return int((int64_t(c) * n_coltiles) / n_chunks);
}

// Work unit u -> (vocab chunk c, row tile rt), blocked: units run in row blocks of kLmRowBlock tiles; inside
// a block, chunk-major. The ~74 pairs running at the same time then share kLmRowBlock tiles of h (~29 MB at d = 3584,
// reused from L2 by every vocab tile of their units) and ~74 / kLmRowBlock chunks of W, so W is read from
// HBM once per row block instead of once per row tile (and h never thrashes L2).
#ifndef OTK_LM_ROWBLOCK
#define OTK_LM_ROWBLOCK 16
#endif
constexpr int kLmRowBlock = OTK_LM_ROWBLOCK;  // measured: 16 ~ 32 > 8 > 64 > 4 (scripts/perf_lmhead.py)
__device__ __forceinline__ void unit_coords(int u, int n_rowtiles, int n_chunks, int& c, int& rt) {
  const int R = min(kLmRowBlock, n_rowtiles);
  const int per_block = R * n_chunks;
  const int rb = u / per_block, w = u - rb * per_block;
  const int Rb = min(R, n_rowtiles - rb * R);  // the last block may hold fewer row tiles
  c = w / Rb;
  rt = rb * R + (w - c * Rb);
}
__global__ void __launch_bounds__(kLmThreads, 1)
    k_lmhead_fwd(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_w,
                 const LmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kLmStages * kLmStageBytes);
  uint64_t* empty = full + kLmStages;
  uint64_t* tfull = empty + kLmStages;  // [2] accumulator buffers
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = int(cluster_ctarank());
  const int pair = int(cluster_id_x()), npairs = int(nclusters_x());
  const int n_units = p.n_rowtiles * p.n_chunks;
  const int kblocks = p.d / kLmK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kLmEpiWarps);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_h);
    prefetch_tmap(&tm_w);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs)
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int c, rt;
        unit_coords(u, p.n_rowtiles, p.n_chunks, c, rt);
        const int t0 = chunk_tile0(c, p.n_chunks, p.n_coltiles), t1 = chunk_tile0(c + 1, p.n_chunks, p.n_coltiles);
        for (int t = t0; t < t1; ++t) {
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[s], ph ^ 1u);
            const uint32_t a = smem_u32(smem + s * kLmStageBytes);
            const uint32_t bar = smem_u32(&full[s]) & kPeerBitMask;
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kLmStageBytes);
            tma_load_2d_pair(a, &tm_h, bar, kb * kLmK, rt * kLmRows + rank * 128);
            tma_load_2d_pair(a + kLmABytes, &tm_w, bar, kb * kLmK, t * kLmCols + rank * 128);
            if (++s == kLmStages) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread)
    if (rank == 0 && lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      uint32_t it = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int c, rt;
        unit_coords(u, p.n_rowtiles, p.n_chunks, c, rt);
        const int t0 = chunk_tile0(c, p.n_chunks, p.n_coltiles), t1 = chunk_tile0(c + 1, p.n_chunks, p.n_coltiles);
        for (int t = t0; t < t1; ++t, ++it) {
          const uint32_t acc = it & 1u;
          mbar_wait(&tempty[acc], ((it >> 1) & 1u) ^ 1u);  // both epilogues drained this buffer
          tc_fence_after();
          const uint32_t d = tmem + acc * kLmCols;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + s * kLmStageBytes);
            const uint32_t b = a + kLmABytes;
#pragma unroll
            for (int k = 0; k < kLmK / 16; ++k)
              umma_pair_bf16<kLmIdesc>(d, sw128_kmajor_desc(a + k * 32), sw128_kmajor_desc(b + k * 32), (kb | k) != 0);
            umma_commit_pair(&empty[s]);  // frees the stage in both CTAs once these MMAs have read it
            if (++s == kLmStages) {
              s = 0;
              ph ^= 1u;
            }
          }
          umma_commit_pair(&tfull[acc]);  // accumulators complete in both CTAs
        }
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): one thread per row
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const uint32_t tlane = tmem + (uint32_t(32 * q) << 16);
    const uint32_t tempty_leader = smem_u32(&tempty[0]) & kPeerBitMask;
    const float k2 = p.k2;
    uint32_t it = 0;
    for (int u = pair; u < n_units; u += npairs) {
      int c, rt;
      unit_coords(u, p.n_rowtiles, p.n_chunks, c, rt);
      const int t0 = chunk_tile0(c, p.n_chunks, p.n_coltiles), t1 = chunk_tile0(c + 1, p.n_chunks, p.n_coltiles);
      const int64_t row = int64_t(rt) * kLmRows + rank * 128 + q * 32 + lane;
      const int64_t yglob = row < p.num_rows ? int64_t(p.targets[row]) : -1;
      if (c == 0 && p.vocab_start == 0 && row < p.num_rows && (!p.row_mask || p.row_mask[row]) &&
          (yglob < 0 || yglob >= p.vocab_total))
        set_error(p.err, OTK_ERR_TARGET_RANGE);  // such a row's logp is -inf (checked once, by shard 0)
      const int64_t yl = yglob - p.vocab_start;  // target column local to this shard
      const int ycol = (yl >= 0 && yl < p.vocab) ? int(yl) : -1;
      float m = -1e30f, s = 0.f, tt = 0.f, zy = -INFINITY;
      for (int t = t0; t < t1; ++t, ++it) {
        const uint32_t acc = it & 1u;
        mbar_wait(&tfull[acc], (it >> 1) & 1u);
        tc_fence_after();
        const int64_t col_t = int64_t(t) * kLmCols;
#pragma unroll 1
        for (int cc = 0; cc < kLmCols / 32; ++cc) {
          float v[32];
          tmem_ld32(tlane + acc * kLmCols + uint32_t(cc * 32), v);
          const int64_t col0 = col_t + cc * 32;
          const int64_t rem = p.vocab - col0;
          const int nvalid = rem < 32 ? int(rem) : 32;
          if (p.logits_out) {  // round to bf16 (RNE), store the row's 32 columns, and keep the rounded values
            uint32_t w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              w[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
              v[2 * j] = bf_lo(w[j]);
              v[2 * j + 1] = bf_hi(w[j]);
            }
            // tile (row / 64, col0 / 64), element offset (row % 64) * 64 + col0 % 64: 64 contiguous bytes
            uint4* dst = reinterpret_cast<uint4*>(p.logits_out) +
                         (((row >> 6) * p.ld_out + (col0 >> 6)) * 4096 + (row & 63) * 64 + (col0 & 63)) / 8;
#ifndef OTK_LM_XSTORE_PLAIN  // the x tiles (re-read only by the backward, from HBM) marked evict-first in L2, so
                             // they do not push the GEMM's h / W tiles out (d = 3584: 18.36-18.55 vs 18.71-18.79 ms)
            const uint64_t pol = policy_evict_first();
            stg256_hint(dst, make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]), pol);
            stg256_hint(dst + 2, make_uint4(w[8], w[9], w[10], w[11]), make_uint4(w[12], w[13], w[14], w[15]), pol);
#else
            stg256(dst, make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
            stg256(dst + 2, make_uint4(w[8], w[9], w[10], w[11]), make_uint4(w[12], w[13], w[14], w[15]));
#endif
          }
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = (j < nvalid) ? v[j] * k2 : -INFINITY;
            cm = fmaxf(cm, v[j]);
          }
          if (cm > m + 32.f) {  // raise the reference only when values would pass 2^32 (rare)
            const float r = ex2(m - cm);
            tt = r * fmaf(m - cm, s, tt);
            s *= r;
            m = cm;
          }
          const int yj = ycol - int(col0);
          if (yj >= 0 && yj < 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j == yj) zy = v[j];
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float dj = v[j] - m;
            const float e = ex2(dj);
            s += e;
            tt = fmaf(e, (j < nvalid) ? dj : 0.f, tt);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
      }
      if (row < p.num_rows)
        p.partials[int64_t(c) * p.num_rows + row] = make_float4(m, s, tt, zy == -INFINITY ? -INFINITY : zy - m);
    }
  }
  tc_fence_before();
  cluster_sync_all();  // every MMA consumed and every remote arrive delivered before TMEM is released
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// ---- host side -----------------------------------------------------------------------------------------
int lmhead_chunks(int64_t num_rows, int64_t vocab, int num_sms) {
  // vocab chunks: enough (row tile, chunk) units for whole waves of the persistent CTA pairs, chunks of
  // nearly equal tile counts (ties: fewer chunks)
  const int64_t rt = (num_rows + kLmRows - 1) / kLmRows;
  const int64_t nt = (vocab + kLmCols - 1) / kLmCols;
  const int64_t pairs = std::max(1, num_sms / 2);
  int best = 1;
  double best_eff = 0.0;
  for (int c = 1; c <= std::min<int64_t>(nt, 256); ++c) {
    const int64_t units = rt * c;
    const int64_t waves = (units + pairs - 1) / pairs;
    const double t = double(waves) * double((nt + c - 1) / c);  // the largest unit has ceil(nt / c) tiles
    const double eff = double(rt * nt) / (t * pairs);
    if (eff > best_eff + 1e-6) {
      best_eff = eff;
      best = c;
    }
  }
  return best;
}

cudaError_t launch_lmhead_fwd(const otk_ctx* ctx, int64_t num_rows, int64_t vocab, int d, const void* hidden,
                              const void* weight, const int32_t* targets, const uint8_t* row_mask, float logit_scale,
                              float4* partials, int n_chunks, cudaStream_t s, int64_t vocab_start,
                              int64_t vocab_total, void* logits_out, int64_t ld_out) {
  CUtensorMap th, tw;
  if (!make_map_2d(&th, hidden, num_rows, d, d, kLmK, 128) || !make_map_2d(&tw, weight, vocab, d, d, kLmK, 128))
    return cudaErrorInvalidValue;
  LmParams p;
  p.num_rows = num_rows;
  p.vocab = vocab;
  p.vocab_start = vocab_start;
  p.vocab_total = vocab_total > 0 ? vocab_total : vocab;
  p.d = d;
  p.n_rowtiles = int((num_rows + kLmRows - 1) / kLmRows);
  p.n_chunks = n_chunks;
  p.n_coltiles = int((vocab + kLmCols - 1) / kLmCols);
  p.targets = targets;
  p.row_mask = row_mask;
  p.err = ctx->d_err;
  p.k2 = logit_scale * 1.4426950408889634f;
  p.partials = partials;
  p.logits_out = reinterpret_cast<uint32_t*>(logits_out);
  p.ld_out = ld_out;
  // per launch (cheap, and correct for every device of the process)
  cudaError_t ea = cudaFuncSetAttribute(k_lmhead_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kLmSmemBytes);
  if (ea != cudaSuccess) return ea;
  const int units = p.n_rowtiles * p.n_chunks;
  const int pairs = std::max(1, std::min(units, ctx->num_sms / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(2 * pairs), 1, 1);
  cfg.blockDim = dim3(kLmThreads, 1, 1);
  cfg.dynamicSmemBytes = kLmSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_lmhead_fwd, th, tw, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace otk
