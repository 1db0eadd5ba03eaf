// k_lmhead.cu — NEXT-1, forward half: the LM-head GEMM fused with the vocab-wide
// log-softmax + gather + entropy of north_star (3), so the [N, V] logits never reach HBM. PAPER.md:188:
// the "forward inference (fwd)" pool computes the log-probs of every trajectory token under the current /
// old / reference policy; with the LM head fused, its input is the final hidden state h [N, d] and the
// head weight W [V, d] (logits z = s * h W^T).
//
// tcgen05 GEMM, one CTA per SM (persistent), warp-specialised:
//   warp 0      TMA producer: 2-D tensor-map loads (128-byte swizzle) of a 256 x 64 tile of h and a
//               256 x 64 tile of W per stage (3 stages x 64 KB);
//   warp 1      MMA issuer: per 64-wide k-block four K=16 steps of two tcgen05.mma (M = 128 each, the two
//               halves of the 256-row tile, N = 256) into TMEM (2 x 256 fp32 columns = all 512);
//               tcgen05.commit frees the smem stage and, after the last k-block, signals the epilogue;
//   warps 2-9   epilogue: warp w reads TMEM lane quadrant w % 4 of accumulator (w - 2) / 4 with
//               tcgen05.ld.32x32b.x32 — one thread per row, 256 logits per vocab tile — and folds them into
//               the row's online (reference m, sum 2^{y-m}, sum 2^{y-m}(y-m)) in the log2 domain
//               (y = s log2(e) z) plus the target logit.
// A work unit is (256-row tile, vocab chunk); each unit writes per-row partials (m, s, t, y_target - m or
// -inf) of its chunk, and k_combine (the vocab-shard combine) turns the chunks into logp / entropy / lse.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

#include "otk_internal.h"
#include "otk_ptx.cuh"

namespace otk {

using namespace ptx;

constexpr int kLmRows = 256;   // rows per tile (two M = 128 MMAs)
constexpr int kLmCols = 256;   // vocab columns per tile (MMA N)
constexpr int kLmK = 64;       // hidden elements per k-block (128 bytes of bf16: one swizzle atom row)
constexpr int kLmStages = 3;
constexpr int kLmABytes = kLmRows * kLmK * 2;  // 32 KB
constexpr int kLmBBytes = kLmCols * kLmK * 2;  // 32 KB
constexpr int kLmStageBytes = kLmABytes + kLmBBytes;
constexpr int kLmEpiWarps = 8;
constexpr int kLmThreads = 32 * (2 + kLmEpiWarps);
constexpr int kLmSmemBytes = kLmStages * kLmStageBytes + 1024 /* 1 KB alignment slack */ + 256 /* barriers */;

struct LmParams {
  int64_t num_rows, vocab;
  int d;                 // hidden size (multiple of 64)
  int n_rowtiles;        // ceil(num_rows / 256)
  int n_chunks;          // vocab chunks per row tile
  int n_coltiles;        // ceil(vocab / 256)
  const int32_t* targets;
  float k2;              // logit_scale * log2(e)
  float4* partials;      // [n_chunks][num_rows]
};

// ---- PTX wrappers specific to the tensor-core path -------------------------------------------------
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
// K-major operand, 128-byte swizzle: rows of 128 B, 8-row atoms 1024 B apart (SBO), LBO unused (1),
// descriptor version 1 (sm_100), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N = 256, M = 128.
constexpr uint32_t kLmIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kLmCols >> 3) << 17) |
                              (uint32_t(128 >> 4) << 24);
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kLmIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ int chunk_tile0(int c, int n_chunks, int n_coltiles) {
  return int((int64_t(c) * n_coltiles) / n_chunks);
}

__global__ void __launch_bounds__(kLmThreads, 1)
    k_lmhead_fwd(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_w,
                 const LmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kLmStages * kLmStageBytes);
  uint64_t* empty = full + kLmStages;
  uint64_t* tfull = empty + kLmStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_units = p.n_rowtiles * p.n_chunks;
  const int kblocks = p.d / kLmK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kLmEpiWarps);
    fence_mbar_init();
    prefetch_tmap(&tm_h);
    prefetch_tmap(&tm_w);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int rt = u / p.n_chunks, c = u % p.n_chunks;
        const int t0 = chunk_tile0(c, p.n_chunks, p.n_coltiles), t1 = chunk_tile0(c + 1, p.n_chunks, p.n_coltiles);
        for (int t = t0; t < t1; ++t) {
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[s], ph ^ 1u);
            const uint32_t a = smem_u32(smem + s * kLmStageBytes);
            mbar_arrive_expect_tx(&full[s], kLmStageBytes);
            tma_load_2d(a, &tm_h, smem_u32(&full[s]), kb * kLmK, rt * kLmRows);
            tma_load_2d(a + kLmABytes, &tm_w, smem_u32(&full[s]), kb * kLmK, t * kLmCols);
            if (++s == kLmStages) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      uint32_t it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int c = u % p.n_chunks;
        const int t0 = chunk_tile0(c, p.n_chunks, p.n_coltiles), t1 = chunk_tile0(c + 1, p.n_chunks, p.n_coltiles);
        for (int t = t0; t < t1; ++t, ++it) {
          mbar_wait(tempty, (it & 1u) ^ 1u);  // the epilogue has drained the accumulators
          tc_fence_after();
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + s * kLmStageBytes);
            const uint32_t b = a + kLmABytes;
#pragma unroll
            for (int k = 0; k < kLmK / 16; ++k) {
              const uint64_t bd = sw128_desc(b + k * 32);
              umma_bf16(tmem, sw128_desc(a + k * 32), bd, (kb | k) != 0);
              umma_bf16(tmem + kLmCols, sw128_desc(a + kLmABytes / 2 + k * 32), bd, (kb | k) != 0);
            }
            umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
            if (++s == kLmStages) {
              s = 0;
              ph ^= 1u;
            }
          }
          umma_commit(tfull);  // accumulators complete
        }
      }
    }
  } else {
    // ---------------- epilogue: one thread per row
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;  // accumulator (row half of the tile)
    const uint32_t tbase = tmem + (uint32_t(32 * q) << 16) + uint32_t(half * kLmCols);
    const float k2 = p.k2;
    uint32_t it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int rt = u / p.n_chunks, c = u % p.n_chunks;
      const int t0 = chunk_tile0(c, p.n_chunks, p.n_coltiles), t1 = chunk_tile0(c + 1, p.n_chunks, p.n_coltiles);
      const int64_t row = int64_t(rt) * kLmRows + half * 128 + q * 32 + lane;
      const int ycol = row < p.num_rows ? p.targets[row] : -1;
      float m = -1e30f, s = 0.f, tt = 0.f, zy = -INFINITY;
      for (int t = t0; t < t1; ++t, ++it) {
        mbar_wait(tfull, it & 1u);
        tc_fence_after();
        const int64_t col_t = int64_t(t) * kLmCols;
#pragma unroll 1
        for (int cc = 0; cc < kLmCols / 32; ++cc) {
          float v[32];
          tmem_ld32(tbase + uint32_t(cc * 32), v);
          const int64_t col0 = col_t + cc * 32;
          const int64_t rem = p.vocab - col0;
          const int nvalid = rem < 32 ? int(rem) : 32;
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
        if (lane == 0) mbar_arrive(tempty);
      }
      if (row < p.num_rows)
        p.partials[int64_t(c) * p.num_rows + row] = make_float4(m, s, tt, zy == -INFINITY ? -INFINITY : zy - m);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---- host side -----------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

bool make_map(CUtensorMap* map, const void* base, int64_t rows, int d, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(d) * 2};
  cuuint32_t box[2] = {cuuint32_t(kLmK), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

int lmhead_chunks(int64_t num_rows, int64_t vocab, int num_sms) {
  // vocab chunks per row tile: enough units for whole waves of the persistent grid (ties: fewer chunks)
  const int64_t rt = (num_rows + kLmRows - 1) / kLmRows;
  const int64_t nt = (vocab + kLmCols - 1) / kLmCols;
  int best = 1;
  double best_eff = 0.0;
  for (int c = 1; c <= std::min<int64_t>(nt, 64); ++c) {
    const int64_t units = rt * c;
    const int64_t waves = (units + num_sms - 1) / num_sms;
    // the largest unit has ceil(nt / c) tiles: time ~ waves * ceil(nt/c); work = rt * nt tiles
    const double t = double(waves) * double((nt + c - 1) / c);
    const double eff = double(rt * nt) / (t * num_sms);
    if (eff > best_eff + 1e-6) {
      best_eff = eff;
      best = c;
    }
  }
  return best;
}

cudaError_t launch_lmhead_fwd(const otk_ctx* ctx, int64_t num_rows, int64_t vocab, int d, const void* hidden,
                              const void* weight, const int32_t* targets, float logit_scale, float4* partials,
                              int n_chunks, cudaStream_t s) {
  CUtensorMap th, tw;
  if (!make_map(&th, hidden, num_rows, d, kLmRows) || !make_map(&tw, weight, vocab, d, kLmCols))
    return cudaErrorInvalidValue;
  LmParams p;
  p.num_rows = num_rows;
  p.vocab = vocab;
  p.d = d;
  p.n_rowtiles = int((num_rows + kLmRows - 1) / kLmRows);
  p.n_chunks = n_chunks;
  p.n_coltiles = int((vocab + kLmCols - 1) / kLmCols);
  p.targets = targets;
  p.k2 = logit_scale * 1.4426950408889634f;
  p.partials = partials;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_lmhead_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kLmSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int units = p.n_rowtiles * p.n_chunks;
  const int grid = std::min(units, ctx->num_sms);
  k_lmhead_fwd<<<grid, kLmThreads, kLmSmemBytes, s>>>(th, tw, p);
  return cudaGetLastError();
}

}  // namespace otk
