// k_masks.cu — otk_build_masks (north_star (1); PAPER.md:167-174 token masking per FSM state,
// PAPER.md:192 per-agent independence). One CTA per trajectory: a block scan over the segment
// lengths gives each segment's first row; the CTA then writes the per-row labels with coalesced
// byte stores, finding each row's segment by binary search in shared memory. Integer work only,
// bit-exact. The last CTA to finish (ticket) sums the per-trajectory counts in index order into
// n_loss (no atomics on the result, deterministic).
#include "otk_internal.h"

namespace otk {

constexpr int kMaskThreads = 256;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* s_warp, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < kMaskThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += y;
    }
    if (lane < kMaskThreads / 32) s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int64_t warp_excl = warp > 0 ? s_warp[warp - 1] : 0;
  *total = s_warp[kMaskThreads / 32 - 1];
  return warp_excl + x - v;
}

__global__ void __launch_bounds__(kMaskThreads) k_build_masks(const MaskParams p) {
  __shared__ int64_t s_start[kMaskThreads];
  __shared__ uint8_t s_flag[kMaskThreads];
  __shared__ int64_t s_warp[kMaskThreads / 32];
  __shared__ unsigned long long s_cnt[5];  // loss, CONTEXT, ACTION, OBSERVATION, PAD
  __shared__ int s_bad;
  __shared__ int s_last;

  const int b = blockIdx.x;
  const otk_traj_batch& tb = p.b;
  const int tid = threadIdx.x;
  const int64_t N = tb.num_rows;
  const int64_t r0 = tb.tok_offsets[b], r1 = tb.tok_offsets[b + 1];
  const int32_t s0 = tb.seg_offsets[b], s1 = tb.seg_offsets[b + 1];
  const int ta = tb.traj_agent ? int(tb.traj_agent[b]) : int(p.train_agent);
  if (tid == 0) {
    int bad = 0;
    if (r0 < 0 || r1 < r0 || r1 > N || s1 < s0) bad = OTK_ERR_BAD_TRAJECTORY;
    if (!bad && tb.terminated && !tb.terminated[b]) bad = OTK_ERR_UNTERMINATED;
    s_bad = bad;
    for (int k = 0; k < 5; ++k) s_cnt[k] = 0ull;
  }
  __syncthreads();

  int64_t running = r0;
  if (!s_bad) {
    for (int32_t base = s0; base < s1; base += kMaskThreads) {
      const int32_t k = base + tid;
      int64_t L = 0;
      uint8_t flag = 0;
      if (k < s1) {
        L = tb.seg_len[k];
        const int src = tb.seg_source[k];
        if (L <= 0 || src > OTK_SRC_PAD) {
          atomicCAS(&s_bad, 0, int(OTK_ERR_BAD_TRAJECTORY));
          L = 0;
        } else {
          // PAPER.md:171 only GENERATING (ACTION) rows are trainable; PAPER.md:192 per-agent policies
          const bool trainable = src == OTK_SRC_ACTION && (ta == OTK_ANY_AGENT || int(tb.seg_agent[k]) == ta);
          // DESIGN.md R13: response = not the leading CONTEXT (prompt) segment, not PAD
          const bool responding = !(k == s0 && src == OTK_SRC_CONTEXT) && src != OTK_SRC_PAD;
          flag = uint8_t(trainable) | uint8_t(responding) << 1;
          atomicAdd(&s_cnt[1 + src], (unsigned long long)L);
          if (trainable) atomicAdd(&s_cnt[0], (unsigned long long)L);
        }
      }
      int64_t total;
      const int64_t excl = block_excl_scan(L, s_warp, &total);
      s_start[tid] = running + excl;
      s_flag[tid] = flag;
      __syncthreads();
      const int nseg = min(kMaskThreads, s1 - base);
      const int64_t tile_end = min(running + total, r1);
      if (!s_bad) {
        for (int64_t row = running + tid; row < tile_end; row += kMaskThreads) {
          int lo = 0, hi = nseg - 1;  // last segment whose start <= row
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_start[mid] <= row) lo = mid; else hi = mid - 1;
          }
          const uint8_t f = s_flag[lo];
          p.loss_mask[row] = f & 1u;
          if (p.response_mask) p.response_mask[row] = (f >> 1) & 1u;
          p.row_traj[row] = b;
          if (p.row_seg) p.row_seg[row] = base + lo;
        }
      }
      running += total;
      __syncthreads();
    }
    if (tid == 0 && !s_bad && running != r1) s_bad = OTK_ERR_BAD_TRAJECTORY;  // SPEC.md:91 partition
  }
  __syncthreads();

  if (s_bad) {
    // keep kernels downstream memory-safe: the trajectory's rows become loss-masked
    if (tid == 0) set_error(p.err, s_bad);
    if (r0 >= 0 && r0 <= N) {
      const int64_t e = min(max(r1, r0), N);
      for (int64_t row = r0 + tid; row < e; row += kMaskThreads) {
        p.loss_mask[row] = 0;
        if (p.response_mask) p.response_mask[row] = 0;
        p.row_traj[row] = b;
        if (p.row_seg) p.row_seg[row] = -1;
      }
    }
  }
  if (tid == 0) {
    p.traj_loss_tokens[b] = s_bad ? 0 : int64_t(s_cnt[0]);
    if (p.traj_source_counts)
      for (int k = 0; k < 4; ++k) p.traj_source_counts[int64_t(b) * 4 + k] = s_bad ? 0 : int64_t(s_cnt[1 + k]);
    __threadfence();
    s_last = atomicAdd(p.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    // last CTA: n_loss = sum of traj_loss_tokens in index order (warp-parallel, exact integers)
    __threadfence();
    int64_t acc = 0, act = 0;
    for (int i = tid; i < tb.num_traj; i += kMaskThreads) {
      const int64_t t = ((volatile int64_t*)p.traj_loss_tokens)[i];
      acc += t;
      act += t > 0 ? 1 : 0;
    }
    int64_t total, nact;
    (void)block_excl_scan(acc, s_warp, &total);
    __syncthreads();
    (void)block_excl_scan(act, s_warp, &nact);
    if (tid == 0) {
      *p.n_loss = total;
      if (p.n_active) *p.n_active = nact;
      if (tb.tok_offsets[0] != 0 || tb.tok_offsets[tb.num_traj] != N) set_error(p.err, OTK_ERR_BAD_TRAJECTORY);
      *p.ticket = 0u;
    }
  }
}

cudaError_t launch_masks(const MaskParams& p, cudaStream_t s) {
  k_build_masks<<<p.b.num_traj, kMaskThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace otk
