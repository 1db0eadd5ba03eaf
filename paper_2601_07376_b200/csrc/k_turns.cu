// k_turns.cu — otk_turn_returns (turn-level credit; R31).
// PAPER.md:177 "rewards are associated with the corresponding action tokens"; SPEC.md:95 per-turn
// scores; SPEC.md:364 discounting as the extension. One thread per segment: it finds its trajectory
// (binary search over seg_offsets), its ordinal k among the trajectory's trainable ACTION segments,
// and evaluates the reward-to-go G_k = sum_{j>=k} gamma^(j-k) r_j by Horner's rule from the last
// score. Segments, turns and scores per trajectory are tens at most, so the work is a few hundred
// float64 operations per thread; one launch.
#include "otk_internal.h"

namespace otk {

constexpr int kTurnThreads = 256;

__global__ void __launch_bounds__(kTurnThreads) k_turn_returns(const TurnParams p) {
  const int32_t s = blockIdx.x * kTurnThreads + threadIdx.x;
  const otk_traj_batch& tb = p.b;
  const int B = tb.num_traj;
  if (s == 0 && tb.seg_offsets[B] != p.num_segments) set_error(p.err, OTK_ERR_BAD_TRAJECTORY);
  if (s >= p.num_segments) return;
  // trajectory b: seg_offsets[b] <= s < seg_offsets[b + 1] (largest b with seg_offsets[b] <= s)
  int lo = 0, hi = B - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tb.seg_offsets[mid] <= s) lo = mid; else hi = mid - 1;
  }
  const int b = lo;
  const int32_t s0 = tb.seg_offsets[b];
  double G = 0.0;
  int32_t grp = -1;
  if (s0 <= s && s < tb.seg_offsets[b + 1]) {
    const int ta = tb.traj_agent ? int(tb.traj_agent[b]) : int(p.train_agent);
    auto trainable = [&](int32_t k) {
      return tb.seg_source[k] == OTK_SRC_ACTION && (ta == OTK_ANY_AGENT || int(tb.seg_agent[k]) == ta);
    };
    if (trainable(s)) {
      int32_t k = 0;  // turn ordinal
      for (int32_t q = s0; q < s; ++q) k += trainable(q) ? 1 : 0;
      const int32_t t0 = p.turn_offsets[b], t1 = p.turn_offsets[b + 1];
      for (int32_t j = t1 - 1; j >= t0 + k; --j) G = p.turn_rewards[j] + p.gamma * G;
      grp = p.group_id[b];
      if (grp < 0) {
        set_error(p.err, OTK_ERR_GROUP_RANGE);
        G = 0.0;
      }
    }
  } else {
    set_error(p.err, OTK_ERR_BAD_TRAJECTORY);
  }
  p.seg_return[s] = G;
  p.seg_group[s] = grp;
}

cudaError_t launch_turn_returns(const TurnParams& p, cudaStream_t s) {
  const int grid = (p.num_segments + kTurnThreads - 1) / kTurnThreads;
  k_turn_returns<<<grid, kTurnThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace otk
