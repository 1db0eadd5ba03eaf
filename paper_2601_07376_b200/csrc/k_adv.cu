// k_adv.cu — otk_group_advantages (north_star (2)). SPEC.md:95: R_b = undiscounted sum of the
// per-turn scores; A_b = (R_b - mean_g) / (std_g if std_g > 1e-8 else 1).
// A single CTA: B (trajectories) and G (groups) are at most thousands, so the cost is one
// launch. All sums run sequentially in trajectory order in float64 (deterministic, and identical
// on every rank when a batch-sharded caller passes the all-gathered arrays).
#include <cmath>

#include "otk_internal.h"

namespace otk {

constexpr int kAdvThreads = 512;

__global__ void __launch_bounds__(kAdvThreads) k_group_advantages(const AdvParams p) {
  const int B = p.num_traj, G = p.num_groups;
  // 1) returns
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    double R;
    if (p.returns) {
      R = p.returns[b];
    } else {
      R = 0.0;
      for (int32_t k = p.turn_offsets[b]; k < p.turn_offsets[b + 1]; ++k) R += p.turn_rewards[k];
    }
    p.returns_out[b] = R;
  }
  __syncthreads();
  // 2) per-group mean and (population | sample) std; one thread per group, trajectory order
  extern __shared__ double s_stats[];  // [2*G] mean, std (G <= kMaxGroupsSmem) else global outputs
  double* s_mean = s_stats;
  double* s_std = s_stats + G;
  const volatile double* R = p.returns_out;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    int64_t n = 0;
    double sum = 0.0;
    for (int b = 0; b < B; ++b)
      if (p.group_id[b] == g) {
        sum += R[b];
        ++n;
      }
    const double mean = n > 0 ? sum / double(n) : 0.0;
    double sq = 0.0;
    for (int b = 0; b < B; ++b)
      if (p.group_id[b] == g) {
        const double d = R[b] - mean;
        sq += d * d;
      }
    const int64_t denom = (p.flags & OTK_ADV_UNBIASED) ? n - 1 : n;
    const double sd = denom > 0 ? sqrt(sq / double(denom)) : 0.0;
    s_mean[g] = mean;
    s_std[g] = sd;
    if (p.group_mean) p.group_mean[g] = mean;
    if (p.group_std) p.group_std[g] = sd;
    if (p.group_size) p.group_size[g] = int32_t(n);
  }
  __syncthreads();
  // 3) advantages
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int g = p.group_id[b];
    if (g < 0 && (p.flags & OTK_ADV_SKIP_UNGROUPED)) {  // turn-level credit: not a turn
      p.adv[b] = 0.0;
      continue;
    }
    if (g < 0 || g >= G) {
      set_error(p.err, OTK_ERR_GROUP_RANGE);
      p.adv[b] = 0.0;
      continue;
    }
    const double centred = R[b] - s_mean[g];
    if (p.flags & OTK_ADV_STD_NORM) {
      const double sd = s_std[g];
      p.adv[b] = centred / (sd > p.std_floor ? sd : 1.0);
    } else {
      p.adv[b] = centred;
    }
  }
}

cudaError_t launch_advantages(const AdvParams& p, cudaStream_t s) {
  const size_t smem = size_t(2) * p.num_groups * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_group_advantages, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  k_group_advantages<<<1, kAdvThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace otk
