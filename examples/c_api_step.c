/* A whole single-GPU step through the C ABI alone (no Python): masks (1) from FSM-labelled segments, GRPO
 * advantages (2), the on-policy log-probs (3) and the fused PPO-clip + KL loss with its dlogits (4), on a
 * two-trajectory batch whose loss has a closed form. Build (tests/test_gpu_c_example.py does this):
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_step.c -o /tmp/c_api_step \
 *       -L paper_2601_07376_b200 -lotk -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2601_07376_b200
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "otk.h"

#define CK(x)                                                                        \
  do {                                                                               \
    otk_status s_ = (x);                                                             \
    if (s_ != OTK_OK) {                                                              \
      fprintf(stderr, "%s -> %s (%s)\n", #x, otk_status_string(s_), otk_last_error()); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)
#define CU(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) {                                                                     \
      fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                                 \
      return 1;                                                                                  \
    }                                                                                            \
  } while (0)

static void* dev_copy(const void* host, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 16) != cudaSuccess) return NULL;
  if (bytes) cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice);
  return d;
}

int main(void) {
  /* trajectory 0: CONTEXT 3 | ACTION 4 | OBSERVATION 2 | ACTION 3 (12 rows); trajectory 1: CONTEXT 2 | ACTION 5 |
     PAD 1 (8 rows). One group; returns 1 and 0 -> population std 0.5 -> A = +1, -1 (R2-R4). */
  const int B = 2, N = 20, V = 64;  /* 7 segments */
  const int64_t tok_offsets[3] = {0, 12, 20};
  const int32_t seg_offsets[3] = {0, 4, 7};
  const uint8_t seg_source[7] = {OTK_SRC_CONTEXT, OTK_SRC_ACTION, OTK_SRC_OBSERVATION, OTK_SRC_ACTION,
                                 OTK_SRC_CONTEXT, OTK_SRC_ACTION, OTK_SRC_PAD};
  const int16_t seg_agent[7] = {-1, 0, -1, 0, -1, 0, -1};
  const int32_t seg_len[7] = {3, 4, 2, 3, 2, 5, 1};
  const int32_t group_id[2] = {0, 0};
  const double returns[2] = {1.0, 0.0};
  float logits[20 * 64];
  int32_t targets[20];
  for (int j = 0; j < N; ++j) {
    for (int v = 0; v < V; ++v) logits[j * V + v] = 0.25f * (float)((j * 7 + v * 13) % 17) - 2.0f;
    targets[j] = (j * 5 + 3) % V;
  }
  otk_ctx* ctx = NULL;
  CK(otk_ctx_create(0, &ctx));
  otk_traj_batch tb;
  memset(&tb, 0, sizeof(tb));
  tb.num_traj = B;
  tb.num_rows = N;
  tb.tok_offsets = (const int64_t*)dev_copy(tok_offsets, sizeof(tok_offsets));
  tb.seg_offsets = (const int32_t*)dev_copy(seg_offsets, sizeof(seg_offsets));
  tb.seg_source = (const uint8_t*)dev_copy(seg_source, sizeof(seg_source));
  tb.seg_agent = (const int16_t*)dev_copy(seg_agent, sizeof(seg_agent));
  tb.seg_len = (const int32_t*)dev_copy(seg_len, sizeof(seg_len));
  uint8_t *loss_mask;
  int32_t *row_traj, *d_targets, *d_group;
  int64_t *traj_tokens, *n_loss;
  double *adv, *d_returns;
  float *d_logits, *dlogits, *logp, *entropy;
  otk_loss_stats* d_stats;
  CU(cudaMalloc((void**)&loss_mask, N));
  CU(cudaMalloc((void**)&row_traj, N * 4));
  CU(cudaMalloc((void**)&traj_tokens, B * 8));
  CU(cudaMalloc((void**)&n_loss, 8));
  CU(cudaMalloc((void**)&adv, B * 8));
  CU(cudaMalloc((void**)&dlogits, sizeof(logits)));
  CU(cudaMalloc((void**)&logp, N * 4));
  CU(cudaMalloc((void**)&entropy, N * 4));
  CU(cudaMalloc((void**)&d_stats, sizeof(otk_loss_stats)));
  d_logits = (float*)dev_copy(logits, sizeof(logits));
  d_targets = (int32_t*)dev_copy(targets, sizeof(targets));
  d_group = (int32_t*)dev_copy(group_id, sizeof(group_id));
  d_returns = (double*)dev_copy(returns, sizeof(returns));
  /* (1) masks, (2) advantages */
  CK(otk_build_masks(ctx, &tb, OTK_ANY_AGENT, loss_mask, NULL, row_traj, traj_tokens, NULL, n_loss, NULL, NULL, NULL));
  CK(otk_group_advantages(ctx, B, d_group, 1, d_returns, NULL, NULL, OTK_ADV_STD_NORM, 1e-8, adv, NULL, NULL, NULL,
                          NULL, NULL));
  /* (3) on-policy old / ref log-probs: the fwd pool's forward on the same logits */
  CK(otk_logprob_entropy_fwd(ctx, N, V, V, OTK_F32, d_logits, d_targets, NULL, 1.0f, logp, entropy, NULL, NULL));
  /* (4) PPO-clip + k3 KL, token mean, fused backward */
  otk_loss_cfg cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.clip_low = 0.2;
  cfg.clip_high = 0.2;
  cfg.kl_beta = 0.04;
  cfg.log_ratio_clamp = 20.0;
  cfg.logit_scale = 1.0;
  cfg.kl_type = OTK_KL_K3;
  cfg.zero_masked_rows = 1;
  cfg.reduction = OTK_TOKEN_MEAN;
  cfg.num_adv = B;
  CK(otk_policy_loss_fwd_bwd(ctx, N, V, V, OTK_F32, d_logits, d_targets, loss_mask, row_traj, adv, logp, logp, n_loss,
                             &cfg, dlogits, NULL, NULL, d_stats, NULL));
  CK(otk_ctx_check(ctx, NULL));
  otk_loss_stats st;
  int64_t nl = 0;
  double a[2];
  uint8_t m[20];
  float g[20 * 64];
  CU(cudaMemcpy(&st, d_stats, sizeof(st), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&nl, n_loss, 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(a, adv, sizeof(a), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(m, loss_mask, N, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(g, dlogits, sizeof(g), cudaMemcpyDeviceToHost));
  /* on policy (old = ref = logp): ratio 1 and KL 0, so loss = -sum_j m_j A_j / N_loss = -(7 * 1 + 5 * -1) / 12 */
  const double want = -(7.0 - 5.0) / 12.0;
  int ok = nl == 12 && fabs(a[0] - 1.0) < 1e-12 && fabs(a[1] + 1.0) < 1e-12 && fabs(st.loss - want) < 1e-6 &&
           st.n_tokens == 12.0 && st.n_clipped == 0.0;
  for (int j = 0; j < N; ++j) {  /* each trainable row of dlogits sums to 0; masked rows are exactly 0 */
    double rs = 0.0, ra = 0.0;
    for (int v = 0; v < V; ++v) {
      rs += g[j * V + v];
      ra += fabs(g[j * V + v]);
    }
    if (m[j] ? (fabs(rs) > 1e-6 || ra == 0.0) : ra != 0.0) ok = 0;
  }
  printf("c api step: n_loss=%lld adv=(%g, %g) loss=%.9f (closed form %.9f) -> %s\n", (long long)nl, a[0], a[1],
         st.loss, want, ok ? "ok" : "MISMATCH");
  otk_ctx_destroy(ctx);
  return ok ? 0 : 1;
}
