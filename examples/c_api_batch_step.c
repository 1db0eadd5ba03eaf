/* A batch-sharded step through the C ABI alone (no Python, no torch.distributed): P processes, one GPU each
 * (rank r on device r % #GPUs), join one NCCL communicator owned by their otk contexts and run the three exchanges
 * of SURVEY.md §8(e) BATCH around the local steps — global token count, group statistics over the union of the
 * shards, loss statistics. The global batch is c_api_step.c's two trajectories (one group straddling the ranks
 * when P = 2), so the loss has the same closed form on every P. Usage: c_api_batch_step [P] (default 1; P <= 2).
 * Build (tests/test_c_example.py does this):
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_batch_step.c -o /tmp/c_api_batch_step \
 *       -L paper_2601_07376_b200 -lotk -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2601_07376_b200
 */
#define _GNU_SOURCE
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/wait.h>
#include <unistd.h>

#include "otk.h"

#define CK(x)                                                                                         \
  do {                                                                                                \
    otk_status s_ = (x);                                                                              \
    if (s_ != OTK_OK) {                                                                               \
      fprintf(stderr, "rank %d: %s -> %s (%s)\n", rank, #x, otk_status_string(s_), otk_last_error()); \
      return 1;                                                                                       \
    }                                                                                                 \
  } while (0)
#define CU(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "rank %d: %s -> %s\n", rank, #x, cudaGetErrorString(e_));           \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

static void* dev_copy(const void* host, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 16) != cudaSuccess) return NULL;
  if (bytes) cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice);
  return d;
}

/* the global batch (c_api_step.c): trajectory 0 = CONTEXT 3 | ACTION 4 | OBSERVATION 2 | ACTION 3,
 * trajectory 1 = CONTEXT 2 | ACTION 5 | PAD 1; one group, returns 1 and 0 -> A = +1, -1 */
static const int V = 64;
static const int64_t g_tok[3] = {0, 12, 20};
static const int32_t g_seg[3] = {0, 4, 7};
static const uint8_t g_src[7] = {OTK_SRC_CONTEXT, OTK_SRC_ACTION, OTK_SRC_OBSERVATION, OTK_SRC_ACTION,
                                 OTK_SRC_CONTEXT, OTK_SRC_ACTION, OTK_SRC_PAD};
static const int16_t g_agent[7] = {-1, 0, -1, 0, -1, 0, -1};
static const int32_t g_len[7] = {3, 4, 2, 3, 2, 5, 1};
static const double g_returns[2] = {1.0, 0.0};

static float logit_of(int j, int v) { return 0.25f * (float)((j * 7 + v * 13) % 17) - 2.0f; }

static int run_rank(int rank, int P, const unsigned char* uid) {
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  otk_ctx* ctx = NULL;
  CK(otk_ctx_create(rank % ndev, &ctx));
  CK(otk_comm_init(ctx, uid, P, rank));
  /* this rank's trajectories: P = 1 -> both; P = 2 -> trajectory `rank` */
  const int b0 = P == 1 ? 0 : rank, b1 = P == 1 ? 2 : rank + 1, B = b1 - b0;
  int32_t counts[2] = {P == 1 ? 2 : 1, 1};
  const int64_t r0 = g_tok[b0], N = g_tok[b1] - r0;
  const int s0 = g_seg[b0], S = g_seg[b1] - s0;
  int64_t tok[3];
  int32_t seg[3];
  for (int b = 0; b <= B; ++b) {
    tok[b] = g_tok[b0 + b] - r0;
    seg[b] = g_seg[b0 + b] - s0;
  }
  float* logits = (float*)malloc(sizeof(float) * N * V);
  int32_t* targets = (int32_t*)malloc(sizeof(int32_t) * N);
  for (int64_t j = 0; j < N; ++j) {
    for (int v = 0; v < V; ++v) logits[j * V + v] = logit_of((int)(r0 + j), v);
    targets[j] = (int32_t)(((r0 + j) * 5 + 3) % V);
  }
  otk_traj_batch tb;
  memset(&tb, 0, sizeof(tb));
  tb.num_traj = B;
  tb.num_rows = N;
  tb.tok_offsets = (const int64_t*)dev_copy(tok, sizeof(int64_t) * (B + 1));
  tb.seg_offsets = (const int32_t*)dev_copy(seg, sizeof(int32_t) * (B + 1));
  tb.seg_source = (const uint8_t*)dev_copy(g_src + s0, S);
  tb.seg_agent = (const int16_t*)dev_copy(g_agent + s0, sizeof(int16_t) * S);
  tb.seg_len = (const int32_t*)dev_copy(g_len + s0, sizeof(int32_t) * S);
  const int32_t gid_local[2] = {0, 0};
  uint8_t* loss_mask;
  int32_t *row_traj, *gid_all;
  int64_t *traj_tokens, *n_loss;
  double *adv_all, *ret_all;
  float *dlogits, *logp;
  otk_loss_stats* d_stats;
  CU(cudaMalloc((void**)&loss_mask, N));
  CU(cudaMalloc((void**)&row_traj, N * 4));
  CU(cudaMalloc((void**)&traj_tokens, B * 8));
  CU(cudaMalloc((void**)&n_loss, 8));
  CU(cudaMalloc((void**)&gid_all, 2 * 4));
  CU(cudaMalloc((void**)&ret_all, 2 * 8));
  CU(cudaMalloc((void**)&adv_all, 2 * 8));
  CU(cudaMalloc((void**)&dlogits, sizeof(float) * N * V));
  CU(cudaMalloc((void**)&logp, N * 4));
  CU(cudaMalloc((void**)&d_stats, sizeof(otk_loss_stats)));
  float* d_logits = (float*)dev_copy(logits, sizeof(float) * N * V);
  int32_t* d_targets = (int32_t*)dev_copy(targets, sizeof(int32_t) * N);
  int32_t* d_gid = (int32_t*)dev_copy(gid_local, sizeof(int32_t) * B);
  double* d_ret = (double*)dev_copy(g_returns + b0, sizeof(double) * B);
  /* (1) local masks; exchange 1: the global token count */
  CK(otk_build_masks(ctx, &tb, OTK_ANY_AGENT, loss_mask, NULL, row_traj, traj_tokens, NULL, n_loss, NULL, NULL, NULL));
  CK(otk_batch_allreduce_i64(ctx, n_loss, 1, NULL));
  /* exchange 2 + (2): group statistics over the union of the shards; this rank's advantages start at b0 */
  CK(otk_batch_group_advantages(ctx, B, d_gid, d_ret, counts, 1, OTK_ADV_STD_NORM, 1e-8, gid_all, ret_all, adv_all,
                                NULL, NULL, NULL, NULL));
  /* (3) on-policy log-probs, (4) the loss on the local rows with the global N_loss; exchange 3: the statistics */
  CK(otk_logprob_entropy_fwd(ctx, N, V, V, OTK_F32, d_logits, d_targets, NULL, 1.0f, logp, NULL, NULL, NULL));
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
  CK(otk_policy_loss_fwd_bwd(ctx, N, V, V, OTK_F32, d_logits, d_targets, loss_mask, row_traj, adv_all + b0, logp,
                             logp, n_loss, &cfg, dlogits, NULL, NULL, d_stats, NULL));
  CK(otk_batch_allreduce_f64(ctx, (double*)d_stats, (int64_t)(sizeof(otk_loss_stats) / sizeof(double)), NULL));
  CK(otk_ctx_check(ctx, NULL));
  otk_loss_stats st;
  int64_t nl = 0;
  double a[2];
  CU(cudaMemcpy(&st, d_stats, sizeof(st), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&nl, n_loss, 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(a, adv_all, sizeof(a), cudaMemcpyDeviceToHost));
  const double want = -(7.0 - 5.0) / 12.0;   /* on policy: loss = -sum_j m_j A_j / N_loss, the same on every P */
  const int ok = nl == 12 && fabs(a[0] - 1.0) < 1e-12 && fabs(a[1] + 1.0) < 1e-12 && fabs(st.loss - want) < 1e-6 &&
                 st.n_tokens == 12.0;
  printf("c api batch step: rank %d of %d: n_loss=%lld adv=(%g, %g) loss=%.9f (closed form %.9f) -> %s\n", rank, P,
         (long long)nl, a[0], a[1], st.loss, want, ok ? "ok" : "MISMATCH");
  fflush(stdout);
  otk_ctx_destroy(ctx);
  free(logits);
  free(targets);
  return ok ? 0 : 1;
}

int main(int argc, char** argv) {
  const int P = argc > 1 ? atoi(argv[1]) : 1;
  int rank = -1;
  if (P < 1 || P > 2) {
    fprintf(stderr, "P must be 1 or 2\n");
    return 2;
  }
  /* one process per rank, forked before any CUDA call; rank 0 creates the NCCL id and hands it over a pipe */
  int fds[2];
  if (pipe(fds) != 0) return 2;
  pid_t pids[2];
  for (int r = 0; r < P; ++r) {
    pids[r] = fork();
    if (pids[r] == 0) {
      rank = r;
      unsigned char uid[OTK_COMM_ID_BYTES];
      close(r == 0 ? fds[0] : fds[1]);   /* a reader sees EOF if rank 0 fails before writing */
      if (r == 0) {
        CK(otk_comm_unique_id(uid));
        for (int q = 1; q < P; ++q)
          if (write(fds[1], uid, sizeof(uid)) != (ssize_t)sizeof(uid)) return 2;
      } else {
        size_t got = 0;
        while (got < sizeof(uid)) {
          const ssize_t k = read(fds[0], uid + got, sizeof(uid) - got);
          if (k <= 0) return 2;
          got += (size_t)k;
        }
      }
      _exit(run_rank(r, P, uid));
    }
  }
  close(fds[0]);
  close(fds[1]);
  int fail = 0;
  for (int r = 0; r < P; ++r) {
    int status = 0;
    waitpid(pids[r], &status, 0);
    if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) fail = 1;
  }
  return fail;
}
