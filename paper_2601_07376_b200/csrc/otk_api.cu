// otk_api.cu — the C ABI (include/otk.h): argument validation, ctx ownership, launches, and the
// host-buffer streaming executor used for the end-to-end measurement.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "otk_internal.h"

namespace {

thread_local std::string tl_err;

otk_status fail(otk_status s, const std::string& msg) {
  tl_err = msg;
  return s;
}

otk_status cuda_fail(cudaError_t e, const char* where) {
  tl_err = std::string(where) + ": " + cudaGetErrorString(e);
  return OTK_ERR_CUDA;
}

#define OTK_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) return fail(code, msg); \
  } while (0)

#define OTK_CUDA(call, where)                      \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

size_t dtype_size(otk_dtype d) { return d == OTK_BF16 ? 2 : 4; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Cluster size for the row kernels: the smallest number of CTAs (1..8, any size: a 3-CTA cluster keeps more SMs
// busy than a 4-CTA one) whose per-CTA column segment fits the tensor-memory-resident budget
// (kMaxChunks chunks). Every mode uses the same rule so that the
// forward (3) and the fused loss (4) reduce in the same order (bitwise-equal logp: on-policy ratio = 1).
int choose_csize(int64_t vocab, size_t es, int* seg_elems) {
  const int64_t budget = int64_t(otk::kMaxChunks) * otk::kChunkBytes;
  for (int c = 1; c <= 8; ++c) {
    int64_t seg = (vocab + c - 1) / c;
    seg = (seg + 7) / 8 * 8;
    if (seg * int64_t(es) <= budget && int64_t(c - 1) * seg < vocab) {
      *seg_elems = int(seg);
      return c;
    }
  }
  return 0;
}

otk_status check_rows(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype, const void* logits,
                      const int32_t* targets, int* csize, int* seg_elems) {
  OTK_REQUIRE(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_REQUIRE(dtype == OTK_BF16 || dtype == OTK_F32, OTK_ERR_DTYPE, "unknown dtype");
  OTK_REQUIRE(num_rows >= 0 && vocab >= 1 && ld >= vocab, OTK_ERR_SHAPE, "need num_rows >= 0, vocab >= 1, ld >= vocab");
  OTK_REQUIRE(num_rows == 0 || (logits && targets), OTK_ERR_INVALID_ARG, "logits / targets is NULL");
  OTK_REQUIRE(aligned16(logits) && (ld * int64_t(dtype_size(dtype))) % 16 == 0, OTK_ERR_ALIGNMENT,
              "logits base and row stride must be 16-byte aligned");
  *csize = choose_csize(vocab, dtype_size(dtype), seg_elems);
  OTK_REQUIRE(*csize > 0, OTK_ERR_SHAPE, "vocab too large for the row kernel (> 8 x 152 KB per row)");
  return OTK_OK;
}

otk_status check_cfg(const otk_loss_cfg* cfg, const float* ref_logp, int64_t num_rows) {
  OTK_REQUIRE(cfg, OTK_ERR_INVALID_ARG, "cfg is NULL");
  OTK_REQUIRE(cfg->clip_low >= 0 && cfg->clip_low < 1 && cfg->clip_high >= 0, OTK_ERR_INVALID_ARG,
              "clip_low must be in [0,1), clip_high >= 0");
  OTK_REQUIRE(cfg->log_ratio_clamp > 0 && std::isfinite(cfg->log_ratio_clamp), OTK_ERR_INVALID_ARG,
              "log_ratio_clamp must be > 0");
  OTK_REQUIRE(cfg->logit_scale > 0 && std::isfinite(cfg->logit_scale), OTK_ERR_INVALID_ARG, "logit_scale must be > 0");
  OTK_REQUIRE(cfg->kl_beta >= 0 && std::isfinite(cfg->kl_beta), OTK_ERR_INVALID_ARG, "kl_beta must be >= 0");
  OTK_REQUIRE(cfg->kl_type >= 1 && cfg->kl_type <= 3, OTK_ERR_INVALID_ARG, "kl_type must be 1, 2 or 3");
  OTK_REQUIRE(cfg->kl_beta == 0 || ref_logp || num_rows == 0, OTK_ERR_INVALID_ARG,
              "ref_logp is required when kl_beta != 0");
  OTK_REQUIRE(std::isfinite(cfg->ent_coef), OTK_ERR_INVALID_ARG, "ent_coef must be finite");
  OTK_REQUIRE(cfg->dual_clip == 0 || (cfg->dual_clip > 1 && std::isfinite(cfg->dual_clip)), OTK_ERR_INVALID_ARG,
              "dual_clip must be 0 (off) or > 1");
  OTK_REQUIRE(cfg->reduction >= OTK_TOKEN_MEAN && cfg->reduction <= OTK_SEQ_MEAN_TOKEN_SUM, OTK_ERR_INVALID_ARG,
              "unknown reduction");
  OTK_REQUIRE(cfg->reduction == OTK_TOKEN_MEAN || (cfg->traj_loss_tokens && cfg->n_active_traj), OTK_ERR_INVALID_ARG,
              "sequence-mean reductions need traj_loss_tokens and n_active_traj");
  OTK_REQUIRE(cfg->sft == 0 || cfg->sft == 1, OTK_ERR_INVALID_ARG, "sft must be 0 or 1");
  OTK_REQUIRE(num_rows == 0 || cfg->num_adv >= 1, OTK_ERR_INVALID_ARG, "cfg->num_adv (elements of adv) must be >= 1");
  OTK_REQUIRE(cfg->reduction == OTK_TOKEN_MEAN || num_rows == 0 || cfg->num_traj >= 1, OTK_ERR_INVALID_ARG,
              "sequence-mean reductions need cfg->num_traj (elements of traj_loss_tokens) >= 1");
  return OTK_OK;
}

otk::RowParams base_params(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, const void* logits,
                           const int32_t* targets, const uint8_t* mask, float scale, int csize, int seg_elems) {
  otk::RowParams p;
  std::memset(&p, 0, sizeof(p));
  p.num_rows = num_rows;
  p.vocab = vocab;
  p.ld = ld;
  p.logits = logits;
  p.targets = targets;
  p.mask = mask;
  p.scale = scale;
  p.vocab_start = 0;
  p.vocab_total = vocab;
  p.csize = csize;
  p.seg_elems = seg_elems;
  p.cta_partials = ctx->d_partials;
  p.ticket = ctx->d_tickets + otk::kTicketRows;
  p.err = ctx->d_err;
  p.nshards = 0;
  return p;
}

void set_loss(otk::RowParams& p, const int32_t* row_traj, const double* adv, const float* old_logp,
              const float* ref_logp, const int64_t* n_loss, const otk_loss_cfg* cfg, void* dlogits, float* logp,
              float* entropy, otk_loss_stats* stats) {
  p.row_traj = row_traj;
  p.adv = adv;
  p.old_logp = old_logp;
  p.ref_logp = cfg->kl_beta != 0 ? ref_logp : nullptr;
  p.n_loss = n_loss;
  p.clip_low = cfg->clip_low;
  p.clip_high = cfg->clip_high;
  p.kl_beta = cfg->kl_beta;
  p.clamp = cfg->log_ratio_clamp;
  p.kl_type = cfg->kl_type;
  p.ent_coef = cfg->ent_coef;
  p.dual_clip = cfg->dual_clip;
  p.reduction = cfg->reduction;
  p.sft = cfg->sft;
  p.traj_tokens = cfg->traj_loss_tokens;
  p.n_active = cfg->n_active_traj;
  p.adv_index = cfg->adv_index;
  p.num_adv = cfg->num_adv;
  p.num_traj = cfg->num_traj;
  p.zero_masked = cfg->zero_masked_rows;
  p.accumulate = cfg->accumulate_stats;
  p.dlogits = dlogits;
  p.logp = logp;
  p.entropy = entropy;
  p.stats = stats;
}

}  // namespace

otk_status otk::host_fail(otk_status s, const char* msg) { return fail(s, msg); }

extern "C" {

int otk_version(void) { return OTK_VERSION; }

const char* otk_last_error(void) { return tl_err.c_str(); }

const char* otk_status_string(otk_status s) {
  switch (s) {
    case OTK_OK: return "OTK_OK";
    case OTK_ERR_INVALID_ARG: return "OTK_ERR_INVALID_ARG";
    case OTK_ERR_SHAPE: return "OTK_ERR_SHAPE";
    case OTK_ERR_ALIGNMENT: return "OTK_ERR_ALIGNMENT";
    case OTK_ERR_DTYPE: return "OTK_ERR_DTYPE";
    case OTK_ERR_EMPTY_GROUP: return "OTK_ERR_EMPTY_GROUP";
    case OTK_ERR_UNTERMINATED: return "OTK_ERR_UNTERMINATED";
    case OTK_ERR_BAD_TRAJECTORY: return "OTK_ERR_BAD_TRAJECTORY";
    case OTK_ERR_TARGET_RANGE: return "OTK_ERR_TARGET_RANGE";
    case OTK_ERR_CUDA: return "OTK_ERR_CUDA";
    case OTK_ERR_GROUP_RANGE: return "OTK_ERR_GROUP_RANGE";
    case OTK_ERR_PEER_TIMEOUT: return "OTK_ERR_PEER_TIMEOUT";
    case OTK_ERR_NCCL: return "OTK_ERR_NCCL";
    case OTK_ERR_NO_COMM: return "OTK_ERR_NO_COMM";
  }
  return "OTK_ERR_UNKNOWN";
}

otk_status otk_ctx_create(int cuda_device, otk_ctx** out) {
  OTK_REQUIRE(out, OTK_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  OTK_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  OTK_REQUIRE(cuda_device >= 0 && cuda_device < ndev, OTK_ERR_INVALID_ARG, "bad device index");
  OTK_CUDA(cudaSetDevice(cuda_device), "cudaSetDevice");
  otk_ctx* c = new otk_ctx();
  c->device = cuda_device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  cudaDeviceGetAttribute(&c->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cuda_device);
  c->cap_returns = int64_t(1) << 20;
  cudaError_t e = cudaMalloc(&c->d_err, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_tickets, 8 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_partials, size_t(otk::kMaxCtas) * otk::kStatSlots * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_scratch_i64, size_t(otk::kMaxCtas) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_returns, size_t(c->cap_returns) * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->d_tickets, 0, 8 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    otk_ctx_destroy(c);
    return cuda_fail(e, "otk_ctx_create");
  }
  if (c->max_smem_optin < int(otk::kSlots * otk::kChunkBytes + 1024)) {
    otk_ctx_destroy(c);
    return fail(OTK_ERR_CUDA, "device lacks the shared memory the row kernel needs (sm_100a required)");
  }
  *out = c;
  return OTK_OK;
}

otk_status otk_ctx_destroy(otk_ctx* c) {
  if (!c) return OTK_OK;
  otk::comm_release(c);
  cudaFree(c->d_err);
  cudaFree(c->d_tickets);
  cudaFree(c->d_partials);
  cudaFree(c->d_scratch_i64);
  cudaFree(c->d_returns);
  for (int i = 0; i < 2; ++i) cudaFree(c->stage[i]);
  for (int i = 0; i < 4; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->exec_stream) cudaStreamDestroy(c->exec_stream);
  delete c;
  return OTK_OK;
}

otk_status otk_ctx_check(otk_ctx* ctx, otk_stream_t stream) {
  OTK_REQUIRE(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
  int err = 0;
  OTK_CUDA(cudaMemcpy(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost), "read error word");
  if (err) {
    OTK_CUDA(cudaMemset(ctx->d_err, 0, sizeof(int)), "clear error word");
    return fail(otk_status(err), std::string("device-side data error: ") + otk_status_string(otk_status(err)));
  }
  return OTK_OK;
}

int64_t otk_ctx_launch_count(const otk_ctx* ctx) { return ctx ? ctx->launches : -1; }

otk_status otk_build_masks(otk_ctx* ctx, const otk_traj_batch* batch, int16_t train_agent, uint8_t* loss_mask,
                           uint8_t* response_mask, int32_t* row_traj, int64_t* traj_loss_tokens,
                           int64_t* traj_source_counts, int64_t* n_loss, int64_t* n_active_traj,
                           int32_t* row_seg, otk_stream_t stream) {
  OTK_REQUIRE(ctx && batch, OTK_ERR_INVALID_ARG, "ctx / batch is NULL");
  OTK_REQUIRE(batch->num_traj >= 1, OTK_ERR_EMPTY_GROUP, "num_traj < 1 (EmptyGroup)");
  OTK_REQUIRE(batch->num_rows >= 0, OTK_ERR_SHAPE, "num_rows < 0");
  OTK_REQUIRE(batch->tok_offsets && batch->seg_offsets && batch->seg_source && batch->seg_agent && batch->seg_len,
              OTK_ERR_INVALID_ARG, "segment arrays must not be NULL");
  OTK_REQUIRE(batch->num_rows == 0 || (loss_mask && row_traj), OTK_ERR_INVALID_ARG, "loss_mask / row_traj is NULL");
  OTK_REQUIRE(traj_loss_tokens && n_loss, OTK_ERR_INVALID_ARG, "traj_loss_tokens / n_loss is NULL");
  OTK_REQUIRE(train_agent >= -1, OTK_ERR_INVALID_ARG, "train_agent must be >= -1");
  otk::MaskParams p;
  p.b = *batch;
  p.train_agent = train_agent;
  p.loss_mask = loss_mask;
  p.response_mask = response_mask;
  p.row_traj = row_traj;
  p.traj_loss_tokens = traj_loss_tokens;
  p.traj_source_counts = traj_source_counts;
  p.n_loss = n_loss;
  p.n_active = n_active_traj;
  p.row_seg = row_seg;
  p.ticket = ctx->d_tickets + otk::kTicketMasks;
  p.err = ctx->d_err;
  OTK_CUDA(otk::launch_masks(p, reinterpret_cast<cudaStream_t>(stream)), "k_build_masks launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_group_advantages(otk_ctx* ctx, int32_t num_traj, const int32_t* group_id, int32_t num_groups,
                                const double* returns, const int32_t* turn_offsets, const double* turn_rewards,
                                uint32_t flags, double std_floor, double* adv, double* returns_out,
                                double* group_mean, double* group_std, int32_t* group_size, otk_stream_t stream) {
  OTK_REQUIRE(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_REQUIRE(num_traj >= 1, OTK_ERR_EMPTY_GROUP, "num_traj < 1 (EmptyGroup)");
  OTK_REQUIRE(num_groups >= 1 && num_groups <= 12000, OTK_ERR_SHAPE, "num_groups must be in [1, 12000]");
  OTK_REQUIRE(group_id && adv, OTK_ERR_INVALID_ARG, "group_id / adv is NULL");
  OTK_REQUIRE((returns != nullptr) != (turn_offsets != nullptr), OTK_ERR_INVALID_ARG,
              "exactly one of returns and turn_offsets must be given");
  OTK_REQUIRE(!turn_offsets || turn_rewards, OTK_ERR_INVALID_ARG, "turn_rewards is NULL");
  OTK_REQUIRE((flags & ~(OTK_ADV_STD_NORM | OTK_ADV_UNBIASED | OTK_ADV_SKIP_UNGROUPED)) == 0, OTK_ERR_INVALID_ARG,
              "unknown flag bits");
  OTK_REQUIRE(std_floor >= 0 && std::isfinite(std_floor), OTK_ERR_INVALID_ARG, "std_floor must be >= 0");
  OTK_REQUIRE(returns_out || num_traj <= ctx->cap_returns, OTK_ERR_SHAPE, "num_traj exceeds ctx scratch");
  otk::AdvParams p;
  p.num_traj = num_traj;
  p.group_id = group_id;
  p.num_groups = num_groups;
  p.returns = returns;
  p.turn_offsets = turn_offsets;
  p.turn_rewards = turn_rewards;
  p.flags = flags;
  p.std_floor = std_floor;
  p.adv = adv;
  p.returns_out = returns_out ? returns_out : ctx->d_returns;
  p.group_mean = group_mean;
  p.group_std = group_std;
  p.group_size = group_size;
  p.err = ctx->d_err;
  OTK_CUDA(otk::launch_advantages(p, reinterpret_cast<cudaStream_t>(stream)), "k_group_advantages launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_turn_returns(otk_ctx* ctx, const otk_traj_batch* batch, int32_t num_segments, int16_t train_agent,
                            const int32_t* group_id, const int32_t* turn_offsets, const double* turn_rewards,
                            double gamma, double* seg_return, int32_t* seg_group, otk_stream_t stream) {
  OTK_REQUIRE(ctx && batch, OTK_ERR_INVALID_ARG, "ctx / batch is NULL");
  OTK_REQUIRE(batch->num_traj >= 1, OTK_ERR_EMPTY_GROUP, "num_traj < 1 (EmptyGroup)");
  OTK_REQUIRE(num_segments >= 0, OTK_ERR_SHAPE, "num_segments < 0");
  OTK_REQUIRE(batch->seg_offsets && batch->seg_source && batch->seg_agent, OTK_ERR_INVALID_ARG,
              "segment arrays must not be NULL");
  OTK_REQUIRE(group_id && turn_offsets && turn_rewards, OTK_ERR_INVALID_ARG, "group_id / turn arrays are NULL");
  OTK_REQUIRE(num_segments == 0 || (seg_return && seg_group), OTK_ERR_INVALID_ARG, "seg_return / seg_group is NULL");
  OTK_REQUIRE(gamma >= 0.0 && gamma <= 1.0, OTK_ERR_INVALID_ARG, "gamma must be in [0, 1]");
  OTK_REQUIRE(train_agent >= -1, OTK_ERR_INVALID_ARG, "train_agent must be >= -1");
  if (num_segments == 0) return OTK_OK;
  otk::TurnParams p;
  p.b = *batch;
  p.num_segments = num_segments;
  p.train_agent = train_agent;
  p.group_id = group_id;
  p.turn_offsets = turn_offsets;
  p.turn_rewards = turn_rewards;
  p.gamma = gamma;
  p.seg_return = seg_return;
  p.seg_group = seg_group;
  p.err = ctx->d_err;
  OTK_CUDA(otk::launch_turn_returns(p, reinterpret_cast<cudaStream_t>(stream)), "k_turn_returns launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_sample_tokens(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                             const void* logits, const float* uniforms, float logit_scale, int32_t greedy,
                             int32_t* tokens, float* logp, otk_stream_t stream) {
  OTK_REQUIRE(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_REQUIRE(dtype == OTK_BF16 || dtype == OTK_F32, OTK_ERR_DTYPE, "unknown dtype");
  OTK_REQUIRE(num_rows >= 0 && vocab >= 1 && ld >= vocab && vocab < (int64_t(1) << 31), OTK_ERR_SHAPE,
              "need num_rows >= 0, 1 <= vocab < 2^31, ld >= vocab");
  OTK_REQUIRE(greedy == 0 || greedy == 1, OTK_ERR_INVALID_ARG, "greedy must be 0 or 1");
  OTK_REQUIRE(logit_scale > 0 && std::isfinite(logit_scale), OTK_ERR_INVALID_ARG, "logit_scale must be > 0");
  if (num_rows == 0) return OTK_OK;
  OTK_REQUIRE(logits && tokens, OTK_ERR_INVALID_ARG, "logits / tokens is NULL");
  OTK_REQUIRE(greedy || uniforms, OTK_ERR_INVALID_ARG, "uniforms is NULL (required unless greedy)");
  OTK_REQUIRE(aligned16(logits) && (ld * int64_t(dtype_size(dtype))) % 16 == 0, OTK_ERR_ALIGNMENT,
              "logits base and row stride must be 16-byte aligned");
  otk::SampleParams p;
  p.num_rows = num_rows;
  p.vocab = vocab;
  p.ld = ld;
  p.logits = logits;
  p.u = uniforms;
  p.scale = logit_scale;
  p.greedy = greedy;
  p.tokens = tokens;
  p.logp = logp;
  p.err = ctx->d_err;
  OTK_CUDA(otk::launch_sample(ctx, p, dtype, reinterpret_cast<cudaStream_t>(stream)), "k_sample launch");
  ctx->launches += 1;
  return OTK_OK;
}

int64_t otk_lmhead_workspace_bytes(const otk_ctx* ctx, int64_t num_rows, int64_t vocab) {
  if (!ctx || num_rows < 0 || vocab < 1) return -1;
  return int64_t(otk::lmhead_chunks(num_rows, vocab, ctx->num_sms)) * num_rows * 16;
}

otk_status otk_lmhead_logprob_fwd(otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab,
                                  const void* hidden, const void* weight, const int32_t* targets,
                                  const uint8_t* row_mask, float logit_scale, void* workspace,
                                  int64_t workspace_bytes, float* logp, float* entropy, float* lse,
                                  otk_stream_t stream) {
  OTK_REQUIRE(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_REQUIRE(num_rows >= 0 && vocab >= 1 && vocab < (int64_t(1) << 31) && num_rows < (int64_t(1) << 31),
              OTK_ERR_SHAPE, "need 0 <= num_rows < 2^31, 1 <= vocab < 2^31");
  OTK_REQUIRE(hidden_dim >= 64 && hidden_dim % 64 == 0 && hidden_dim <= 65536, OTK_ERR_SHAPE,
              "hidden_dim must be a positive multiple of 64 (<= 65536)");
  OTK_REQUIRE(logit_scale > 0 && std::isfinite(logit_scale), OTK_ERR_INVALID_ARG, "logit_scale must be > 0");
  if (num_rows == 0) return OTK_OK;
  OTK_REQUIRE(hidden && weight && targets && logp && workspace, OTK_ERR_INVALID_ARG,
              "hidden / weight / targets / logp / workspace is NULL");
  OTK_REQUIRE(aligned16(hidden) && aligned16(weight) && aligned16(workspace), OTK_ERR_ALIGNMENT,
              "hidden, weight and workspace must be 16-byte aligned");
  const int n_chunks = otk::lmhead_chunks(num_rows, vocab, ctx->num_sms);
  OTK_REQUIRE(workspace_bytes >= int64_t(n_chunks) * num_rows * 16, OTK_ERR_SHAPE,
              "workspace smaller than otk_lmhead_workspace_bytes()");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float4* part = reinterpret_cast<float4*>(workspace);
  OTK_CUDA(otk::launch_lmhead_fwd(ctx, num_rows, vocab, int(hidden_dim), hidden, weight, targets, row_mask,
                                  logit_scale, part, n_chunks, s),
           "k_lmhead_fwd launch");
  ctx->launches += 1;
  OTK_CUDA(otk::launch_combine(ctx, num_rows, n_chunks, part, row_mask, logp, entropy, lse, s), "k_combine launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_lmhead_row_partials(otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab_local,
                                   const void* hidden, const void* weight, const int32_t* targets,
                                   const uint8_t* row_mask, const otk_vocab_shard* shard, float logit_scale,
                                   void* workspace, int64_t workspace_bytes, float* partials, otk_stream_t stream) {
  OTK_REQUIRE(ctx && shard, OTK_ERR_INVALID_ARG, "ctx / shard is NULL");
  OTK_REQUIRE(num_rows >= 0 && vocab_local >= 1 && vocab_local < (int64_t(1) << 31) && num_rows < (int64_t(1) << 31),
              OTK_ERR_SHAPE, "need 0 <= num_rows < 2^31, 1 <= vocab_local < 2^31");
  OTK_REQUIRE(shard->vocab_start >= 0 && shard->vocab_start + vocab_local <= shard->vocab_total &&
                  shard->vocab_total < (int64_t(1) << 31),
              OTK_ERR_SHAPE, "shard outside [0, vocab_total)");
  OTK_REQUIRE(hidden_dim >= 64 && hidden_dim % 64 == 0 && hidden_dim <= 65536, OTK_ERR_SHAPE,
              "hidden_dim must be a positive multiple of 64 (<= 65536)");
  OTK_REQUIRE(logit_scale > 0 && std::isfinite(logit_scale), OTK_ERR_INVALID_ARG, "logit_scale must be > 0");
  if (num_rows == 0) return OTK_OK;
  OTK_REQUIRE(hidden && weight && targets && workspace && partials, OTK_ERR_INVALID_ARG,
              "hidden / weight / targets / workspace / partials is NULL");
  OTK_REQUIRE(aligned16(hidden) && aligned16(weight) && aligned16(workspace) && aligned16(partials),
              OTK_ERR_ALIGNMENT, "hidden, weight, workspace and partials must be 16-byte aligned");
  const int n_chunks = otk::lmhead_chunks(num_rows, vocab_local, ctx->num_sms);
  OTK_REQUIRE(workspace_bytes >= int64_t(n_chunks) * num_rows * 16, OTK_ERR_SHAPE,
              "workspace smaller than otk_lmhead_workspace_bytes()");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float4* part = reinterpret_cast<float4*>(workspace);
  OTK_CUDA(otk::launch_lmhead_fwd(ctx, num_rows, vocab_local, int(hidden_dim), hidden, weight, targets, row_mask,
                                  logit_scale, part, n_chunks, s, shard->vocab_start, shard->vocab_total),
           "k_lmhead_fwd launch");
  ctx->launches += 1;
  OTK_CUDA(otk::launch_combine_to_partial(ctx, num_rows, n_chunks, part, row_mask, reinterpret_cast<float4*>(partials),
                                          s),
           "k_combine_to_partial launch");
  ctx->launches += 1;
  return OTK_OK;
}

namespace {
struct LmLossWs {
  int n_chunks, splits;
  int64_t cols_pad, x_off, dx_off, part_off, rowc_off, dh_off, bytes;
};
// workspace: x tiles [rows_pad/64][cols_pad/64][64][64] bf16 | dx tiles (same layout) | chunk partials |
// row constants | dh split-K partials
LmLossWs lm_loss_ws(const otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab) {
  LmLossWs w;
  w.n_chunks = otk::lmhead_chunks(num_rows, vocab, ctx->num_sms);
  w.splits = otk::lmhead_dh_splits(num_rows, vocab, int(hidden_dim), ctx->num_sms);
  const int64_t rows_pad = (num_rows + 255) / 256 * 256;
  w.cols_pad = (vocab + 255) / 256 * 256;
  auto up = [](int64_t b) { return (b + 255) / 256 * 256; };  // every region 256-byte aligned (256-bit stores)
  w.x_off = 0;
  w.dx_off = up(rows_pad * w.cols_pad * 2);
  w.part_off = up(w.dx_off + rows_pad * w.cols_pad * 2);
  w.rowc_off = up(w.part_off + int64_t(w.n_chunks) * num_rows * 16);
  w.dh_off = up(w.rowc_off + num_rows * 16);
  w.bytes = w.dh_off + (w.splits > 1 ? int64_t(w.splits) * num_rows * hidden_dim * 4 : 0);
  return w;
}
}  // namespace

int64_t otk_lmhead_loss_workspace_bytes(const otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab) {
  if (!ctx || num_rows < 0 || vocab < 1 || hidden_dim < 64 || hidden_dim % 64 != 0) return -1;
  return lm_loss_ws(ctx, num_rows, hidden_dim, vocab).bytes;
}

otk_status otk_lmhead_policy_loss_fwd_bwd(otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab,
                                          const void* hidden, const void* weight, const int32_t* targets,
                                          const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                          const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                          const otk_loss_cfg* cfg, void* workspace, int64_t workspace_bytes,
                                          void* dhidden, void* dweight, float* logp, float* entropy,
                                          otk_loss_stats* stats, otk_stream_t stream) {
  OTK_REQUIRE(ctx, OTK_ERR_INVALID_ARG, "ctx is NULL");
  OTK_REQUIRE(num_rows >= 0 && vocab >= 8 && vocab % 8 == 0 && vocab < (int64_t(1) << 31) &&
                  num_rows < (int64_t(1) << 31),
              OTK_ERR_SHAPE, "need 0 <= num_rows < 2^31 and vocab a positive multiple of 8 (< 2^31)");
  OTK_REQUIRE(hidden_dim >= 64 && hidden_dim % 64 == 0 && hidden_dim <= 65536, OTK_ERR_SHAPE,
              "hidden_dim must be a positive multiple of 64 (<= 65536)");
  otk_status st = check_cfg(cfg, ref_logp, num_rows);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(stats, OTK_ERR_INVALID_ARG, "stats is NULL");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (num_rows == 0) {  // no rows: dW = 0 and (unless accumulating) zero stats, as otk_policy_loss_fwd_bwd
    OTK_REQUIRE(dweight, OTK_ERR_INVALID_ARG, "dweight is NULL");
    OTK_CUDA(cudaMemsetAsync(dweight, 0, size_t(vocab) * size_t(hidden_dim) * 2, s), "zero dweight");
    if (!cfg->accumulate_stats) OTK_CUDA(cudaMemsetAsync(stats, 0, sizeof(otk_loss_stats), s), "zero stats");
    return OTK_OK;
  }
  OTK_REQUIRE(hidden && weight && targets && loss_mask && row_traj && adv && old_logp && n_loss && workspace &&
                  dhidden && dweight,
              OTK_ERR_INVALID_ARG, "a required pointer is NULL");
  auto aligned32 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 31u) == 0; };
  OTK_REQUIRE(aligned16(hidden) && aligned16(weight) && aligned32(workspace) && aligned32(dhidden) &&
                  aligned32(dweight),
              OTK_ERR_ALIGNMENT, "hidden / weight must be 16-byte, workspace / dhidden / dweight 32-byte aligned");
  OTK_REQUIRE(dhidden != hidden && dhidden != weight && dweight != hidden && dweight != weight && dhidden != dweight,
              OTK_ERR_INVALID_ARG, "outputs must not alias inputs");
  const LmLossWs w = lm_loss_ws(ctx, num_rows, hidden_dim, vocab);
  OTK_REQUIRE(workspace_bytes >= w.bytes, OTK_ERR_SHAPE, "workspace smaller than otk_lmhead_loss_workspace_bytes()");
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  void* logits = ws + w.x_off;
  void* dx_tiles = ws + w.dx_off;
  float4* part = reinterpret_cast<float4*>(ws + w.part_off);
  float4* rowc = reinterpret_cast<float4*>(ws + w.rowc_off);
  float* dh_part = reinterpret_cast<float*>(ws + w.dh_off);
  const float scale = float(cfg->logit_scale);
  // (a) x = h W^T on tcgen05: bf16 x tiles out + per-(row, vocab chunk) log-softmax partials of the rounded x
  OTK_CUDA(otk::launch_lmhead_fwd(ctx, num_rows, vocab, int(hidden_dim), hidden, weight, targets, loss_mask, scale,
                                  part, w.n_chunks, s, 0, vocab, logits, w.cols_pad / 64),
           "k_lmhead_fwd launch");
  ctx->launches += 1;
  // (b) per row: combine, finalize, loss terms of (4), stats; the backward's per-row constants
  int csize = 1, seg = 0;
  otk::RowParams p = base_params(ctx, num_rows, vocab, vocab, logits, targets, loss_mask, scale, csize, seg);
  p.partials_in = part;
  p.nshards = w.n_chunks;
  set_loss(p, row_traj, adv, old_logp, ref_logp, n_loss, cfg, nullptr, logp, entropy, stats);
  OTK_CUDA(otk::launch_lmhead_loss_rows(ctx, p, rowc, s), "k_lmhead_loss_rows launch");
  ctx->launches += 1;
  // (c) dh = dx W and dW = dx^T h on tcgen05, dx formed in shared memory from x and the row constants
  int nl = 0;
  OTK_CUDA(otk::launch_lmhead_bwd(ctx, num_rows, vocab, int(hidden_dim), hidden, weight, logits, dx_tiles, rowc,
                                  targets, 0,
                                  scale, cfg->ent_coef != 0, dhidden, dweight, dh_part, w.splits, s, &nl),
           "k_lmhead_bwd launch");
  ctx->launches += nl;
  return OTK_OK;
}

otk_status otk_logprob_entropy_fwd(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                                   const void* logits, const int32_t* targets, const uint8_t* row_mask,
                                   float logit_scale, float* logp, float* entropy, float* lse, otk_stream_t stream) {
  int csize = 0, seg = 0;
  otk_status st = check_rows(ctx, num_rows, vocab, ld, dtype, logits, targets, &csize, &seg);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(logp || num_rows == 0, OTK_ERR_INVALID_ARG, "logp is NULL");
  OTK_REQUIRE(logit_scale > 0 && std::isfinite(logit_scale), OTK_ERR_INVALID_ARG, "logit_scale must be > 0");
  if (num_rows == 0) return OTK_OK;
  otk::RowParams p = base_params(ctx, num_rows, vocab, ld, logits, targets, row_mask, logit_scale, csize, seg);
  p.logp = logp;
  p.entropy = entropy;
  p.lse = lse;
  OTK_CUDA(otk::launch_rows(ctx, otk::kModeFwd, dtype, p, reinterpret_cast<cudaStream_t>(stream), nullptr),
           "k_rows<fwd> launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_policy_loss_fwd_bwd(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                                   const void* logits, const int32_t* targets, const uint8_t* loss_mask,
                                   const int32_t* row_traj, const double* adv, const float* old_logp,
                                   const float* ref_logp, const int64_t* n_loss, const otk_loss_cfg* cfg,
                                   void* dlogits, float* logp, float* entropy, otk_loss_stats* stats,
                                   otk_stream_t stream) {
  int csize = 0, seg = 0;
  otk_status st = check_rows(ctx, num_rows, vocab, ld, dtype, logits, targets, &csize, &seg);
  if (st != OTK_OK) return st;
  st = check_cfg(cfg, ref_logp, num_rows);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(n_loss && stats, OTK_ERR_INVALID_ARG, "n_loss and stats are required");
  OTK_REQUIRE(num_rows == 0 || (loss_mask && row_traj && adv && old_logp && dlogits), OTK_ERR_INVALID_ARG,
              "loss_mask, row_traj, adv, old_logp and dlogits are required (num_rows > 0)");
  OTK_REQUIRE(dlogits != logits || num_rows == 0, OTK_ERR_INVALID_ARG, "dlogits must not alias logits");
  OTK_REQUIRE(aligned16(dlogits), OTK_ERR_ALIGNMENT, "dlogits must be 16-byte aligned");
  otk::RowParams p = base_params(ctx, num_rows, vocab, ld, logits, targets, loss_mask, float(cfg->logit_scale),
                                 csize, seg);
  set_loss(p, row_traj, adv, old_logp, ref_logp, n_loss, cfg, dlogits, logp, entropy, stats);
  OTK_CUDA(otk::launch_rows(ctx, otk::kModeBwd, dtype, p, reinterpret_cast<cudaStream_t>(stream), nullptr),
           "k_rows<bwd> launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_row_partials(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld, otk_dtype dtype,
                            const void* logits, const int32_t* targets, const uint8_t* row_mask,
                            const otk_vocab_shard* shard, float logit_scale, float* partials, otk_stream_t stream) {
  int csize = 0, seg = 0;
  otk_status st = check_rows(ctx, num_rows, vocab_local, ld, dtype, logits, targets, &csize, &seg);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(shard && (partials || num_rows == 0), OTK_ERR_INVALID_ARG, "shard / partials is NULL");
  OTK_REQUIRE(shard->vocab_start >= 0 && shard->vocab_start + vocab_local <= shard->vocab_total, OTK_ERR_SHAPE,
              "shard outside [0, vocab_total)");
  OTK_REQUIRE(aligned16(partials), OTK_ERR_ALIGNMENT, "partials must be 16-byte aligned");
  OTK_REQUIRE(logit_scale > 0 && std::isfinite(logit_scale), OTK_ERR_INVALID_ARG, "logit_scale must be > 0");
  if (num_rows == 0) return OTK_OK;
  otk::RowParams p = base_params(ctx, num_rows, vocab_local, ld, logits, targets, row_mask, logit_scale, csize, seg);
  p.vocab_start = shard->vocab_start;
  p.vocab_total = shard->vocab_total;
  p.partials_out = reinterpret_cast<float4*>(partials);
  OTK_CUDA(otk::launch_rows(ctx, otk::kModePartial, dtype, p, reinterpret_cast<cudaStream_t>(stream), nullptr),
           "k_rows<partial> launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_logprob_entropy_combine(otk_ctx* ctx, int64_t num_rows, int32_t nshards, const float* partials,
                                       const uint8_t* row_mask, float* logp, float* entropy, float* lse,
                                       otk_stream_t stream) {
  OTK_REQUIRE(ctx && ((partials && logp) || num_rows == 0), OTK_ERR_INVALID_ARG, "ctx / partials / logp is NULL");
  OTK_REQUIRE(num_rows >= 0 && nshards >= 1, OTK_ERR_SHAPE, "num_rows >= 0 and nshards >= 1 required");
  OTK_REQUIRE(aligned16(partials), OTK_ERR_ALIGNMENT, "partials must be 16-byte aligned");
  if (num_rows == 0) return OTK_OK;
  OTK_CUDA(otk::launch_combine(ctx, num_rows, nshards, reinterpret_cast<const float4*>(partials), row_mask, logp,
                               entropy, lse, reinterpret_cast<cudaStream_t>(stream)),
           "k_combine launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_policy_loss_fwd_bwd_partials(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld,
                                            otk_dtype dtype, const void* logits, const int32_t* targets,
                                            const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                            const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                            const otk_loss_cfg* cfg, const otk_vocab_shard* shard, int32_t nshards,
                                            const float* partials, void* dlogits, float* logp, float* entropy,
                                            otk_loss_stats* stats, otk_stream_t stream) {
  int csize = 0, seg = 0;
  otk_status st = check_rows(ctx, num_rows, vocab_local, ld, dtype, logits, targets, &csize, &seg);
  if (st != OTK_OK) return st;
  st = check_cfg(cfg, ref_logp, num_rows);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(loss_mask && row_traj && adv && old_logp && n_loss && dlogits && stats && shard && partials,
              OTK_ERR_INVALID_ARG, "a required pointer is NULL");
  OTK_REQUIRE(nshards >= 1, OTK_ERR_SHAPE, "nshards >= 1 required");
  OTK_REQUIRE(shard->vocab_start >= 0 && shard->vocab_start + vocab_local <= shard->vocab_total, OTK_ERR_SHAPE,
              "shard outside [0, vocab_total)");
  OTK_REQUIRE(dlogits != logits || num_rows == 0, OTK_ERR_INVALID_ARG, "dlogits must not alias logits");
  OTK_REQUIRE(aligned16(dlogits) && aligned16(partials), OTK_ERR_ALIGNMENT, "dlogits / partials alignment");
  otk::RowParams p = base_params(ctx, num_rows, vocab_local, ld, logits, targets, loss_mask,
                                 float(cfg->logit_scale), csize, seg);
  p.vocab_start = shard->vocab_start;
  p.vocab_total = shard->vocab_total;
  p.partials_in = reinterpret_cast<const float4*>(partials);
  p.nshards = nshards;
  set_loss(p, row_traj, adv, old_logp, ref_logp, n_loss, cfg, dlogits, logp, entropy, stats);
  OTK_CUDA(otk::launch_rows(ctx, otk::kModeBwdPartials, dtype, p, reinterpret_cast<cudaStream_t>(stream), nullptr),
           "k_rows<bwd_partials> launch");
  ctx->launches += 1;
  return OTK_OK;
}

// ---- K4-VPF: (4) on a vocab shard with the row-partial exchange fused into the kernel -------------------
int64_t otk_vpf_xchg_bytes(int64_t rows_cap, int32_t nranks) {
  if (rows_cap < 1 || nranks < 1 || nranks > OTK_VPF_MAX_RANKS) return -1;
  return 2 * rows_cap * nranks * 32 + 64;  // [2][cap][P] records of four (value | epoch) words + tail: call
                                            // counter (u32), abort epoch (u32)
}

}  // extern "C"

// One rank's K4-VPF call: host checks + its RowParams (shared by the single-call and the grouped entry points).
static otk_status vpf_params(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld, otk_dtype dtype,
                             const void* logits, const int32_t* targets, const uint8_t* loss_mask,
                             const int32_t* row_traj, const double* adv, const float* old_logp, const float* ref_logp,
                             const int64_t* n_loss, const otk_loss_cfg* cfg, const otk_vocab_shard* shard,
                             const otk_vpf_peers* peers, void* dlogits, float* logp, float* entropy,
                             otk_loss_stats* stats, otk::RowParams* out) {
  int csize = 0, seg = 0;
  otk_status st = check_rows(ctx, num_rows, vocab_local, ld, dtype, logits, targets, &csize, &seg);
  if (st != OTK_OK) return st;
  st = check_cfg(cfg, ref_logp, num_rows);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(n_loss && stats && shard && peers, OTK_ERR_INVALID_ARG, "n_loss, stats, shard and peers are required");
  OTK_REQUIRE(num_rows == 0 || (loss_mask && row_traj && adv && old_logp && dlogits), OTK_ERR_INVALID_ARG,
              "loss_mask, row_traj, adv, old_logp and dlogits are required (num_rows > 0)");
  OTK_REQUIRE(shard->vocab_start >= 0 && shard->vocab_start + vocab_local <= shard->vocab_total, OTK_ERR_SHAPE,
              "shard outside [0, vocab_total)");
  OTK_REQUIRE(peers->nranks >= 1 && peers->nranks <= OTK_VPF_MAX_RANKS && peers->rank >= 0 &&
                  peers->rank < peers->nranks, OTK_ERR_INVALID_ARG, "need 0 <= rank < nranks <= OTK_VPF_MAX_RANKS");
  OTK_REQUIRE(peers->rows_cap >= num_rows && peers->rows_cap >= 1, OTK_ERR_SHAPE, "num_rows > rows_cap");
  OTK_REQUIRE(peers->max_ctas >= 0, OTK_ERR_INVALID_ARG, "max_ctas must be >= 0");
  for (int q = 0; q < peers->nranks; ++q)
    OTK_REQUIRE(peers->xchg[q] && aligned16(peers->xchg[q]), OTK_ERR_ALIGNMENT,
                "every xchg[q] must be a 16-byte aligned device pointer");
  OTK_REQUIRE(dlogits != logits || num_rows == 0, OTK_ERR_INVALID_ARG, "dlogits must not alias logits");
  OTK_REQUIRE(aligned16(dlogits), OTK_ERR_ALIGNMENT, "dlogits must be 16-byte aligned");
  OTK_REQUIRE(peers->max_ctas == 0 || peers->max_ctas >= csize, OTK_ERR_INVALID_ARG, "max_ctas below the cluster size");
  otk::RowParams p = base_params(ctx, num_rows, vocab_local, ld, logits, targets, loss_mask,
                                 float(cfg->logit_scale), csize, seg);
  p.vocab_start = shard->vocab_start;
  p.vocab_total = shard->vocab_total;
  set_loss(p, row_traj, adv, old_logp, ref_logp, n_loss, cfg, dlogits, logp, entropy, stats);
  for (int q = 0; q < peers->nranks; ++q) p.vpf_xchg[q] = peers->xchg[q];
  p.vpf_rank = peers->rank;
  p.vpf_nranks = peers->nranks;
  p.vpf_counter = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(peers->xchg[peers->rank]) +
                                              2 * peers->rows_cap * peers->nranks * 32);
  p.vpf_abort = p.vpf_counter + 1;
  p.vpf_rows_cap = peers->rows_cap;
  // pipelined loop (exchange latency hidden behind the next row's pass 1) when a CTA holds the whole shard row
  // and two rows fit its tensor memory
  {
    const int64_t seg_bytes = int64_t(seg) * int64_t(dtype_size(dtype));
    p.pipe = csize != 1 ? 0 : seg_bytes <= otk::kLag3Chunks * int64_t(otk::kChunkBytes) ? 3
                               : seg_bytes <= int64_t(otk::kPipeChunks) * otk::kChunkBytes ? 1 : 0;
  }
#ifdef OTK_VPF_LAG1  // experiment builds only: the lag-1 pipeline for every segment that fits it
  if (p.pipe == 3) p.pipe = 1;
#endif
#ifdef OTK_VPF_NOPIPE  // experiment builds only: measure the unpipelined loop
  p.pipe = 0;
#endif
  *out = p;
  return OTK_OK;
}

extern "C" {

otk_status otk_policy_loss_fwd_bwd_vpf(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld,
                                       otk_dtype dtype, const void* logits, const int32_t* targets,
                                       const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                       const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                       const otk_loss_cfg* cfg, const otk_vocab_shard* shard,
                                       const otk_vpf_peers* peers, void* dlogits, float* logp, float* entropy,
                                       otk_loss_stats* stats, otk_stream_t stream) {
  otk::RowParams p;
  otk_status st = vpf_params(ctx, num_rows, vocab_local, ld, dtype, logits, targets, loss_mask, row_traj, adv,
                             old_logp, ref_logp, n_loss, cfg, shard, peers, dlogits, logp, entropy, stats, &p);
  if (st != OTK_OK) return st;
  OTK_CUDA(otk::launch_rows(ctx, otk::kModeBwdVpf, dtype, p, reinterpret_cast<cudaStream_t>(stream), nullptr,
                            peers->max_ctas),
           "k_rows<bwd_vpf> launch");
  ctx->launches += 1;
  return OTK_OK;
}

otk_status otk_policy_loss_fwd_bwd_vpf_group(int32_t nranks, const otk_vpf_rank_call* calls, int64_t num_rows,
                                             int64_t ld, otk_dtype dtype, const int32_t* targets,
                                             const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                             const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                             const otk_loss_cfg* cfg, otk_stream_t stream) {
  OTK_REQUIRE(calls && nranks >= 1 && nranks <= OTK_VPF_MAX_RANKS, OTK_ERR_INVALID_ARG,
              "need 1 <= nranks <= OTK_VPF_MAX_RANKS calls");
  otk::RowParams ps[OTK_VPF_MAX_RANKS];
  for (int k = 0; k < nranks; ++k) {
    const otk_vpf_rank_call& c = calls[k];
    OTK_REQUIRE(c.ctx && c.peers, OTK_ERR_INVALID_ARG, "every call needs a ctx and peers");
    OTK_REQUIRE(c.peers->rank == k && c.peers->nranks == nranks, OTK_ERR_INVALID_ARG,
                "calls[k] must be rank k of an nranks-rank exchange");
    for (int q = 0; q < k; ++q)
      OTK_REQUIRE(calls[q].ctx != c.ctx, OTK_ERR_INVALID_ARG, "every rank needs its own ctx (scratch, ticket)");
    OTK_REQUIRE(c.ctx->device == calls[0].ctx->device, OTK_ERR_INVALID_ARG, "all ctxs must be on one device");
    otk_status st = vpf_params(c.ctx, num_rows, c.vocab_local, ld, dtype, c.logits, targets, loss_mask, row_traj, adv,
                               old_logp, ref_logp, n_loss, cfg, &c.shard, c.peers, c.dlogits, c.logp, c.entropy,
                               c.stats, &ps[k]);
    if (st != OTK_OK) return st;
    OTK_REQUIRE(ps[k].csize == ps[0].csize && ps[k].pipe == ps[0].pipe, OTK_ERR_SHAPE,
                "every rank's shard must use the same cluster size and loop (near-equal shard widths)");
  }
  OTK_CUDA(otk::launch_rows_vpf_group(calls[0].ctx, dtype, ps, nranks, ps[0].pipe,
                                      reinterpret_cast<cudaStream_t>(stream), nullptr),
           "k_rows_vpf_group launch (all ranks co-resident)");
  calls[0].ctx->launches += 1;
  return OTK_OK;
}

static_assert(sizeof(cudaIpcMemHandle_t) == OTK_IPC_HANDLE_BYTES, "IPC handle size");

otk_status otk_xchg_alloc(otk_ctx* ctx, int64_t bytes, void** dev_ptr_out) {
  OTK_REQUIRE(ctx && dev_ptr_out && bytes > 0, OTK_ERR_INVALID_ARG, "need ctx, dev_ptr_out and bytes > 0");
  OTK_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  void* p = nullptr;
  OTK_CUDA(cudaMalloc(&p, size_t(bytes)), "exchange buffer cudaMalloc");
  cudaError_t e = cudaMemset(p, 0, size_t(bytes));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any peer can map and write it
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "exchange buffer zeroing");
  }
  *dev_ptr_out = p;
  return OTK_OK;
}

otk_status otk_xchg_free(otk_ctx* ctx, void* dev_ptr) {
  OTK_REQUIRE(ctx && dev_ptr, OTK_ERR_INVALID_ARG, "NULL pointer");
  OTK_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  OTK_CUDA(cudaFree(dev_ptr), "cudaFree");
  return OTK_OK;
}

otk_status otk_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  OTK_REQUIRE(dev_ptr && handle_out, OTK_ERR_INVALID_ARG, "NULL pointer");
  cudaIpcMemHandle_t h;
  OTK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof(h));
  return OTK_OK;
}

otk_status otk_ipc_open(const void* handle, void** dev_ptr_out) {
  OTK_REQUIRE(handle && dev_ptr_out, OTK_ERR_INVALID_ARG, "NULL pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  OTK_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return OTK_OK;
}

otk_status otk_ipc_close(void* dev_ptr) {
  OTK_REQUIRE(dev_ptr, OTK_ERR_INVALID_ARG, "NULL pointer");
  OTK_CUDA(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  return OTK_OK;
}

// ---- host-buffer streaming executor (e2e measurement) -------------------------------------------------
otk_status otk_policy_loss_fwd_bwd_host(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                                        const void* logits_host, const int32_t* targets_host,
                                        const uint8_t* loss_mask_host, const int32_t* row_traj_host, int32_t num_traj,
                                        const double* adv_host, const float* old_logp_host,
                                        const float* ref_logp_host, int64_t n_loss, const otk_loss_cfg* cfg,
                                        void* dlogits_host, otk_loss_stats* stats_host, int64_t rows_per_chunk) {
  int csize = 0, seg = 0;
  otk_status st = check_rows(ctx, num_rows, vocab, ld, dtype, logits_host, targets_host, &csize, &seg);
  if (st != OTK_OK) return st;
  otk_loss_cfg hc = *cfg;
  hc.num_adv = num_traj;
  st = check_cfg(&hc, ref_logp_host, num_rows);
  if (st != OTK_OK) return st;
  OTK_REQUIRE(loss_mask_host && row_traj_host && adv_host && old_logp_host && stats_host && num_traj >= 1,
              OTK_ERR_INVALID_ARG, "a required host pointer is NULL");
  OTK_REQUIRE(rows_per_chunk >= 1, OTK_ERR_SHAPE, "rows_per_chunk >= 1 required");
  OTK_REQUIRE(cfg->reduction == OTK_TOKEN_MEAN, OTK_ERR_INVALID_ARG, "host entry point: token-mean reduction only");
  OTK_REQUIRE(!cfg->adv_index, OTK_ERR_INVALID_ARG, "host entry point: adv_index not supported");
  const size_t es = dtype_size(dtype);
  const size_t row_bytes = size_t(ld) * es;
  const bool has_ref = cfg->kl_beta != 0;
  // staging layout per buffer: logits | dlogits | targets | mask | row_traj | old | ref
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t R = size_t(rows_per_chunk);
  const size_t off_dl = al(R * row_bytes);
  const size_t off_tg = off_dl + al(R * row_bytes);
  const size_t off_m = off_tg + al(R * 4);
  const size_t off_rt = off_m + al(R);
  const size_t off_old = off_rt + al(R * 4);
  const size_t off_ref = off_old + al(R * 4);
  const size_t off_end = off_ref + al(R * 4);
  const size_t shared_bytes = al(size_t(num_traj) * 8) + al(8) + al(sizeof(otk_loss_stats));
  const size_t need = off_end + shared_bytes;
  if (ctx->stage_bytes < need) {
    for (int i = 0; i < 2; ++i) {
      cudaFree(ctx->stage[i]);
      ctx->stage[i] = nullptr;
    }
    ctx->stage_bytes = 0;
    for (int i = 0; i < 2; ++i) OTK_CUDA(cudaMalloc(&ctx->stage[i], need), "staging cudaMalloc");
    ctx->stage_bytes = need;
  }
  if (!ctx->copy_stream) OTK_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "stream");
  if (!ctx->exec_stream) OTK_CUDA(cudaStreamCreateWithFlags(&ctx->exec_stream, cudaStreamNonBlocking), "stream");
  for (int i = 0; i < 4; ++i)
    if (!ctx->ev[i]) OTK_CUDA(cudaEventCreateWithFlags(&ctx->ev[i], cudaEventDisableTiming), "event");
  cudaStream_t cs = ctx->copy_stream, xs = ctx->exec_stream;
  char* shared = reinterpret_cast<char*>(ctx->stage[0]) + off_end;  // adv | n_loss | stats live in buffer 0
  double* d_adv = reinterpret_cast<double*>(shared);
  int64_t* d_nl = reinterpret_cast<int64_t*>(shared + al(size_t(num_traj) * 8));
  otk_loss_stats* d_stats = reinterpret_cast<otk_loss_stats*>(shared + al(size_t(num_traj) * 8) + al(8));
  OTK_CUDA(cudaMemcpyAsync(d_adv, adv_host, size_t(num_traj) * 8, cudaMemcpyHostToDevice, xs), "H2D adv");
  OTK_CUDA(cudaMemcpyAsync(d_nl, &n_loss, 8, cudaMemcpyHostToDevice, xs), "H2D n_loss");
  OTK_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(otk_loss_stats), xs), "zero stats");
  OTK_CUDA(cudaStreamSynchronize(xs), "sync");  // n_loss lives on the host stack
  int64_t k = 0;
  for (int64_t r0 = 0; r0 < num_rows || (num_rows == 0 && k == 0); r0 += rows_per_chunk, ++k) {
    const int b = int(k & 1);
    const int64_t n = std::min<int64_t>(rows_per_chunk, num_rows - r0);
    char* sb = reinterpret_cast<char*>(ctx->stage[b]);
    if (k >= 2) OTK_CUDA(cudaStreamWaitEvent(cs, ctx->ev[2 + b], 0), "wait free");
    if (n > 0) {
      // logits: only the runs of trainable rows — the kernel never reads a loss-masked row (it only writes
      // its zero gradient), so its bytes need not cross PCIe
      for (int64_t a = 0; a < n;) {
        while (a < n && !loss_mask_host[r0 + a]) ++a;
        int64_t e = a;
        while (e < n && loss_mask_host[r0 + e]) ++e;
        if (e > a)
          OTK_CUDA(cudaMemcpyAsync(sb + size_t(a) * row_bytes,
                                   reinterpret_cast<const char*>(logits_host) + size_t(r0 + a) * row_bytes,
                                   size_t(e - a) * row_bytes, cudaMemcpyHostToDevice, cs),
                   "H2D logits");
        a = e;
      }
      OTK_CUDA(cudaMemcpyAsync(sb + off_tg, targets_host + r0, size_t(n) * 4, cudaMemcpyHostToDevice, cs), "H2D");
      OTK_CUDA(cudaMemcpyAsync(sb + off_m, loss_mask_host + r0, size_t(n), cudaMemcpyHostToDevice, cs), "H2D");
      OTK_CUDA(cudaMemcpyAsync(sb + off_rt, row_traj_host + r0, size_t(n) * 4, cudaMemcpyHostToDevice, cs), "H2D");
      OTK_CUDA(cudaMemcpyAsync(sb + off_old, old_logp_host + r0, size_t(n) * 4, cudaMemcpyHostToDevice, cs), "H2D");
      if (has_ref)
        OTK_CUDA(cudaMemcpyAsync(sb + off_ref, ref_logp_host + r0, size_t(n) * 4, cudaMemcpyHostToDevice, cs), "H2D");
    }
    OTK_CUDA(cudaEventRecord(ctx->ev[b], cs), "record ready");
    OTK_CUDA(cudaStreamWaitEvent(xs, ctx->ev[b], 0), "wait ready");
    otk_loss_cfg c2 = *cfg;
    c2.accumulate_stats = 1;
    c2.num_adv = num_traj;  // adv_host holds num_traj advantages
    st = otk_policy_loss_fwd_bwd(ctx, std::max<int64_t>(n, 0), vocab, ld, dtype, sb,
                                 reinterpret_cast<const int32_t*>(sb + off_tg),
                                 reinterpret_cast<const uint8_t*>(sb + off_m),
                                 reinterpret_cast<const int32_t*>(sb + off_rt), d_adv,
                                 reinterpret_cast<const float*>(sb + off_old),
                                 has_ref ? reinterpret_cast<const float*>(sb + off_ref) : nullptr, d_nl, &c2,
                                 sb + off_dl, nullptr, nullptr, d_stats, reinterpret_cast<otk_stream_t>(xs));
    if (st != OTK_OK) return st;
    if (dlogits_host && n > 0) {
      // columns [0, vocab) only (the padding of a host row is never written); with zero_masked_rows = 0 only the
      // runs of trainable rows come back, so masked rows of the host buffer stay untouched (otk.h)
      const size_t wb = size_t(vocab) * es;
      for (int64_t a = 0; a < n;) {
        if (!cfg->zero_masked_rows)
          while (a < n && !loss_mask_host[r0 + a]) ++a;
        int64_t e = a;
        while (e < n && (cfg->zero_masked_rows || loss_mask_host[r0 + e])) ++e;
        if (e > a)
          OTK_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(dlogits_host) + size_t(r0 + a) * row_bytes, row_bytes,
                                     sb + off_dl + size_t(a) * row_bytes, row_bytes, wb, size_t(e - a),
                                     cudaMemcpyDeviceToHost, xs),
                   "D2H dlogits");
        a = e;
      }
    }
    OTK_CUDA(cudaEventRecord(ctx->ev[2 + b], xs), "record free");
    if (num_rows == 0) break;
  }
  OTK_CUDA(cudaMemcpyAsync(stats_host, d_stats, sizeof(otk_loss_stats), cudaMemcpyDeviceToHost, xs), "D2H stats");
  OTK_CUDA(cudaStreamSynchronize(xs), "sync exec");
  // the call is blocking, so it reports the device-side data errors of its own launches (sticky word) itself
  return otk_ctx_check(ctx, reinterpret_cast<otk_stream_t>(xs));
}

}  // extern "C"
