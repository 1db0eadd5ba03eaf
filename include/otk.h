/*
 * otk.h — C ABI of the OpenTinker (arxiv 2601.07376) policy-gradient hot path on B200 (sm_100a).
 *
 * The paper's Task Server runs every RL job's update in "forward inference (fwd)" and "parameter
 * updates" resource pools (caption of Fig. mas-framework). BASELINE.json's north_star
 * names the computation those pools run; each step is one entry point here:
 *
 *   (1) otk_build_masks          loss/response masks from FSM-labelled segments
 *   (2) otk_group_advantages     GRPO group-relative advantages
 *   (2') otk_turn_returns        turn-level credit: reward-to-go per ACTION turn
 *   (3) otk_logprob_entropy_fwd  fused vocab-wide log-softmax + gather + entropy  north_star (3)
 *   (4) otk_policy_loss_fwd_bwd  PPO-clip + KL surrogate, token-mean, fused       north_star (4)
 *                                backward dlogits = coef * (softmax - onehot)
 *   LM head fused with (3) (NEXT-1, fwd): otk_lmhead_logprob_fwd — tcgen05 GEMM + log-softmax epilogue
 *   LM head fused with (4) (NEXT-1, fwd + bwd): otk_lmhead_policy_loss_fwd_bwd — loss, dh, dW; the
 *                                dlogits exist only as SMEM tiles inside the backward tcgen05 GEMMs
 *   rollout sampling (NEXT-3): otk_sample_tokens — softmax / greedy token per row
 *   batch sharding over NCCL: otk_comm_* and otk_batch_* — the three exchanges of a
 *       batch-sharded step (global token count, group statistics, loss statistics).
 *   vocab sharding (north_star "vocab-sharding logits with an all-reduce of row max and sum-exp"):
 *       otk_row_partials → (caller all-gathers partials) → otk_logprob_entropy_combine /
 *       otk_policy_loss_fwd_bwd_partials; or, fused: otk_policy_loss_fwd_bwd_vpf (the exchange runs inside
 *       the kernel over NVLink peer memory, one read of the shard).
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless stated otherwise. All buffers are caller-owned; the library
 *    never allocates on the hot path (the ctx owns a small scratch area, the sticky error word and the
 *    staging buffers of the host-buffer entry point).
 *  - Every call is asynchronous on `stream` (a cudaStream_t), performs no host synchronisation, and is
 *    CUDA-graph capturable (except otk_ctx_check and otk_policy_loss_fwd_bwd_host).
 *  - Host-checkable errors (NULL pointers, sizes, alignment, dtype, empty batch) return immediately and
 *    launch nothing. Data-dependent errors (segment lengths, unterminated trajectory, group id or target
 *    out of range) set the ctx's sticky device error word; the offending rows / trajectories are then
 *    treated as loss-masked so kernels stay memory-safe; otk_ctx_check reports the first such error.
 *  - Outputs never alias inputs. A ctx may be used from one stream at a time (its scratch is shared).
 *  - num_rows == 0 is valid: per-row arrays may then be NULL and nothing is launched, except by
 *    otk_policy_loss_fwd_bwd, which still writes its (zero) stats unless cfg->accumulate_stats.
 *  - Layout: logits / dlogits are row-major [num_rows, ld] with ld >= vocab and ld * sizeof(dtype) a
 *    multiple of 16 bytes, base pointer 16-byte aligned. Row j's logits score target j (the caller
 *    shifts; R7). Only columns [0, vocab) are read or written.
 */
#ifndef OTK_H_
#define OTK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTK_VERSION 100 /* 0.1.0 */

typedef struct CUstream_st* otk_stream_t; /* identical to cudaStream_t; NULL = legacy default stream */

typedef enum {
  OTK_OK = 0,
  OTK_ERR_INVALID_ARG = 1,   /* NULL pointer, bad flag, bad config value                   */
  OTK_ERR_SHAPE = 2,         /* negative / inconsistent sizes, vocab larger than supported  */
  OTK_ERR_ALIGNMENT = 3,     /* logits/dlogits base or row stride not 16-byte aligned       */
  OTK_ERR_DTYPE = 4,         /* unknown otk_dtype                                           */
  OTK_ERR_EMPTY_GROUP = 5,   /* num_traj < 1 (SPEC.md:324 EmptyGroup)                      */
  OTK_ERR_UNTERMINATED = 6,  /* terminated[b] == 0 (SPEC.md:324 UnterminatedTrajectory)     */
  OTK_ERR_BAD_TRAJECTORY = 7,/* segment lengths/sources inconsistent with the row count     */
  OTK_ERR_TARGET_RANGE = 8,  /* target outside [0, vocab_total)                             */
  OTK_ERR_CUDA = 9,          /* a CUDA runtime call failed (see otk_last_error)             */
  OTK_ERR_GROUP_RANGE = 10,  /* group_id outside [0, num_groups)                            */
  OTK_ERR_PEER_TIMEOUT = 11, /* K4-VPF: a peer rank's row partial did not arrive in time     */
  OTK_ERR_NCCL = 12,         /* NCCL could not be loaded or a collective failed (otk_last_error) */
  OTK_ERR_NO_COMM = 13       /* a batch-sharded call on a ctx without otk_comm_init            */
} otk_status;

typedef enum { OTK_SRC_CONTEXT = 0, OTK_SRC_ACTION = 1, OTK_SRC_OBSERVATION = 2, OTK_SRC_PAD = 3 } otk_source;
typedef enum { OTK_F32 = 0, OTK_BF16 = 1 } otk_dtype;
typedef enum { OTK_KL_K1 = 1, OTK_KL_K2 = 2, OTK_KL_K3 = 3 } otk_kl_type;
/* loss = sum_j w_j L_j with w_j = m_j / N (token mean), m_j / (n_b B) (mean over trajectories of the
 * per-trajectory token mean) or m_j / B (mean over trajectories of the token sum); n_b = loss tokens of
 * row j's trajectory, B = trajectories with n_b > 0 (global). DESIGN.md R17, R29. */
typedef enum { OTK_TOKEN_MEAN = 0, OTK_SEQ_MEAN_TOKEN_MEAN = 1, OTK_SEQ_MEAN_TOKEN_SUM = 2 } otk_reduction;

#define OTK_ANY_AGENT (-1)
#define OTK_ADV_STD_NORM 0x1u /* divide by the group std (default on)        */
#define OTK_ADV_UNBIASED 0x2u /* std with n-1 instead of n (R2; default off)    */
#define OTK_ADV_SKIP_UNGROUPED 0x4u /* group_id < 0: no group, A = 0, no error (turn-level credit) */

/* ---------------------------------------------------------------------------------------------
 * Context. Owns: the device index, SM count, a sticky device error word, O(#SM) scratch for the
 * deterministic reductions, and (lazily, on first use of the host entry point) staging buffers.
 * ------------------------------------------------------------------------------------------- */
typedef struct otk_ctx otk_ctx;

otk_status otk_ctx_create(int cuda_device, otk_ctx** out);
otk_status otk_ctx_destroy(otk_ctx* ctx);
/* Synchronises `stream`, returns (and clears) the first device-side data error since the last check. */
otk_status otk_ctx_check(otk_ctx* ctx, otk_stream_t stream);
const char* otk_status_string(otk_status s);
const char* otk_last_error(void); /* thread-local detail of the last host-side error */
int otk_version(void);

/* ---------------------------------------------------------------------------------------------
 * (1) Masks — PAPER.md §2.2 (lines 167-174): PENDING (context) tokens "are excluded from loss
 * computation"; only GENERATING (action) tokens "are marked as trainable"; INTERACTING (observation)
 * tokens "are masked from the loss". PAPER.md:192: "Model parameters and gradients are not shared
 * across agents", so an ACTION row is trainable only for the agent that emitted it.
 *
 * One trajectory = a list of segments (SPEC.md:37-50 Segment{source, tokens}) packed into rows
 * [tok_offsets[b], tok_offsets[b+1]) of the batch, in order.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t num_traj;             /* B >= 1, else OTK_ERR_EMPTY_GROUP                                */
  int64_t num_rows;             /* N = tok_offsets[B] (host copy; checked on device)               */
  const int64_t* tok_offsets;   /* [B+1] row offsets, tok_offsets[0] = 0, non-decreasing           */
  const int32_t* seg_offsets;   /* [B+1] offsets into the segment arrays                          */
  const uint8_t* seg_source;    /* [S] otk_source                                                  */
  const int16_t* seg_agent;     /* [S] emitting agent of an ACTION segment (ignored otherwise)     */
  const int32_t* seg_len;       /* [S] > 0; a trajectory's lengths sum to its row count            */
  const uint8_t* terminated;    /* [B] or NULL (= all terminated); 0 => OTK_ERR_UNTERMINATED        */
  const int16_t* traj_agent;    /* [B] or NULL: agent trained on trajectory b (overrides train_agent) */
} otk_traj_batch;

/*
 * Outputs (device): loss_mask[N] u8 = (src == ACTION) && (agent matches); response_mask[N] u8 (NULL ok)
 * = every non-PAD row outside the trajectory's leading CONTEXT segment (R13);
 * row_traj[N] i32 = b; traj_loss_tokens[B] i64; traj_source_counts[B*4] i64 (NULL ok; SPEC.md:408-416
 * mask_report, order CONTEXT, ACTION, OBSERVATION, PAD); n_loss[1] i64 = sum of loss_mask (this batch;
 * a batch-sharded caller all-reduces it to the global token count before step (4)); n_active_traj[1]
 * (NULL ok) = trajectories with >= 1 loss token; row_seg[N] i32 (NULL ok) = global index of the row's
 * segment (-1 for rows of an invalid trajectory).
 * Rows of an invalid trajectory get loss_mask 0 and the error word is set. Bit-exact.
 */
otk_status otk_build_masks(otk_ctx* ctx, const otk_traj_batch* batch /* host struct, device arrays */,
                           int16_t train_agent, uint8_t* loss_mask, uint8_t* response_mask, int32_t* row_traj,
                           int64_t* traj_loss_tokens, int64_t* traj_source_counts, int64_t* n_loss,
                           int64_t* n_active_traj /* [1] or NULL: trajectories with >= 1 loss token */,
                           int32_t* row_seg /* [N] or NULL: global segment index of each row (turn-level credit) */,
                           otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * (2) Group-relative advantages — PAPER.md:177 ("rewards are associated with the corresponding action
 * tokens"), SPEC.md:95 (return = undiscounted sum of per-turn scores), SPEC.md:323:
 *   A_b = (R_b - mean_g) / (std_g if std_g > std_floor else 1)   (flags & OTK_ADV_STD_NORM)
 *   A_b =  R_b - mean_g                                         (otherwise)
 * over the trajectories b' with group_id[b'] == group_id[b]; std is the population std unless
 * OTK_ADV_UNBIASED (std = 0 for groups of size <= 1). Sums run in trajectory order, float64.
 * Returns come either from returns[B] or from per-turn scores (turn_offsets[B+1], turn_rewards[...]):
 * exactly one of `returns` and `turn_offsets` must be non-NULL. A batch-sharded caller passes the
 * all-gathered (group_id, return) arrays of all ranks, so every rank computes identical statistics.
 * Outputs: adv[B] f64; returns_out[B], group_mean[G], group_std[G] f64, group_size[G] i32 (NULL ok).
 * Tolerance vs the float64 oracle: 1e-6 abs (north_star). Out-of-range group ids set
 * OTK_ERR_GROUP_RANGE and give A = 0 for that trajectory.
 * ------------------------------------------------------------------------------------------- */
otk_status otk_group_advantages(otk_ctx* ctx, int32_t num_traj, const int32_t* group_id, int32_t num_groups,
                                const double* returns, const int32_t* turn_offsets, const double* turn_rewards,
                                uint32_t flags, double std_floor, double* adv, double* returns_out,
                                double* group_mean, double* group_std, int32_t* group_size, otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * (2') Turn-level credit (R31). PAPER.md:177 "rewards are associated
 * with the corresponding action tokens"; SPEC.md:95 stores one score per turn, SPEC.md:364 lists
 * discounting as the extension. Turn k of trajectory b is its k-th trainable ACTION segment (source
 * ACTION, agent = traj_agent[b] or train_agent, as in (1)); its return is the discounted reward-to-go
 *   G_{b,k} = sum_{j=k}^{R_b-1} gamma^(j-k) r_{b,j}     (r_{b,.} = turn_rewards[turn_offsets[b] ..]; 0 if k >= R_b)
 * Outputs per segment s (device, [num_segments] = seg_offsets[B]): seg_return[s] f64 = G of the turn
 * (0 otherwise), seg_group[s] i32 = group_id[b] for a turn, -1 otherwise. The advantages then come
 * from otk_group_advantages(num_traj = num_segments, group_id = seg_group, returns = seg_return,
 * flags | OTK_ADV_SKIP_UNGROUPED), and step (4) reads them per row with cfg->adv_index = row_seg.
 * gamma in [0, 1]. A negative group_id or seg_offsets[B] != num_segments sets the error word.
 * Tolerance vs oracle: 1e-12 relative (float64, Horner order).
 * ------------------------------------------------------------------------------------------- */
otk_status otk_turn_returns(otk_ctx* ctx, const otk_traj_batch* batch /* host struct, device arrays */,
                            int32_t num_segments, int16_t train_agent, const int32_t* group_id,
                            const int32_t* turn_offsets, const double* turn_rewards, double gamma,
                            double* seg_return, int32_t* seg_group, otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * (3) Forward: per row j with row_mask[j] != 0 (row_mask NULL = all rows), z = logit_scale * x:
 *   M = max_v z_v, S = sum_v e^{z_v - M}, lse = M + ln S, logp_j = z_{y_j} - lse,
 *   entropy_j = ln S - sum_v e^{z_v - M}(z_v - M) / S.
 * logits: [num_rows, ld] of dtype (bf16 or fp32); targets[num_rows] i32 in [0, vocab).
 * Outputs logp / entropy / lse [num_rows] f32 (entropy, lse may be NULL); masked rows get 0.
 * fp32 accumulation, one HBM read of each logit. Tolerance vs oracle: 2e-3 abs (bf16), 1e-5 (fp32).
 * logit_scale > 0 (= 1/temperature, R19).
 * ------------------------------------------------------------------------------------------- */
otk_status otk_logprob_entropy_fwd(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                                   const void* logits, const int32_t* targets, const uint8_t* row_mask,
                                   float logit_scale, float* logp, float* entropy, float* lse,
                                   otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * (4) Loss forward + fused backward. Per row j (A = adv[row_traj[j]], m = loss_mask[j], N = *n_loss):
 *   delta = clamp(logp - old, -C, C), r = e^delta, rbar = clamp(r, 1 - clip_low, 1 + clip_high)
 *   pg = max(-A r, -A rbar); clipped <=> (A > 0 && r > 1 + clip_high) || (A < 0 && r < 1 - clip_low)
 *   KL: k3 = e^d - d - 1, d = clamp(ref - logp, -C, C); k1 = logp - ref; k2 = (logp - ref)^2 / 2
 *   L_j = pg + kl_beta * KL - ent_coef * H_j;   loss = sum_j w_j L_j  (w_j = m_j / N: token mean over the
 *   GLOBAL batch, R17; or a sequence-mean reduction, see otk_reduction)
 *   dlogits[j, v] = coef_j * (softmax_jv - [v == y_j]) + w_j ent_coef s p_jv (ln p_jv + H_j),
 *   coef_j = -s * w_j * dL_j/dlogp_j  (dual clip / SFT variants: see otk_loss_cfg)
 * with dL/dlogp = (clipped or |logp - old| > C ? 0 : -A r) + beta * (k3: |ref-logp| > C ? 0 : 1 - e^d;
 * k1: 1; k2: logp - ref). old/ref are detached constants; ref_logp may be NULL iff kl_beta == 0.
 * n_loss is a DEVICE pointer (never read on the host). Rows with m == 0: dlogits row = 0 if
 * cfg->zero_masked_rows (else untouched), logp = entropy = 0; they are not read (write-only rows).
 * stats (device): accumulated (+=) when cfg->accumulate_stats, else overwritten; reduced in a fixed
 * order (deterministic, no float atomics). A step over several micro-batches sets accumulate_stats = 0
 * on the first call. dlogits has the logits' dtype and layout and must not alias them.
 * Tolerances vs oracle: loss 1e-4 relative (R22), dlogits |d| <= 2^-7 |ref| + 1e-5 |coef_j| (bf16).
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  double clip_low;          /* epsilon_low, default 0.2  (R14) */
  double clip_high;         /* epsilon_high, default 0.2                  */
  double kl_beta;           /* beta, default 0.04; 0 disables KL and ref  */
  double log_ratio_clamp;   /* C, default 20 (R15)                         */
  double logit_scale;       /* s = 1/temperature > 0, default 1 (R19)      */
  int32_t kl_type;          /* otk_kl_type, default OTK_KL_K3 (R16)        */
  int32_t zero_masked_rows; /* default 1                                   */
  int32_t accumulate_stats; /* default 0                                   */
  int32_t reserved;         /* must be 0                                   */
  /* A4 variants (R27-R30) */
  double ent_coef;          /* entropy bonus c_H: L -= c_H * H, dlogits += w c_H s p (ln p + H); default 0 */
  double dual_clip;         /* c > 1: loss of A < 0 tokens capped at -c*A (zero gradient); 0 = off     */
  int32_t reduction;        /* otk_reduction, default OTK_TOKEN_MEAN                                   */
  int32_t sft;              /* 1: supervised L = -logp (A, old_logp and the clip unused)   */
  const int64_t* traj_loss_tokens; /* device [B]: loss tokens per trajectory (seq-mean reductions)     */
  const int64_t* n_active_traj;    /* device [1]: trajectories with >= 1 loss token, global (seq-mean) */
  const int32_t* adv_index;        /* device [num_rows] or NULL: A_j = adv[adv_index[j]] instead of
                                      adv[row_traj[j]] (turn-level credit: row_seg + segment advantages) */
  int64_t num_adv;                 /* elements of adv (>= 1 when num_rows > 0): a row whose index into adv
                                      (row_traj[j] or adv_index[j]) is outside [0, num_adv) sets
                                      OTK_ERR_GROUP_RANGE and is treated as loss-masked (memory-safe)      */
  int64_t num_traj;                /* elements of traj_loss_tokens (sequence-mean reductions; row_traj[j]
                                      outside [0, num_traj) is a GROUP_RANGE data error as above)         */
} otk_loss_cfg;

typedef struct {
  double loss;        /* sum_j m_j L_j / N                     */
  double n_clipped;   /* number of trainable rows with clipping */
  double kl_sum;      /* sum_j m_j KL_j                         */
  double entropy_sum; /* sum_j m_j H_j                          */
  double n_tokens;    /* number of trainable rows seen          */
} otk_loss_stats;

otk_status otk_policy_loss_fwd_bwd(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                                   const void* logits, const int32_t* targets, const uint8_t* loss_mask,
                                   const int32_t* row_traj, const double* adv, const float* old_logp,
                                   const float* ref_logp, const int64_t* n_loss, const otk_loss_cfg* cfg,
                                   void* dlogits, float* logp, float* entropy, otk_loss_stats* stats,
                                   otk_stream_t stream);

/* Same computation as otk_policy_loss_fwd_bwd but every array argument is a HOST pointer (pinned
 * memory recommended): rows are streamed through ctx-owned device staging buffers in chunks, with the
 * host->device copies of chunk k+1 overlapping the kernel on chunk k. Only the logits rows with
 * loss_mask != 0 are copied (runs of consecutive rows, one copy each): a masked row is never read.
 * dlogits_host ([num_rows, ld], same dtype) may be NULL (the gradient is then computed on the device and
 * discarded). Otherwise columns [0, vocab) of its rows are written: every row when cfg->zero_masked_rows
 * (masked rows get zeros), else only the trainable rows (masked rows stay untouched, and only the trainable
 * rows' gradients cross PCIe — pre-zero the buffer once to hold the complete gradient). stats_host receives
 * the result. Token-mean reduction only; cfg->adv_index must be NULL. Blocking: returns after the
 * stats and dlogits have been copied back, with the first device-side data error of this call (as
 * otk_ctx_check would report it; the sticky word is cleared). Used to measure the end-to-end (e2e) metric. */
otk_status otk_policy_loss_fwd_bwd_host(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld,
                                        otk_dtype dtype, const void* logits_host, const int32_t* targets_host,
                                        const uint8_t* loss_mask_host, const int32_t* row_traj_host,
                                        int32_t num_traj, const double* adv_host, const float* old_logp_host,
                                        const float* ref_logp_host, int64_t n_loss, const otk_loss_cfg* cfg,
                                        void* dlogits_host, otk_loss_stats* stats_host, int64_t rows_per_chunk);

/* ---------------------------------------------------------------------------------------------
 * Vocab sharding. A rank holds columns [vocab_start, vocab_start + vocab_local) of every row, with
 * global targets. otk_row_partials writes per row (m2, s, t2, w) as 4 floats: m2 = a reference max of
 * y = log2(e) * s * x over the shard, s = sum 2^{y - m2}, t2 = sum 2^{y - m2}(y - m2), and w = y_target - m2
 * if the target column is in the shard, else -inf (rows with row_mask 0: (-inf, 0, 0, -inf)). The caller
 * all-gathers them into [nshards][num_rows][4] (rank order); the combine (R25) is exact
 * rescaling in rank order, identical on all ranks.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int64_t vocab_start; /* first global column held by this rank */
  int64_t vocab_total; /* global vocabulary (targets are checked against it) */
} otk_vocab_shard;

otk_status otk_row_partials(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld, otk_dtype dtype,
                            const void* logits, const int32_t* targets, const uint8_t* row_mask,
                            const otk_vocab_shard* shard, float logit_scale, float* partials, otk_stream_t stream);

otk_status otk_logprob_entropy_combine(otk_ctx* ctx, int64_t num_rows, int32_t nshards, const float* partials,
                                       const uint8_t* row_mask, float* logp, float* entropy, float* lse,
                                       otk_stream_t stream);

/* (4) on a vocab shard: the row statistics come from the all-gathered partials; this rank writes the
 * dlogits of its columns. loss/stats are the global values on every rank. */
otk_status otk_policy_loss_fwd_bwd_partials(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld,
                                            otk_dtype dtype, const void* logits, const int32_t* targets,
                                            const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                            const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                            const otk_loss_cfg* cfg, const otk_vocab_shard* shard,
                                            int32_t nshards, const float* partials, void* dlogits, float* logp,
                                            float* entropy, otk_loss_stats* stats, otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * (4) on a vocab shard with the exchange fused into the kernel (K4-VPF; SURVEY.md §8(e) VOCAB row,
 * DESIGN.md §7). Same result as otk_row_partials -> all-gather -> otk_policy_loss_fwd_bwd_partials
 * (logp / entropy bitwise equal; loss stats up to fp64 summation order; dlogits within the bf16 tolerance of
 * (4)), but in ONE launch
 * per rank and ONE read of the shard: after pass 1 of a row, the CTA pushes the row's 16-byte partial
 * (m2, s, t2, w — the otk_row_partials form) into every peer's exchange buffer over NVLink (P2P stores of
 * four 64-bit words, each = value | call epoch << 32, so every word validates itself and no memory fence
 * is needed), waits until the peers' words of the same row carry this call's epoch,
 * combines them in rank order (identical on every rank) and runs pass 2 from the tensor-memory-resident
 * exponentials. The all-reduce of row max / sum-exp the north_star names is this exchange.
 * logits / dlogits: this rank's column shard [num_rows, vocab_local] with row stride ld (e.g. a column slice of
 * a wider row buffer); every other argument as in otk_policy_loss_fwd_bwd_partials (targets global).
 *   rank, nranks: this rank's index in rank order (= shard order) and the number of ranks (<= 8).
 *   rows_cap  : the row capacity the exchange buffers were sized for (the same value on every call on them).
 *   xchg[q]   : device pointer, valid in THIS process, to rank q's exchange buffer (xchg[rank] = own
 *               buffer; peers' buffers mapped with otk_ipc_open, or plain buffers of the same device when
 *               several ranks share one GPU), each otk_vpf_xchg_bytes(rows_cap, nranks) bytes, 16-byte
 *               aligned, ZEROED once before the first call and then owned by the library's calls.
 *   (epoch)   : the call's tag = 1 + the calls completed on this buffer set, kept in the own buffer's tail
 *               by the kernel itself (its last CTA bumps it), so calls may be captured in a CUDA graph and
 *               replayed; all ranks must issue the same sequence of calls (lockstep).
 *   max_ctas  : 0 = one CTA per SM; otherwise at most this many CTAs (lets several ranks share a GPU).
 * Every rank must make the same sequence of calls with the same num_rows / masks / targets; a partial that
 * does not arrive within ~20 s sets OTK_ERR_PEER_TIMEOUT (sticky; later waits give up at once) instead of
 * hanging. Host-checked (nothing launched): ctx / shard / peers / required arrays NULL, rank / nranks out of range,
 * num_rows > rows_cap, an xchg pointer NULL or not 16-byte aligned, max_ctas below the cluster size, dlogits
 * aliasing logits (OTK_ERR_INVALID_ARG / OTK_ERR_SHAPE / OTK_ERR_ALIGNMENT).
 * ------------------------------------------------------------------------------------------- */
#define OTK_VPF_MAX_RANKS 8
typedef struct {
  int32_t rank;
  int32_t nranks;
  int64_t rows_cap;
  void* xchg[OTK_VPF_MAX_RANKS];
  int32_t max_ctas;
} otk_vpf_peers;

int64_t otk_vpf_xchg_bytes(int64_t rows_cap, int32_t nranks); /* -1: bad args */
otk_status otk_policy_loss_fwd_bwd_vpf(otk_ctx* ctx, int64_t num_rows, int64_t vocab_local, int64_t ld,
                                       otk_dtype dtype, const void* logits, const int32_t* targets,
                                       const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                       const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                       const otk_loss_cfg* cfg, const otk_vocab_shard* shard,
                                       const otk_vpf_peers* peers /* host struct */, void* dlogits, float* logp,
                                       float* entropy, otk_loss_stats* stats, otk_stream_t stream);

/* K4-VPF ranks EMULATED on one GPU in ONE launch (single-GPU tests, smoke and bench only; a real multi-GPU job
 * makes one otk_policy_loss_fwd_bwd_vpf call per rank). calls[k] is rank k's call: its own ctx (distinct per
 * rank: scratch and ticket), column shard, exchange view (peers->rank == k, peers->nranks == nranks) and outputs;
 * the row-side arrays are shared. The launch hosts every rank's CTAs (the SMs split evenly between the ranks,
 * one CTA per SM) and is cooperative — all CTAs are resident at once, so the in-kernel exchange never waits on an
 * unscheduled rank (separate launches on separate streams carry no such guarantee, and a profiler serialising
 * them would time out). Returns OTK_ERR_CUDA if the grid cannot be co-resident. Same results, bit for bit, as
 * the per-rank calls. Counts as one launch on calls[0].ctx. */
typedef struct {
  otk_ctx* ctx;
  int64_t vocab_local;
  const void* logits;             /* this rank's shard [num_rows, vocab_local], row stride ld */
  otk_vocab_shard shard;
  const otk_vpf_peers* peers;
  void* dlogits;                  /* [num_rows, vocab_local], row stride ld */
  float* logp;                    /* [num_rows] or NULL */
  float* entropy;                 /* [num_rows] or NULL */
  otk_loss_stats* stats;          /* device */
} otk_vpf_rank_call;
otk_status otk_policy_loss_fwd_bwd_vpf_group(int32_t nranks, const otk_vpf_rank_call* calls, int64_t num_rows,
                                             int64_t ld, otk_dtype dtype, const int32_t* targets,
                                             const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                             const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                             const otk_loss_cfg* cfg, otk_stream_t stream);

/* Exchange buffers and their CUDA IPC plumbing (setup, not the hot path). otk_xchg_alloc: a zeroed device
 * buffer of `bytes` on the ctx's device (its own cudaMalloc allocation, so an IPC handle maps exactly it);
 * free with otk_xchg_free. For ranks on different GPUs of one node: otk_ipc_get_handle (cudaIpcGetMemHandle)
 * gives 64 opaque bytes the caller exchanges (e.g. an all-gather over torch.distributed); otk_ipc_open
 * (cudaIpcOpenMemHandle, peer access enabled) maps a peer's buffer into this process; otk_ipc_close unmaps. */
#define OTK_IPC_HANDLE_BYTES 64
otk_status otk_xchg_alloc(otk_ctx* ctx, int64_t bytes, void** dev_ptr_out);
otk_status otk_xchg_free(otk_ctx* ctx, void* dev_ptr);
otk_status otk_ipc_get_handle(const void* dev_ptr /* from otk_xchg_alloc */, void* handle_out /* 64 B, host */);
otk_status otk_ipc_open(const void* handle /* host */, void** dev_ptr_out);
otk_status otk_ipc_close(void* dev_ptr);

/* ---------------------------------------------------------------------------------------------
 * Rollout-side token sampling (R32). PAPER.md:170-171 GENERATING
 * ("generates tokens autoregressively"); SPEC.md:300-306 sample_token: a draw from softmax(s x),
 * s = logit_scale = 1/temperature, returned with its probability; SPEC.md:309-318 greedy_token.
 *   greedy == 0: tokens[j] = min{ t : sum_{v <= t} p_jv > u_j },  p_j = softmax(s x_j),  u_j = uniforms[j]
 *                (inverse transform; the caller draws u_j in [0, 1) — out-of-range u sets
 *                OTK_ERR_INVALID_ARG in the error word and is clamped);
 *   greedy == 1: tokens[j] = argmax_v x_jv, ties to the lowest id (uniforms may be NULL).
 * logp[j] (NULL ok) = log p_j(tokens[j]). A row whose logits are all -inf gives token 0, logp -inf.
 * Greedy with logp == NULL computes no exponentials (a pure max pass over the row).
 * logits: [num_rows, ld] bf16 / fp32, 16-byte aligned rows; tokens[num_rows] i32 (device).
 * One HBM read of each logit (the re-reads of pass 2/3 hit L2). Parity: greedy bit-exact; a sampled
 * token is exact unless u_j lies within 2e-5 of a cdf boundary, where either neighbour is accepted.
 * ------------------------------------------------------------------------------------------- */
otk_status otk_sample_tokens(otk_ctx* ctx, int64_t num_rows, int64_t vocab, int64_t ld, otk_dtype dtype,
                             const void* logits, const float* uniforms, float logit_scale, int32_t greedy,
                             int32_t* tokens, float* logp, otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * LM head fused with step (3) (forward half; R33). The fwd pool
 * evaluates log-probs from the policy's final hidden states: z_j = s * h_j W^T, then
 * (3) on z_j, without writing the [num_rows, vocab] logits to memory:
 *   logp_j = z_{j,y_j} - lse_j,  entropy_j = lse_j - sum_v p_jv z_jv,  lse_j = log sum_v e^{z_jv}.
 * hidden: [num_rows, hidden_dim] bf16 row-major; weight: [vocab, hidden_dim] bf16 row-major (the LM-head
 * matrix as stored by an nn.Linear(hidden_dim, vocab)); hidden_dim a multiple of 64; base pointers
 * 16-byte aligned. GEMM on the tcgen05 tensor cores with fp32 accumulation in TMEM; the log-softmax
 * statistics are folded in the epilogue. workspace: device scratch of otk_lmhead_workspace_bytes()
 * bytes (per-row partials of each vocab chunk), caller-owned. Outputs as in (3) (row_mask NULL = all
 * rows; masked rows get 0). A target outside [0, vocab) on an unmasked row sets OTK_ERR_TARGET_RANGE
 * (that row's logp is -inf). Tolerance vs the float64 oracle on the same bf16 h and W: 2e-3 abs.
 * ------------------------------------------------------------------------------------------- */
int64_t otk_lmhead_workspace_bytes(const otk_ctx* ctx, int64_t num_rows, int64_t vocab); /* -1: bad args */
otk_status otk_lmhead_logprob_fwd(otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab,
                                  const void* hidden, const void* weight, const int32_t* targets,
                                  const uint8_t* row_mask, float logit_scale, void* workspace,
                                  int64_t workspace_bytes, float* logp, float* entropy, float* lse,
                                  otk_stream_t stream);

/* Vocab-sharded LM head (tensor-parallel head: this rank holds rows [vocab_start, vocab_start + vocab_local)
 * of W, targets are global): writes this rank's per-row partials (m2, s, t2, w) — the otk_row_partials form —
 * for the caller to all-gather into [nshards][num_rows][4] (rank order) and finish with
 * otk_logprob_entropy_combine. workspace: otk_lmhead_workspace_bytes(ctx, num_rows, vocab_local) bytes. */
otk_status otk_lmhead_row_partials(otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab_local,
                                   const void* hidden, const void* weight, const int32_t* targets,
                                   const uint8_t* row_mask, const otk_vocab_shard* shard, float logit_scale,
                                   void* workspace, int64_t workspace_bytes, float* partials, otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * Policy loss and its gradients THROUGH the LM head (both halves; PAPER.md:188,
 * the "parameter updates" pool; DESIGN.md §6 "LM head, backward"). With x = h W^T (bf16 logits) and
 * (4) on x with cfg->logit_scale = s:
 *   loss / stats / logp / entropy  exactly as otk_policy_loss_fwd_bwd on the bf16-rounded x,
 *   dhidden = dx W   [num_rows, hidden_dim] bf16,    dweight = dx^T h   [vocab, hidden_dim] bf16,
 * where dx = dL/dx (the dlogits of (4)) is formed tile by tile inside the two backward tcgen05 GEMMs from
 * x and four per-row constants — it is never written to memory. Three tensor-core GEMMs (x, dh, dW) and
 * two small kernels (chunk-partial combine + loss terms; dh split-K reduction), in this stream order.
 * hidden: [num_rows, hidden_dim] bf16, weight: [vocab, hidden_dim] bf16 (row-major, 16-byte aligned; dhidden,
 * dweight and workspace 32-byte aligned: the epilogues write whole 32-byte sectors);
 * hidden_dim a multiple of 64; vocab a multiple of 8 (16-byte rows of x). targets, loss_mask, row_traj,
 * adv, old_logp, ref_logp, n_loss, cfg as in otk_policy_loss_fwd_bwd (token-mean or sequence-mean
 * reductions, all A4 variants; targets global ids in [0, vocab)).
 * workspace: otk_lmhead_loss_workspace_bytes() bytes, 16-byte aligned, caller-owned: x rounded to bf16 (RNE)
 * in 64 x 64 tiles [rows_pad/64][cols_pad/64][64][64] (rows_pad, cols_pad = num_rows, vocab rounded up to 256;
 * contiguous 8 KB tiles for the backward's TMA), then chunk partials, per-row constants, dh split-K partials. dhidden / dweight: outputs, bf16, must not alias any input. logp / entropy: NULL or
 * [num_rows] f32 (loss-masked rows 0). stats: device otk_loss_stats (accumulated if cfg->accumulate_stats).
 * num_rows == 0: dweight is zeroed and the stats written as zeros (unless accumulate_stats); nothing else runs.
 * Errors: host-checkable ones return at once; a target out of range sets OTK_ERR_TARGET_RANGE and an index
 * out of range OTK_ERR_GROUP_RANGE (those rows are treated as loss-masked: zero gradient).
 * Tolerance vs the float64 oracle on the same bf16 h and W (tests/test_gpu_lmhead_loss.py): loss 1e-3
 * relative; dh, dW element-wise 2^-8 |ref| + 6 * 2^-8 * sqrt(sum_v (dx_jv W_vi)^2).
 * ------------------------------------------------------------------------------------------- */
int64_t otk_lmhead_loss_workspace_bytes(const otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim,
                                        int64_t vocab); /* -1: bad args */
otk_status otk_lmhead_policy_loss_fwd_bwd(otk_ctx* ctx, int64_t num_rows, int64_t hidden_dim, int64_t vocab,
                                          const void* hidden, const void* weight, const int32_t* targets,
                                          const uint8_t* loss_mask, const int32_t* row_traj, const double* adv,
                                          const float* old_logp, const float* ref_logp, const int64_t* n_loss,
                                          const otk_loss_cfg* cfg, void* workspace, int64_t workspace_bytes,
                                          void* dhidden, void* dweight, float* logp, float* entropy,
                                          otk_loss_stats* stats, otk_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * Batch sharding over NCCL (SURVEY.md §8(b), §8(e) BATCH; PAPER.md:64 and :84 — one job's update spread over
 * the GPUs of the shared cluster): rank r holds a contiguous range of the global batch's trajectories (groups
 * may straddle ranks) and runs (1), (2), (4) on it; three exchanges make the result identical to one GPU's:
 *   otk_build_masks (local)                    -> otk_batch_allreduce_i64(n_loss [, n_active_traj])
 *   returns of the local trajectories          -> otk_batch_group_advantages (all-gather in rank order + (2) on
 *                                                 the whole batch: every rank gets identical group statistics)
 *   otk_policy_loss_fwd_bwd per micro-batch    -> otk_batch_allreduce_f64(stats, 5)
 * The communicator belongs to the ctx (one ctx per rank / GPU). NCCL is bound at the first otk_comm_* call
 * (dlopen of libnccl.so.2, or $OTK_NCCL_LIB; in a PyTorch process the copy torch already loaded), so the
 * library has no link-time NCCL dependency; without NCCL these calls return OTK_ERR_NCCL. Collectives are
 * stream-ordered on `stream`, capturable in a CUDA graph, and must be issued in the same order on every rank.
 * ------------------------------------------------------------------------------------------- */
#define OTK_COMM_ID_BYTES 128
/* Host: a fresh NCCL unique id (on one rank; the caller hands the 128 bytes to every rank). */
otk_status otk_comm_unique_id(unsigned char id[OTK_COMM_ID_BYTES]);
/* Collective over the nranks processes (blocking until all have joined): ctx's device, rank in [0, nranks). */
otk_status otk_comm_init(otk_ctx* ctx, const unsigned char id[OTK_COMM_ID_BYTES], int32_t nranks, int32_t rank);
otk_status otk_comm_destroy(otk_ctx* ctx); /* also done by otk_ctx_destroy; no-op without a communicator */
otk_status otk_comm_size(const otk_ctx* ctx, int32_t* nranks, int32_t* rank); /* OTK_ERR_NO_COMM if none */
/* In place: buf[0, n) = sum over ranks (device int64 / float64). n >= 0. */
otk_status otk_batch_allreduce_i64(otk_ctx* ctx, int64_t* buf, int64_t n, otk_stream_t stream);
otk_status otk_batch_allreduce_f64(otk_ctx* ctx, double* buf, int64_t n, otk_stream_t stream);
/* Step (2) over the global batch. group_id / returns: this rank's [num_traj_local] (device); counts: HOST
 * [nranks] trajectories per rank (counts[rank] == num_traj_local; the shard plan knows them, so no size exchange);
 * gid_all / ret_all: device [B = sum counts], filled with every rank's (group_id, return) in rank order;
 * adv_all [B] and group_mean / group_std [num_groups] f64, group_size [num_groups] i32 (NULL ok): as
 * otk_group_advantages on the whole batch, identical on every rank. This rank's advantages are
 * adv_all + sum(counts[0 .. rank)). */
otk_status otk_batch_group_advantages(otk_ctx* ctx, int32_t num_traj_local, const int32_t* group_id,
                                      const double* returns, const int32_t* counts, int32_t num_groups,
                                      uint32_t flags, double std_floor, int32_t* gid_all, double* ret_all,
                                      double* adv_all, double* group_mean, double* group_std, int32_t* group_size,
                                      otk_stream_t stream);

/* Harness helper (not on the path): number of kernel launches the library issued since ctx creation. */
int64_t otk_ctx_launch_count(const otk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* OTK_H_ */
