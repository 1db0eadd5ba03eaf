// otk_internal.h — the ctx object and the kernel parameter blocks shared by the .cu files.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/otk.h"

struct otk_ctx {
  int device = 0;
  int num_sms = 0;
  int max_smem_optin = 0;
  int* d_err = nullptr;            // sticky device error word (first otk_status != OK wins)
  unsigned int* d_tickets = nullptr;  // [8] last-CTA tickets (one per kernel family)
  double* d_partials = nullptr;    // [kMaxCtas * kStatSlots] per-CTA deterministic partials
  int64_t* d_scratch_i64 = nullptr;  // [kMaxCtas] per-CTA integer partials
  double* d_returns = nullptr;     // [cap_returns] scratch for otk_group_advantages
  int64_t cap_returns = 0;
  // staging for the host entry point (allocated lazily, reused)
  void* stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t exec_stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t launches = 0;
  int sample_occ[4] = {0, 0, 0, 0};  // k_sample resident CTAs per SM (bf16, fp32; x2 register budgets), on first use
  void* comm = nullptr;            // ncclComm_t of the batch-sharded step (otk_comm_init), or none
  int comm_nranks = 0, comm_rank = 0;
};

namespace otk {

otk_status host_fail(otk_status s, const char* msg);   // records otk_last_error's message (otk_api.cu)
void comm_release(otk_ctx* ctx);                        // otk_comm.cu

constexpr int kMaxCtas = 1024;
constexpr int kStatSlots = 8;
enum Ticket { kTicketMasks = 0, kTicketRows = 1 };

// Fused row kernel configuration.
// Warp 0 loads (bulk TMA), warps 1..12 compute (3 per SM sub-partition / TMEM lane quadrant; <= 128
// registers per thread), warp 13 zero-fills masked rows (bulk async stores). A 12 KB chunk is exactly
// 2 x 16-byte vectors per consumer thread.
#ifndef OTK_K4_CW16
constexpr int kChunkBytes = 12288;       // one bulk-TMA transfer / ring slot
constexpr int kSlots = 18;               // ring depth: 216 KB of shared memory per CTA
constexpr int kSlotsFwd = 8;             // FWD / PARTIAL: 96 KB ring, so two CTAs share an SM (twice the warps)
constexpr int kConsumerWarps = 12;       // 384 compute threads
constexpr int kMaxChunks = 18;           // a CTA's row segment (<= 18 chunks, 216 KB) is kept in TMEM (162 columns)
constexpr int kTmemWindow = 168;         // TMEM columns per consumer warp (3 windows per lane quadrant: 504 of 512)
constexpr int kPipeChunks = 7;           // pipelined K4-VPF: <= 7 chunks (84 KB) per CTA, two rows per TMEM window
constexpr int kLag3Chunks = 4;           // pipelined K4-VPF, lag 3: <= 4 chunks, four rows per TMEM window
#else  // experiment: 16 consumer warps (4 per TMEM lane quadrant), 16 KB chunks
constexpr int kChunkBytes = 16384;
constexpr int kSlots = 13;               // 208 KB
constexpr int kSlotsFwd = 6;             // 96 KB
constexpr int kConsumerWarps = 16;
constexpr int kMaxChunks = 14;           // 224 KB segments; 8 x 14 + 14 = 126 of a 128-column window
constexpr int kTmemWindow = 128;
constexpr int kPipeChunks = 7;           // 2 x 64-column slots
constexpr int kLag3Chunks = 3;           // 4 x 32-column slots
#endif
constexpr int kThreads = 32 * (2 + kConsumerWarps);  // + loader warp 0 + zero-fill warp (last)

enum RowMode : int {
  kModeFwd = 0,       // (3): logp / entropy / lse
  kModePartial = 1,   // vocab shard pass 1: per-row (m2, s, t2, zy)
  kModeBwd = 2,       // (4): pass 1 + loss + pass 2 from the SMEM-resident row segment
  kModeBwdPartials = 3,  // (4) on a vocab shard: stats from gathered partials, streaming pass 2
  kModeBwdVpf = 4        // (4) on a vocab shard, exchange fused in-kernel over peer memory (K4-VPF)
};

struct RowParams {
  int64_t num_rows;
  int64_t vocab;         // columns of this call (local vocab under sharding)
  int64_t ld;            // row stride in elements
  const void* logits;
  const int32_t* targets;
  const uint8_t* mask;   // row_mask (FWD/PARTIAL) or loss_mask (BWD); may be NULL in FWD/PARTIAL
  float scale;           // logit scale s
  int64_t vocab_start;   // global column of local column 0
  int64_t vocab_total;   // global vocabulary (target range check)
  int seg_elems;         // per-CTA column segment (multiple of 8) when the cluster splits a row
  int csize;             // CTAs per row (cluster size)
  int pipe;              // BWD_VPF: pipelined consumer loop, lag in rows (csize 1): 3 for segments <= 4 chunks,
                         // 1 for <= kPipeChunks, 0 = unpipelined
  // forward outputs
  float* logp;
  float* entropy;
  float* lse;
  float4* partials_out;
  // partial-combine input
  const float4* partials_in;  // [nshards][num_rows]
  int nshards;
  // loss
  const int32_t* row_traj;
  const double* adv;
  const float* old_logp;
  const float* ref_logp;
  const int64_t* n_loss;
  double clip_low, clip_high, kl_beta, clamp;
  double ent_coef, dual_clip;
  int reduction, sft;
  const int64_t* traj_tokens;
  const int64_t* n_active;
  const int32_t* adv_index;  // NULL: adv[row_traj[row]]
  int64_t num_adv;           // elements of adv (index bound)
  int64_t num_traj;          // elements of traj_tokens (index bound, sequence-mean reductions)
  int kl_type;
  int zero_masked;
  int accumulate;
  void* dlogits;
  otk_loss_stats* stats;
  // K4-VPF: in-kernel exchange of the 16-byte row partials with the other ranks
  void* vpf_xchg[OTK_VPF_MAX_RANKS];  // exchange buffer of every rank (peer-mapped), [vpf_rank] = own
  int vpf_rank, vpf_nranks;
  uint32_t* vpf_counter;  // calls completed on this buffer set (own buffer tail); epoch = counter + 1
  uint32_t* vpf_abort;    // epoch of a call that hit a peer timeout (own buffer tail + 4): its later waits end
  int64_t vpf_rows_cap;
  // ctx scratch
  double* cta_partials;
  unsigned int* ticket;
  int* err;
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_rows(const otk_ctx* ctx, RowMode mode, otk_dtype dtype, const RowParams& p, cudaStream_t s,
                        int* grid_out, int max_ctas = 0);
cudaError_t launch_rows_vpf_group(const otk_ctx* ctx, otk_dtype dtype, const RowParams* ps, int nsets, int pipe,
                                  cudaStream_t s, int* grid_out);
cudaError_t launch_combine(const otk_ctx* ctx, int64_t num_rows, int nshards, const float4* partials,
                           const uint8_t* row_mask, float* logp, float* entropy, float* lse, cudaStream_t s);

struct MaskParams {
  otk_traj_batch b;
  int16_t train_agent;
  uint8_t* loss_mask;
  uint8_t* response_mask;
  int32_t* row_traj;
  int64_t* traj_loss_tokens;
  int64_t* traj_source_counts;
  int64_t* n_loss;
  int64_t* n_active;
  int32_t* row_seg;
  unsigned int* ticket;
  int* err;
};
cudaError_t launch_masks(const MaskParams& p, cudaStream_t s);

struct AdvParams {
  int32_t num_traj;
  const int32_t* group_id;
  int32_t num_groups;
  const double* returns;
  const int32_t* turn_offsets;
  const double* turn_rewards;
  uint32_t flags;
  double std_floor;
  double* adv;
  double* returns_out;   // never NULL here (ctx scratch when the caller passed NULL)
  double* group_mean;
  double* group_std;
  int32_t* group_size;
  int* err;
};
cudaError_t launch_advantages(const AdvParams& p, cudaStream_t s);

struct TurnParams {
  otk_traj_batch b;
  int32_t num_segments;
  int16_t train_agent;
  const int32_t* group_id;
  const int32_t* turn_offsets;
  const double* turn_rewards;
  double gamma;
  double* seg_return;
  int32_t* seg_group;
  int* err;
};
cudaError_t launch_turn_returns(const TurnParams& p, cudaStream_t s);

struct SampleParams {
  int64_t num_rows, vocab, ld;
  const void* logits;
  const float* u;
  float scale;
  int greedy;
  int csize;  // CTAs per row (thread-block cluster), set by the launcher
  int32_t* tokens;
  float* logp;
  int* err;
};
cudaError_t launch_sample(otk_ctx* ctx, const SampleParams& p, int dtype, cudaStream_t s);
constexpr int kSampleTmMaxChunks = 64;   // k_sample_tm: rows of <= 64 x 12 KB (bf16 V <= 393216, fp32 V <= 196608)
bool sample_tm_fits(int64_t vocab, int dtype);
bool sample_dec_shape(int64_t num_rows, int64_t vocab, int dtype, int num_sms, int* csize, int* nseg_c);
cudaError_t launch_sample_dec(otk_ctx* ctx, SampleParams p, int dtype, int csize, int nseg_c, cudaStream_t s);
cudaError_t launch_sample_tm(otk_ctx* ctx, const SampleParams& p, int dtype, cudaStream_t s);

int lmhead_chunks(int64_t num_rows, int64_t vocab, int num_sms);
cudaError_t launch_lmhead_fwd(const otk_ctx* ctx, int64_t num_rows, int64_t vocab, int d, const void* hidden,
                              const void* weight, const int32_t* targets, const uint8_t* row_mask, float logit_scale,
                              float4* partials, int n_chunks, cudaStream_t s, int64_t vocab_start = 0,
                              int64_t vocab_total = 0, void* logits_out = nullptr, int64_t ld_out = 0);
// NEXT-1 backward (k_rows.cu / k_lmhead_bwd.cu)
cudaError_t launch_lmhead_loss_rows(const otk_ctx* ctx, const RowParams& p, float4* rowc, cudaStream_t s);
int lmhead_dh_splits(int64_t num_rows, int64_t vocab, int d, int num_sms);
cudaError_t launch_lmhead_bwd(const otk_ctx* ctx, int64_t num_rows, int64_t vocab, int d, const void* hidden,
                              const void* weight, const void* logits, void* dx_tiles, const float4* rowc,
                              const int32_t* targets, int64_t vocab_start, float logit_scale, bool ent, void* dh,
                              void* dw, float* dh_part, int dh_splits, cudaStream_t s, int* launches);
cudaError_t launch_combine_to_partial(const otk_ctx* ctx, int64_t num_rows, int nparts, const float4* partials,
                                      const uint8_t* row_mask, float4* out, cudaStream_t s);

__device__ __forceinline__ void set_error(int* err, int code) { atomicCAS(err, 0, code); }

}  // namespace otk
