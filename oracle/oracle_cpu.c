/*
 * oracle_cpu.c — plain float64 C oracle for the row-wise steps of the otk hot path.
 * TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs. Shares no code with paper_2601_07376_b200/csrc (the CUDA path).
 *
 * Same definitions as oracle_ref.py (which is pinned by tests/test_oracle_pins.py; this file is
 * cross-checked against it in tests/test_oracle_cpu.py):
 *   O3 (north_star (3)): z = s*x; M = max z; S = sum e^{z-M}; lse = M + ln S; logp = z_y - lse;
 *      H = ln S - sum e^{z-M}(z-M) / S   (terms with e^{z-M} == 0 contribute 0)
 *   O4 (north_star (4)): PPO-clip + KL surrogate per token and dL/dlogp; dlogits = coef (p - onehot)
 *      with coef = -s * (m / N) * G.  The loss sum over rows is left to the caller (row_L output).
 * Sums over the vocabulary use Neumaier compensated summation; rows are independent, so OpenMP
 * splits rows across threads (schedule(static)); no other reordering.
 * Inputs are read at their stored precision (fp32, or bf16 bits) and widened exactly to double.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORC_F32 0
#define ORC_BF16 1

typedef struct {
  double clip_low, clip_high, kl_beta, log_ratio_clamp, logit_scale;
  int32_t kl_type; /* 1, 2, 3 */
  int32_t zero_masked_rows;
} orc_cfg;

static inline double widen(const void* base, int dtype, int64_t idx) {
  if (dtype == ORC_F32) return (double)((const float*)base)[idx];
  uint32_t bits = ((uint32_t)((const uint16_t*)base)[idx]) << 16;
  float f;
  memcpy(&f, &bits, 4);
  return (double)f;
}

/* Neumaier compensated sum of a stream of terms. */
typedef struct { double s, c; } nsum;
static inline void nadd(nsum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
  a->s = t;
}
static inline double nget(const nsum* a) { return a->s + a->c; }

/* O3 for one row. Returns 0 on success, 1 if the target is out of range. */
static int row_forward(const void* logits, int dtype, int64_t row_off, int64_t V, int32_t y, double s,
                       double* logp, double* H, double* lse) {
  if (y < 0 || y >= V) return 1;
  double M = -INFINITY;
  for (int64_t v = 0; v < V; ++v) {
    double z = s * widen(logits, dtype, row_off + v);
    if (z > M) M = z;
  }
  nsum S = {0, 0}, T = {0, 0};
  for (int64_t v = 0; v < V; ++v) {
    double d = s * widen(logits, dtype, row_off + v) - M;
    double e = exp(d);
    nadd(&S, e);
    if (e > 0) nadd(&T, e * d);
  }
  double Sv = nget(&S);
  *lse = M + log(Sv);
  *logp = s * widen(logits, dtype, row_off + y) - *lse;
  *H = log(Sv) - nget(&T) / Sv;
  return 0;
}

int orc_logprob_entropy(int64_t n_rows, int64_t V, int64_t ld, int32_t dtype, const void* logits,
                        const int32_t* targets, const uint8_t* row_mask, double logit_scale,
                        double* logp, double* entropy, double* lse) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t j = 0; j < n_rows; ++j) {
    logp[j] = entropy[j] = lse[j] = 0.0;
    if (row_mask && !row_mask[j]) continue;
    bad |= row_forward(logits, dtype, j * ld, V, targets[j], logit_scale, &logp[j], &entropy[j], &lse[j]);
  }
  return bad;
}

/* Per-token surrogate and its derivative wrt logp (same definition as oracle_ref.row_loss_terms). */
static void row_loss_terms(double logp, double old, double ref, double A, const orc_cfg* c,
                           double* L, double* G, int* clipped, double* kl_out) {
  double C = c->log_ratio_clamp;
  double draw = logp - old;
  double delta = fmin(fmax(draw, -C), C);
  double r = exp(delta);
  double rbar = fmin(fmax(r, 1.0 - c->clip_low), 1.0 + c->clip_high);
  double pg = fmax(-A * r, -A * rbar);
  int clip = (A > 0 && r > 1.0 + c->clip_high) || (A < 0 && r < 1.0 - c->clip_low);
  double g = (clip || fabs(draw) > C) ? 0.0 : -A * r;
  double kl = 0.0;
  if (c->kl_beta != 0.0) {
    double gk;
    if (c->kl_type == 3) {
      double dr = ref - logp;
      double d = fmin(fmax(dr, -C), C);
      kl = exp(d) - d - 1.0;
      gk = fabs(dr) > C ? 0.0 : 1.0 - exp(d);
    } else if (c->kl_type == 1) {
      kl = logp - ref;
      gk = 1.0;
    } else {
      kl = 0.5 * (logp - ref) * (logp - ref);
      gk = logp - ref;
    }
    g += c->kl_beta * gk;
  }
  *L = pg + c->kl_beta * kl;
  *G = g;
  *clipped = clip;
  *kl_out = kl;
}

/* Fused O3 + O4 per row. dlogits (row-major [n_rows, V] doubles) may be NULL (then only the
 * per-row scalars are produced, e.g. for timing the forward + loss without the gradient store).
 * Returns nonzero if any trainable row has an out-of-range target. */
int orc_policy_loss(int64_t n_rows, int64_t V, int64_t ld, int32_t dtype, const void* logits,
                    const int32_t* targets, const uint8_t* loss_mask, const int32_t* row_traj,
                    const double* adv, const float* old_logp, const float* ref_logp, int64_t n_loss,
                    const orc_cfg* cfg, double* dlogits, double* logp, double* entropy,
                    double* row_L, uint8_t* row_clipped, double* row_kl, double* row_lse, double* row_coef) {
  const double s = cfg->logit_scale;
  const double invN = n_loss > 0 ? 1.0 / (double)n_loss : 0.0;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t j = 0; j < n_rows; ++j) {
    double* dl = dlogits ? dlogits + j * V : 0;
    logp[j] = entropy[j] = row_L[j] = row_kl[j] = 0.0;
    if (row_lse) row_lse[j] = 0.0;
    if (row_coef) row_coef[j] = 0.0;
    row_clipped[j] = 0;
    if (!loss_mask[j]) {
      if (dl && cfg->zero_masked_rows) for (int64_t v = 0; v < V; ++v) dl[v] = 0.0;
      continue;
    }
    double lp, H, lse;
    if (row_forward(logits, dtype, j * ld, V, targets[j], s, &lp, &H, &lse)) { bad = 1; continue; }
    double L, G, kl;
    int clipped;
    double ref = ref_logp ? (double)ref_logp[j] : 0.0;
    row_loss_terms(lp, (double)old_logp[j], ref, adv[row_traj[j]], cfg, &L, &G, &clipped, &kl);
    logp[j] = lp;
    entropy[j] = H;
    row_L[j] = L;
    row_kl[j] = kl;
    row_clipped[j] = (uint8_t)clipped;
    const double coef = -s * invN * G;
    if (row_lse) row_lse[j] = lse;
    if (row_coef) row_coef[j] = coef;
    if (dl) {
      for (int64_t v = 0; v < V; ++v) {
        double p = exp(s * widen(logits, dtype, j * ld + v) - lse);
        dl[v] = coef * (p - (v == targets[j] ? 1.0 : 0.0));
      }
    }
  }
  return bad;
}

/* O1 masks, plain sequential walk over the segment CSR.
 * Returns 0 ok, 6 unterminated, 7 bad trajectory. */
int orc_build_masks(int32_t B, const int64_t* tok_offsets, const int32_t* seg_offsets,
                    const uint8_t* seg_source, const int16_t* seg_agent, const int32_t* seg_len,
                    const uint8_t* terminated, int16_t train_agent, const int16_t* traj_agent,
                    uint8_t* loss_mask, uint8_t* response_mask, int32_t* row_traj,
                    int64_t* traj_loss_tokens, int64_t* n_loss) {
  int64_t total = 0;
  for (int32_t b = 0; b < B; ++b) {
    if (terminated && !terminated[b]) return 6;
    int ta = traj_agent ? traj_agent[b] : train_agent;
    int64_t row = tok_offsets[b];
    int64_t cnt = 0;
    for (int32_t k = seg_offsets[b]; k < seg_offsets[b + 1]; ++k) {
      if (seg_len[k] <= 0 || seg_source[k] > 3) return 7;
      if (row + seg_len[k] > tok_offsets[b + 1]) return 7;
      int trainable = seg_source[k] == 1 && (ta == -1 || seg_agent[k] == ta);
      int responding = !(k == seg_offsets[b] && seg_source[k] == 0) && seg_source[k] != 3;
      for (int32_t i = 0; i < seg_len[k]; ++i, ++row) {
        loss_mask[row] = (uint8_t)trainable;
        if (response_mask) response_mask[row] = (uint8_t)responding;
        row_traj[row] = b;
      }
      if (trainable) cnt += seg_len[k];
    }
    if (row != tok_offsets[b + 1]) return 7;
    traj_loss_tokens[b] = cnt;
    total += cnt;
  }
  *n_loss = total;
  return 0;
}

/* ------------------------------------------------------------------------------------------------
 * Comparison helper (test infrastructure; the tolerance policy is passed in by the caller, see
 * oracle/parity.py). For each selected row j it re-forms the O4 gradient element by element in
 * float64 from the row's own lse_j and coef_j (outputs of orc_policy_loss, or an alternative coef for
 * a row on a clip / clamp kink):
 *     p_v = exp(s x_v - lse_j),  q_v = p_v - [v == y_j],  want_v = coef_j q_v
 * and compares it with the CUDA path's value got_v (fp32, or bf16 bits, row stride got_ld):
 *     floor_v = dcoef_j |q_v| + [v == y_j] |coef_j| p_v logp_err + abs_floor
 *     tol_v   = rel |want_v| + floor_v
 * dcoef_j is the absolute error bound of coef_j, the target column's extra term is the error p_y * dlogp of
 * coef * expm1(logp), and abs_floor covers values below the output format's smallest normal (flushed to 0).
 * Outputs per row: max_v |got_v - want_v| / tol_v (0/0 = 0, x/0 = inf), and over the non-target columns
 * sum |got - want|, sum |want|, sum want^2, sum floor. Rows with sel[j] == 0 are skipped (outputs untouched). */
int orc_dlogits_compare(int64_t n_rows, int64_t V, int64_t ld, int32_t dtype, const void* logits,
                        const int32_t* targets, const uint8_t* sel, double logit_scale, const double* lse,
                        const double* coef, const double* dcoef, double logp_err, double rel, double abs_floor,
                        const void* got, int64_t got_ld, int32_t got_dtype,
                        double* max_ratio, double* l1_err, double* l1_ref, double* l2_ref, double* l1_floor) {
  const double s = logit_scale;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n_rows; ++j) {
    if (sel && !sel[j]) continue;
    double worst = 0.0;
    nsum E = {0, 0}, R = {0, 0}, R2 = {0, 0}, F = {0, 0};
    for (int64_t v = 0; v < V; ++v) {
      double p = exp(s * widen(logits, dtype, j * ld + v) - lse[j]);
      double q = p - (v == targets[j] ? 1.0 : 0.0);
      double want = coef[j] * q;
      double floor_v = dcoef[j] * fabs(q) + (v == targets[j] ? fabs(coef[j]) * p * logp_err : 0.0) + abs_floor;
      double tol = rel * fabs(want) + floor_v;
      double d = fabs(widen(got, got_dtype, j * got_ld + v) - want);
      double r = d == 0.0 ? 0.0 : (tol > 0.0 ? d / tol : INFINITY);
      if (r > worst || r != r) worst = r != r ? INFINITY : r;
      if (v != targets[j]) {  /* row sums over the non-target columns (the target column is one element) */
        nadd(&E, d);
        nadd(&R, fabs(want));
        nadd(&R2, want * want);
        nadd(&F, floor_v);
      }
    }
    max_ratio[j] = worst;
    l1_err[j] = nget(&E);
    l1_ref[j] = nget(&R);
    l2_ref[j] = nget(&R2);
    l1_floor[j] = nget(&F);
  }
  return 0;
}
