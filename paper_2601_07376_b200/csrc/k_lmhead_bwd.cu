// k_lmhead_bwd.cu — NEXT-1, backward half: the policy-loss gradient THROUGH the LM head,
//   dh = dx W      [N, d]        and        dW = dxᵀ h      [V, d],
// with dx = dL/dx = coef_j (p_jv - [v = y_j]) (north_star (4), the "update" pool) formed on chip
// from the bf16 logits x and four per-row constants: dx is never written to HBM and the loss kernel's 4V bytes
// per row (read x, write dx) disappear. x is written once by the forward (k_lmhead_fwd with logits_out), the
// per-row constants by k_lmhead_loss_rows (k_rows.cu).
//
// tcgen05 GEMM on CTA pairs (cta_group::2, M = 256 rows per pair, N = 512 hidden columns per pair = two
// N = 256 MMAs, K = 64 per stage; each CTA holds its 128 rows x 512 fp32 accumulators = all 512 TMEM columns):
//   dh : A = x tile   [128 rows x 64 vocab]  K-major (x is row-major [N, V], K = V)     B = W  [64 v x 256 d] MN-major
//   dW : A = xᵀ tile  [128 vocab x 64 rows]  MN-major (M = V contiguous in x, K = rows)  B = h  [64 j x 256 d] MN-major
// Per stage and CTA: A (16 KB) lands by TMA on the CTA's own barrier; 8 transform warps rewrite it IN PLACE
// (same swizzled position, new value) as
//   dx = 2^d (alpha'_j + beta'_j d),   d = s log2(e) x - m_j,
// replaced by gy_j at the target column (gy = coef expm1(logp), no cancellation), then fence the generic-proxy
// writes for the async proxy and arrive on the leader CTA's "ready" barrier; the leader's MMA thread waits for
// ready (both CTAs) + B (both CTAs' TMA on the leader's barrier) and issues 8 MMAs per stage. The transform
// costs 2 MUFU ex2 per pair of elements = 8192 ex2 per CTA per stage against 1024 clocks of MMA (N = 512 keeps
// it at half the SFU rate; N = 256 would saturate it).
// After a unit's last stage the transform warps drain TMEM (tcgen05.ld 32x32b, one row per thread, 128 columns
// per warp) into the output — bf16, or fp32 split-K partials for dh — and release the accumulators.
// dh's hidden tile 0 runs first (its own launch); its units also TMA-store each transformed A stage, so dx exists
// once in HBM as 64 x 64 tiles (2 bytes per logit written). dh's hidden tiles 1 .. d/512 - 1 (a second launch) and
// dW = dxᵀ h then run as plain GEMMs over those tiles: dx is formed once per element instead of once per hidden tile
// of each GEMM (2 x d/512 times).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "otk_internal.h"
#include "otk_ptx.cuh"
#include "otk_umma.cuh"

namespace otk {

using namespace ptx;
using namespace umma;

constexpr int kBwK = 64;
// A and B have rings of their own: A needs TMA + the transform before the MMA may read it, B only TMA, so A
// runs deeper (6 stages = 6 k-blocks ahead) than B (4) in the 227 KB of shared memory.
#ifndef OTK_BW_ASTAGES
#define OTK_BW_ASTAGES 6
#define OTK_BW_BSTAGES 4
#endif
constexpr int kBwAStages = OTK_BW_ASTAGES, kBwBStages = OTK_BW_BSTAGES;
constexpr int kBwABytes = 128 * kBwK * 2;  // 16 KB: this CTA's 128 M-rows x 64 k
constexpr int kBwBBytes = 256 * kBwK * 2;  // 32 KB: this CTA's 2 x 128 N-columns x 64 k (4 TMA boxes of 64 x 64)
constexpr int kBwXWarps = 16;  // transform + epilogue warps (2..17); warp 0 loads A, warp 18 loads B, warp 1 MMAs,
                               // warp 19 stores dx tiles (dh)
constexpr int kBwThreads = 32 * (4 + kBwXWarps);
constexpr int kBwBOff = kBwAStages * kBwABytes;
constexpr int kBwSmemBytes = kBwBOff + kBwBStages * kBwBBytes + 1024 /* alignment slack */ + 512 /* barriers */;
static_assert(kBwSmemBytes <= 232448, "shared memory of one CTA");
constexpr int kBwMtile = 256, kBwNtile = 512;

constexpr uint32_t kIdescDh = idesc_bf16(256, 256, false, true);  // A K-major, B MN-major
constexpr uint32_t kIdescDw = idesc_bf16(256, 256, true, true);   // A MN-major, B MN-major

struct LmBwdParams {
  int64_t num_rows, vocab;
  int d;
  int n_mt, n_nt;        // M tiles (rows for dh, vocab for dW), N tiles of 512 hidden columns (of this launch)
  int nt0;               // first hidden tile of this launch
  int kb_total, kb_per_split, splits;
  const float4* rowc;    // [num_rows] {m, alpha', beta', gy}
  const int32_t* targets;
  int64_t vocab_start;   // global id of local vocab column 0
  float s2;              // logit_scale * log2(e)
  int store_dx;          // dh: units of hidden tile 0 also store the transformed A (= dx tiles) through tm_dx
  int xform;             // 0: A already holds dx (dW, and dh's hidden tiles >= 1, after dh's tile 0 stored it):
                         //    no transform, the GEMM alone
  int f32out;            // dh: fp32 split-K partials [split][num_rows][d] (reduced afterwards) instead of bf16
  void* out;             // dh: fp32 partials (f32out) or bf16 [num_rows][d]; dW: bf16 [vocab][d]
};

__device__ __forceinline__ void bw_unit(const LmBwdParams& p, int u, int& mt, int& nt, int& kb0, int& kb1, int& sp) {
  const int per = p.n_mt * p.n_nt;
  sp = u / per;
  const int r = u - sp * per;
  mt = r / p.n_nt;
  nt = p.nt0 + (r - mt * p.n_nt);
  kb0 = sp * p.kb_per_split;
  kb1 = min(p.kb_total, kb0 + p.kb_per_split);
}

// Per-row constants of the transform. General form (entropy bonus on): g = 2^d (al + be d), d = x s2 - m.
// Without the bonus (be = 0 for every row) the coefficient is folded into the exponent and its sign into the
// packed result: g = sgn * 2^(x s2 - m + log2|al|) — per pair of elements 2 unpacks, FFMA2, 2 MUFU.EX2, F2FP,
// LOP3 (|al| = 0 gives 2^-inf = 0: masked rows cost nothing special).
struct RowK {
  uint64_t negm2, al2, be2;
  uint32_t sgn;  // 0x80008000 when al < 0 (folded form)
  bool dead;     // no gradient through this row (loss-masked / padding): all zeros
  float gy;
  int ycol;      // local vocab column of the target, or -1
};
struct RawK {
  float4 c;
  int32_t y;     // local target column (vocab_start subtracted)
};
__device__ __forceinline__ RawK raw_consts(const LmBwdParams& p, int64_t j) {
  RawK r{make_float4(1e30f, 0.f, 0.f, 0.f), -1};  // inactive / out-of-range row: d = -1e30 -> 2^d = 0, g = 0
#ifdef OTK_BW_NO_ROWLOAD  // experiment: no per-row constant loads
  return r;
#endif
  if (j < p.num_rows) {
    r.c = p.rowc[j];
    r.y = int32_t(int64_t(p.targets[j]) - p.vocab_start);
  }
  return r;
}
template <bool kEnt>
__device__ __forceinline__ RowK cook(const RawK& r, int64_t vocab) {
  RowK k;
  if (kEnt) {
    k.negm2 = f2(-r.c.x, -r.c.x);
    k.sgn = 0u;
  } else {
    const float nm = __fsub_rn(lg2(fabsf(r.c.y)), r.c.x);  // log2|al| - m  (-inf when al = 0)
    k.negm2 = f2(nm, nm);
    k.sgn = r.c.y < 0.f ? 0x80008000u : 0u;
  }
  k.al2 = f2(r.c.y, r.c.y);
  k.be2 = f2(r.c.z, r.c.z);
  k.gy = r.c.w;
  k.ycol = (r.y >= 0 && r.y < vocab) ? r.y : -1;
  k.dead = r.c.y == 0.f && r.c.z == 0.f && r.c.w == 0.f;
  return k;
}

// 2^d for a pair on the FMA / ALU pipes (the FA4-style split of the exponentials between MUFU and FMA): n = RN(d)
// via the 1.5 * 2^23 magic add, 2^(d - n) by a degree-3 minimax polynomial on [-1/2, 1/2] (relative error
// 7.5e-5 = 2^-13.7, against 2^-9 of the bf16 output), n added to the exponent bits. d is clamped at -127 (the
// result is then below 2^-126; fully masked rows are zeroed separately).
#ifndef OTK_BW_POLY_WORDS
#define OTK_BW_POLY_WORDS 1
#endif
constexpr int kPolyWords = OTK_BW_POLY_WORDS;  // of the 4 words (8 elements) of a chunk
__device__ __forceinline__ void exp2_poly_pair(uint64_t d2, float& el, float& eh) {
  float dl, dh;
  f2_split(d2, dl, dh);
  const uint64_t dc = f2(fmaxf(dl, -127.f), fmaxf(dh, -127.f));
  const uint64_t t2 = fadd2(dc, f2(12582912.f, 12582912.f));
  const uint64_t n2 = fadd2(t2, f2(-12582912.f, -12582912.f));
  const uint64_t fr = ffma2(n2, f2(-1.f, -1.f), dc);
  uint64_t p2 = ffma2(f2(0.055176056984240475f, 0.055176056984240475f), fr, f2(0.24261150977353746f, 0.24261150977353746f));
  p2 = ffma2(p2, fr, f2(0.6932601800070715f, 0.6932601800070715f));
  p2 = ffma2(p2, fr, f2(0.9999280269520706f, 0.9999280269520706f));
  float tl, th, pl, ph;
  f2_split(t2, tl, th);
  f2_split(p2, pl, ph);
  el = __uint_as_float(__float_as_uint(tl) * 8388608u + __float_as_uint(pl));  // + n << 23 (magic bits wrap to 0)
  eh = __uint_as_float(__float_as_uint(th) * 8388608u + __float_as_uint(ph));
}
template <bool kEnt, bool kPoly = false>
__device__ __forceinline__ uint32_t bw_word(uint32_t w, uint64_t s2x2, const RowK& k) {
  const uint64_t d2 = ffma2(f2(bf_lo(w), bf_hi(w)), s2x2, k.negm2);
  float dl, dh;
  f2_split(d2, dl, dh);
  if (kEnt) {
    const uint64_t e2 = f2(ex2(dl), ex2(dh));
    float gl, gh;
    f2_split(fmul2(e2, ffma2(k.be2, d2, k.al2)), gl, gh);
    return pack_bf16x2(gl, gh);
  } else if (kPoly) {
    float el, eh;
    exp2_poly_pair(d2, el, eh);
    return pack_bf16x2(el, eh) ^ k.sgn;
  } else {
    return pack_bf16x2(ex2(dl), ex2(dh)) ^ k.sgn;
  }
}
// one 16-byte chunk (8 consecutive vocab columns of one row) rewritten in place
template <bool kEnt>
__device__ __forceinline__ void bw_chunk(uint32_t addr, int yoff, bool zero, uint64_t s2x2, const RowK& k) {
#ifdef OTK_BW_NO_TRANSFORM  // experiment: the GEMM pipeline alone (operands left as loaded)
  return;
#endif
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  uint32_t g[4] = {bw_word<kEnt, (kPolyWords > 3)>(v.x, s2x2, k), bw_word<kEnt, (kPolyWords > 1)>(v.y, s2x2, k),
                   bw_word<kEnt, (kPolyWords > 2)>(v.z, s2x2, k), bw_word<kEnt, (kPolyWords > 0)>(v.w, s2x2, k)};
  if (unsigned(yoff) < 8u) {  // the target column: coef (p_y - 1) formed without cancellation
    const uint32_t gb = pack_bf16x2(k.gy, k.gy) & 0xFFFFu;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // masks for every word (no dynamic index: g[] stays in registers)
      const int r = yoff - 2 * q;  // 0 / 1: the target is the low / high half of word q
      const uint32_t keep = r == 0 ? 0xFFFF0000u : (r == 1 ? 0x0000FFFFu : 0xFFFFFFFFu);
      const uint32_t ins = r == 0 ? gb : (r == 1 ? (gb << 16) : 0u);
      g[q] = (g[q] & keep) | ins;
    }
  }
  if (zero || k.dead) g[0] = g[1] = g[2] = g[3] = 0u;
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(g[0]), "r"(g[1]), "r"(g[2]), "r"(g[3])
               : "memory");
}

#ifdef OTK_BW_TIMING  // experiments only: clock64 sums (MMA thread of each pair; transform warp 2 lane 0 of each CTA)
__device__ unsigned long long g_bw_timing[2][2][8];  // [dh, dW][MMA thread, transform warp][slot]
#define BW_T0() const long long _t0 = clock64()
#define BW_ACC(slot) tacc[slot] += clock64() - _t0
#else
#define BW_T0()
#define BW_ACC(slot)
#endif

template <int MODE, bool kEnt>
__global__ void __launch_bounds__(kBwThreads, 1)
    k_lmhead_bwd(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 const __grid_constant__ CUtensorMap tm_dx, const LmBwdParams p) {
  constexpr bool kDh = MODE == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + kBwBOff + kBwBStages * kBwBBytes);
  uint64_t* readyA = fullA + kBwAStages;
  uint64_t* emptyA = readyA + kBwAStages;
  uint64_t* fullB = emptyA + kBwAStages;
  uint64_t* emptyB = fullB + kBwBStages;
  uint64_t* tfull = emptyB + kBwBStages;
  uint64_t* tempty = tfull + 1;
  uint64_t* xdone = tempty + 1;  // [kBwAStages] this CTA's transform of a stage is complete (dx store)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xdone + kBwAStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = int(cluster_ctarank());
  const int pair = int(cluster_id_x()), npairs = int(nclusters_x());
  const int n_units = p.n_mt * p.n_nt * p.splits;
#ifdef OTK_BW_TIMING
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < kBwAStages; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&readyA[s], 2 * kBwXWarps);
      mbar_init(&emptyA[s], p.store_dx ? 2 : 1);  // + the dx storer's release
      mbar_init(&xdone[s], kBwXWarps);
    }
    for (int s = 0; s < kBwBStages; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * kBwXWarps);
    fence_mbar_init();
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
    if (p.store_dx) prefetch_tmap(&tm_dx);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer of A (both CTAs): the x tiles, on this CTA's own barrier
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int mt, nt, kb0, kb1, sp;
        bw_unit(p, u, mt, nt, kb0, kb1, sp);
        const int m0 = mt * kBwMtile + rank * 128;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&emptyA[s], ph ^ 1u);
          const uint32_t a = smem_u32(smem + s * kBwABytes);
          if (!p.xform) {  // A is the operand as loaded: both CTAs' bytes counted on the leader's barrier, no relay
            if (rank == 0) mbar_arrive_expect_tx(&fullA[s], 2 * kBwABytes);
            if (kDh)  // dx tiles (row block m0/64 .. +1, vocab block kb), K-major rows
              tma_load_4d_pair(a, &tm_a, smem_u32(&fullA[s]) & kPeerBitMask, 0, 0, kb, m0 >> 6);
            else      // dx tiles (row block kb, vocab blocks m0/64 .. +1), MN-major
              tma_load_4d_pair(a, &tm_a, smem_u32(&fullA[s]) & kPeerBitMask, 0, 0, m0 >> 6, kb);
          } else {
            mbar_arrive_expect_tx(&fullA[s], kBwABytes);
            if (kDh)  // x tiles (row block m0/64 .. +1, vocab block kb): [2][64 rows][64 v], K-major rows
              tma_load_4d(a, &tm_a, &fullA[s], 0, 0, kb, m0 >> 6);
            else      // x tiles (row block kb, vocab blocks m0/64 .. +1): [2][64 rows][64 v], MN-major
              tma_load_4d(a, &tm_a, &fullA[s], 0, 0, m0 >> 6, kb);
          }

          if (++s == kBwAStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 2 + kBwXWarps) {
    // ---------------- TMA producer of B (both CTAs): W / h tiles, counted on the leader's barrier
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int mt, nt, kb0, kb1, sp;
        bw_unit(p, u, mt, nt, kb0, kb1, sp);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&emptyB[s], ph ^ 1u);
          const uint32_t b = smem_u32(smem + kBwBOff + s * kBwBBytes);
          const uint32_t barB = smem_u32(&fullB[s]) & kPeerBitMask;
#ifdef OTK_BW_NO_B  // experiment (with OTK_BW_NO_MMA): no B traffic
          if (rank == 0) mbar_arrive(&fullB[s]);
          if (++s == kBwBStages) {
            s = 0;
            ph ^= 1u;
          }
          continue;
#endif
          if (rank == 0) mbar_arrive_expect_tx(&fullB[s], 2 * kBwBBytes);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              tma_load_2d_pair(b + h * 16384 + q * 8192, &tm_b, barB, nt * kBwNtile + h * 256 + rank * 128 + q * 64,
                               kb * kBwK);
            }
          if (++s == kBwBStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 3 + kBwXWarps) {
    // ---------------- dx storer (dh, both CTAs): once the transform of a stage of a hidden-tile-0 unit is complete,
    // TMA-store it (the dx tiles the dW GEMM reads), wait for the store to have read it, and release the stage
    // (emptyA's second arrival; other units release at once)
    if (lane == 0 && p.store_dx) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int mt, nt, kb0, kb1, sp;
        bw_unit(p, u, mt, nt, kb0, kb1, sp);
        const int m0 = mt * kBwMtile + rank * 128;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&xdone[s], ph);
          if (nt == 0) {
            tma_store_4d(&tm_dx, smem_u32(smem + s * kBwABytes), 0, 0, kb, m0 >> 6);
            bulk_commit();
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          mbar_arrive(&emptyA[s]);
          if (++s == kBwAStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
      bulk_wait_all();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread)
    if (rank == 0 && lane == 0) {
      int sa = 0, sb = 0;
      uint32_t pha = 0, phb = 0, it = 0;
      for (int u = pair; u < n_units; u += npairs, ++it) {
        int mt, nt, kb0, kb1, sp;
        bw_unit(p, u, mt, nt, kb0, kb1, sp);
        {
          BW_T0();
          mbar_wait(tempty, (it & 1u) ^ 1u);  // the epilogues drained the previous unit's accumulators
          BW_ACC(2);
        }
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            BW_T0();
            mbar_wait(&fullB[sb], phb);
            BW_ACC(0);
          }
          {
            BW_T0();
            if (p.xform)
              mbar_wait_cluster(&readyA[sa], pha);
            else
              mbar_wait(&fullA[sa], pha);
            BW_ACC(1);
          }
#ifdef OTK_BW_TIMING
          tacc[7] += 1;
#endif
          tc_fence_after();
          const uint32_t a = smem_u32(smem + sa * kBwABytes);
          const uint32_t b = smem_u32(smem + kBwBOff + sb * kBwBBytes);
#pragma unroll
          for (int k = 0; k < kBwK / 16; ++k) {
            const uint64_t ad = kDh ? sw128_kmajor_desc(a + k * 32) : sw128_mnmajor_desc(a + k * 2048, 8192);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint64_t bd = sw128_mnmajor_desc(b + h * 16384 + k * 2048, 8192);
              const uint32_t acc = (kb > kb0 || k > 0) ? 1u : 0u;
#ifdef OTK_BW_NO_MMA  // experiment: the load + transform pipeline alone
              continue;
#endif
              if (kDh)
                umma_pair_bf16<kIdescDh>(tmem + h * 256, ad, bd, acc);
              else
                umma_pair_bf16<kIdescDw>(tmem + h * 256, ad, bd, acc);
            }
          }
          umma_commit_pair(&emptyA[sa]);
          umma_commit_pair(&emptyB[sb]);
          if (++sa == kBwAStages) {
            sa = 0;
            pha ^= 1u;
          }
          if (++sb == kBwBStages) {
            sb = 0;
            phb ^= 1u;
          }
        }
        umma_commit_pair(tfull);
      }
#ifdef OTK_BW_TIMING
      tacc[3] = clock64() - t_start;
      for (int k = 0; k < 8; ++k) atomicAdd(&g_bw_timing[kDh ? 0 : 1][0][k], (unsigned long long)tacc[k]);
#endif
    }
  } else {
    // ---------------- transform + epilogue (both CTAs, warps 2..17)
    const int xt = threadIdx.x - 64;
    const uint32_t ready_leader = smem_u32(&readyA[0]) & kPeerBitMask;
    const uint32_t tempty_leader = smem_u32(tempty) & kPeerBitMask;
    const uint64_t s2x2 = f2(p.s2, p.s2);
    int s = 0;
    uint32_t ph = 0, it = 0;
    for (int u = pair; u < n_units; u += npairs, ++it) {
      int mt, nt, kb0, kb1, sp;
      bw_unit(p, u, mt, nt, kb0, kb1, sp);
      const int64_t m0 = int64_t(mt) * kBwMtile + rank * 128;
      if (kDh) {
        // thread -> (row r, quarter qq): 2 of the 8 16-byte chunks of row r's 128-byte K row; constants fixed
        // for the unit. A quarter-warp covers 2 rows x 4 quarters: chunk sets of opposite parity, no conflict.
        const int r = xt >> 2, qq = xt & 3;
        const RowK rk = cook<kEnt>(raw_consts(p, m0 + r), p.vocab);
        for (int kb = kb0; kb < kb1 && p.xform; ++kb) {  // (A as loaded: nothing to transform, no relay)
          {
            BW_T0();
            mbar_wait(&fullA[s], ph);
            BW_ACC(4);
          }
          BW_T0();
          const uint32_t a = smem_u32(smem + s * kBwABytes);
          const int v0 = kb * kBwK;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int c = qq * 2 + i;
            const int vc = v0 + c * 8;
            bw_chunk<kEnt>(a + r * 128 + ((c ^ (r & 7)) << 4), rk.ycol - vc, vc >= p.vocab, s2x2, rk);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_remote(ready_leader + s * 8);
            if (p.store_dx) mbar_arrive(&xdone[s]);
          }
          BW_ACC(5);
          if (++s == kBwAStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      } else {
        // thread -> (k row jj, box b, quarter qq): the row constants change with every stage (K = rows); their raw
        // values are loaded two stages ahead so the global-load latency never sits in front of a transform. A
        // quarter-warp is one k row: box 1 takes the chunks of the other parity (no bank conflict with box 0).
        const int jj = xt >> 3, b = (xt >> 2) & 1, qq = xt & 3;
        RawK q0, q1;
        if (p.xform) {
          q0 = raw_consts(p, int64_t(kb0) * kBwK + jj);
          q1 = raw_consts(p, int64_t(kb0 + 1) * kBwK + jj);
        }
        for (int kb = kb0; kb < kb1 && p.xform; ++kb) {  // (A as loaded: nothing to transform, no relay)
          const RowK cur = cook<kEnt>(q0, p.vocab);
          q0 = q1;
          q1 = raw_consts(p, int64_t(kb + 2) * kBwK + jj);
          {
            BW_T0();
            mbar_wait(&fullA[s], ph);
            BW_ACC(4);
          }
          BW_T0();
          const uint32_t a = smem_u32(smem + s * kBwABytes) + b * 8192 + jj * 128;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int c = qq * 2 + (i ^ b);
            const int64_t vc = m0 + b * 64 + c * 8;
            bw_chunk<kEnt>(a + ((c ^ (jj & 7)) << 4), int(cur.ycol - vc), vc >= p.vocab, s2x2, cur);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_remote(ready_leader + s * 8);
            if (p.store_dx) mbar_arrive(&xdone[s]);
          }
          BW_ACC(5);
          if (++s == kBwAStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
      // ---- epilogue: warp (quadrant q, column quarter ch) drains 32 rows x 128 columns of the accumulators
      BW_T0();
      mbar_wait(tfull, it & 1u);
      tc_fence_after();
      const int q = warp & 3, ch = (warp - 2) >> 2;  // TMEM lane quadrant, 128-column quarter
      const int64_t row = m0 + q * 32 + lane;
      const int64_t M = kDh ? p.num_rows : p.vocab;
      const uint32_t tl = tmem + (uint32_t(q * 32) << 16) + uint32_t(ch * 128);
      const int col0 = nt * kBwNtile + ch * 128;
      const bool f32out = kDh && p.f32out;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        float v[32];
        tmem_ld32(tl + uint32_t(cc * 32), v);
        const int col = col0 + cc * 32;
#ifdef OTK_BW_NO_EPI_STORE  // experiment: epilogue without the global stores
        if (v[0] == 12345.f) asm volatile("" ::"f"(v[1]));
        continue;
#endif
        if (row < M && col < p.d) {
          // 256-bit stores: every instruction writes whole 32-byte sectors (rows are 32-byte aligned: d % 64 == 0)
          if (f32out) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<float*>(p.out) +
                                                  (int64_t(sp) * p.num_rows + row) * p.d + col);
            const uint32_t* u = reinterpret_cast<const uint32_t*>(v);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              stg256(dst + 2 * k, make_uint4(u[8 * k], u[8 * k + 1], u[8 * k + 2], u[8 * k + 3]),
                     make_uint4(u[8 * k + 4], u[8 * k + 5], u[8 * k + 6], u[8 * k + 7]));
          } else {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.d + col);
            uint32_t w[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) w[k] = pack_bf16x2(v[2 * k], v[2 * k + 1]);
            stg256(dst, make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
            stg256(dst + 2, make_uint4(w[8], w[9], w[10], w[11]), make_uint4(w[12], w[13], w[14], w[15]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader);
      BW_ACC(6);
    }
#ifdef OTK_BW_TIMING
    if (xt == 0)
      for (int k = 4; k < 7; ++k) atomicAdd(&g_bw_timing[kDh ? 0 : 1][1][k], (unsigned long long)tacc[k]);
#endif
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// dh = sum over splits of the fp32 partials (fixed order: deterministic), rounded once to bf16; hidden columns
// [0, 512) (tile 0, its own launch) have splits0 partials, the others splits1
__global__ void k_lmhead_dh_reduce(const float4* __restrict__ part, int splits0, int splits1, int d, int64_t n4,
                                   uint2* __restrict__ dh) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const int splits = int((i * 4) % d) < kBwNtile ? splits0 : splits1;
    float4 a = part[i];
    for (int s = 1; s < splits; ++s) {
      const float4 b = part[int64_t(s) * n4 + i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    dh[i] = make_uint2(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w));
  }
}

// ---- host side -----------------------------------------------------------------------------------------
// split-K of dh: (row tiles x hidden tiles) units are few (e.g. 32 x 7 at N = 8192, d = 3584) against 74 CTA
// pairs; splitting the vocab (K) dimension fills whole waves. Cost model in stages: waves x (stages per unit +
// an epilogue of ~8 stages), plus the partials' round trip through HBM; at most 16 splits.
static int dh_splits_for(int64_t num_rows, int64_t vocab, int n_nt, int num_sms) {
  const int64_t units = ((num_rows + kBwMtile - 1) / kBwMtile) * n_nt;
  const int64_t kb = (vocab + kBwK - 1) / kBwK;
  const int64_t pairs = std::max(1, num_sms / 2);
  int best = 1;
  double best_t = 1e300;
  // a split's fp32 partials cost 8 bytes per dh element (write + read) at ~5 TB/s, a stage ~0.55 us
  const double part_stages = double(num_rows) * double(n_nt) * kBwNtile * 8.0 / 5e12 / 0.55e-6;
  for (int s = 1; s <= 16; ++s) {
    const int64_t waves = (units * s + pairs - 1) / pairs;
    const double t = double(waves) * double((kb + s - 1) / s + 8) + (s > 1 ? s * part_stages : 0.0);
    if (t < best_t - 1e-9) {
      best_t = t;
      best = s;
    }
  }
  return best;
}
// dh runs as two launches when d > 512: hidden tile 0 with the transform (storing the dx tiles), then tiles
// 1 .. n-1 as a plain GEMM over those tiles — each with its own split-K
static void dh_plan(int64_t num_rows, int64_t vocab, int d, int num_sms, int* s0, int* s1) {
  const int n_nt = (d + kBwNtile - 1) / kBwNtile;
#ifdef OTK_BW_ONE_DH  // experiment: one dh launch, the transform in every hidden tile
  *s0 = *s1 = dh_splits_for(num_rows, vocab, n_nt, num_sms);
  return;
#endif
  *s0 = dh_splits_for(num_rows, vocab, 1, num_sms);
  *s1 = n_nt > 1 ? dh_splits_for(num_rows, vocab, n_nt - 1, num_sms) : 1;
#ifdef OTK_BW_S1  // experiment: the plain dh launch's split count
  if (n_nt > 1) *s1 = OTK_BW_S1;
#endif
}
// slices of the fp32 dh partial buffer [slices][num_rows][d] (1: no partials, dh written as bf16 directly)
int lmhead_dh_splits(int64_t num_rows, int64_t vocab, int d, int num_sms) {
  int s0, s1;
  dh_plan(num_rows, vocab, d, num_sms, &s0, &s1);
  return std::max(s0, s1);
}

static cudaError_t launch_bwd(const otk_ctx* ctx, int mode, bool ent, const CUtensorMap& ta, const CUtensorMap& tb,
                              const CUtensorMap& tdx, const LmBwdParams& p, cudaStream_t s) {
  auto kern = mode == 0 ? (ent ? k_lmhead_bwd<0, true> : k_lmhead_bwd<0, false>)
                        : (ent ? k_lmhead_bwd<1, true> : k_lmhead_bwd<1, false>);
  cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwSmemBytes);
  if (ea != cudaSuccess) return ea;
  const int units = p.n_mt * p.n_nt * p.splits;
  const int pairs = std::max(1, std::min(units, ctx->num_sms / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(2 * pairs), 1, 1);
  cfg.blockDim = dim3(kBwThreads, 1, 1);
  cfg.dynamicSmemBytes = kBwSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tdx, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_lmhead_bwd(const otk_ctx* ctx, int64_t num_rows, int64_t vocab, int d, const void* hidden,
                              const void* weight, const void* logits, void* dx_tiles, const float4* rowc,
                              const int32_t* targets, int64_t vocab_start, float logit_scale, bool ent, void* dh,
                              void* dw, float* dh_part, int dh_splits, cudaStream_t s, int* launches) {
  LmBwdParams p;
  p.num_rows = num_rows;
  p.vocab = vocab;
  p.d = d;
  p.n_nt = (d + kBwNtile - 1) / kBwNtile;
  p.rowc = rowc;
  p.targets = targets;
  p.vocab_start = vocab_start;
  p.s2 = logit_scale * 1.4426950408889634f;
  *launches = 0;
  const int64_t rows_pad = (num_rows + 255) / 256 * 256, cols_pad = (vocab + 255) / 256 * 256;
  // dh: A = x [N, V] K-major (box 64 vocab x 128 rows), B = W [V, d] MN-major (box 64 hidden x 64 vocab)
  {
    CUtensorMap ta, tb, tdx;
    if (!make_map_tiles(&ta, logits, rows_pad, cols_pad, 1, 2) || !make_map_2d(&tb, weight, vocab, d, d, 64, kBwK) ||
        !make_map_tiles(&tdx, dx_tiles, rows_pad, cols_pad, 1, 2))
      return cudaErrorInvalidValue;
    int s0, s1;
    dh_plan(num_rows, vocab, d, ctx->num_sms, &s0, &s1);
    p.n_mt = int((num_rows + kBwMtile - 1) / kBwMtile);
    p.kb_total = int((vocab + kBwK - 1) / kBwK);
    p.f32out = std::max(s0, s1) > 1 ? 1 : 0;
    p.out = p.f32out ? static_cast<void*>(dh_part) : dh;
    const int n_nt = p.n_nt;
#ifdef OTK_BW_ONE_DH
    const bool one = true;
#else
    const bool one = n_nt == 1;
#endif
    // (a) hidden tile 0 (every tile when `one`): the transform, and the dx tiles stored for the other GEMMs
    p.store_dx = 1;
    p.xform = 1;
    p.nt0 = 0;
    p.n_nt = one ? n_nt : 1;
    p.splits = s0;
    p.kb_per_split = (p.kb_total + s0 - 1) / s0;
    cudaError_t e = launch_bwd(ctx, 0, ent, ta, tb, tdx, p, s);
    if (e != cudaSuccess) return e;
    ++*launches;
    // (b) hidden tiles 1 .. n-1: a plain GEMM over the stored dx tiles (A K-major, the same tile layout as x)
    if (!one) {
      CUtensorMap tdxa;
      if (!make_map_tiles(&tdxa, dx_tiles, rows_pad, cols_pad, 1, 2)) return cudaErrorInvalidValue;
      p.store_dx = 0;
      p.xform = 0;
      p.nt0 = 1;
      p.n_nt = n_nt - 1;
      p.splits = s1;
      p.kb_per_split = (p.kb_total + s1 - 1) / s1;
      e = launch_bwd(ctx, 0, ent, tdxa, tb, tdxa, p, s);
      if (e != cudaSuccess) return e;
      ++*launches;
    }
    p.n_nt = n_nt;
    if (p.f32out) {
      const int64_t n4 = num_rows * d / 4;
      int64_t blocks = std::min<int64_t>((n4 + 255) / 256, int64_t(ctx->num_sms) * 8);
      k_lmhead_dh_reduce<<<int(blocks), 256, 0, s>>>(reinterpret_cast<const float4*>(dh_part), s0, one ? s0 : s1, d,
                                                       n4, reinterpret_cast<uint2*>(dh));
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      ++*launches;
    }
  }
  // dW = dxᵀ h: A = the dx tiles dh stored (boxes of 64 vocab x 64 rows, MN-major) — a plain GEMM, no transform;
  // B = h [N, d] MN-major (box 64 hidden x 64 rows)
  {
    CUtensorMap ta, tb;
    if (!make_map_tiles(&ta, dx_tiles, rows_pad, cols_pad, 2, 1) || !make_map_2d(&tb, hidden, num_rows, d, d, 64, kBwK))
      return cudaErrorInvalidValue;
    p.store_dx = 0;
    p.xform = 0;
    p.nt0 = 0;
    p.f32out = 0;
    p.n_mt = int((vocab + kBwMtile - 1) / kBwMtile);
    p.kb_total = int((num_rows + kBwK - 1) / kBwK);
    p.splits = 1;
    p.kb_per_split = p.kb_total;
    p.out = dw;
    cudaError_t e = launch_bwd(ctx, 1, ent, ta, tb, ta, p, s);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  return cudaSuccess;
}

}  // namespace otk

#ifdef OTK_BW_TIMING
extern "C" void otk_debug_bw(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, otk::g_bw_timing, sizeof(unsigned long long) * 32);
  unsigned long long z[32] = {0};
  cudaMemcpyToSymbol(otk::g_bw_timing, z, sizeof(z));
}
#endif
