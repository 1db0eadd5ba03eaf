// k_rows.cu — the fused vocab-row kernels behind otk_logprob_entropy_fwd (north_star (3)),
// otk_policy_loss_fwd_bwd (north_star (4)) and the vocab-sharded variants.
//
// k_rows_tm (modes FWD / PARTIAL / BWD / BWD_VPF): persistent CTAs (BWD: one per SM; FWD / PARTIAL: two per
// SM); a row is split over a thread-block cluster of `csize` CTAs (any size 1-8, the fewest whose segment fits
// kMaxChunks chunks; csize = 2 for bf16 V = 151936: 148 KB per CTA), the grid capped at the resident clusters.
//   warp 0, lane 0 : loader — 1-D bulk TMA (cp.async.bulk) of 12 KB chunks of every active row's segment into
//                    an 18-slot (216 KB; FWD / PARTIAL: 8-slot) shared-memory ring, L2 evict_first, paced by
//                    per-slot empty mbarriers. Loss-masked rows are never read.
//   warps 1..12    : consumers — read each chunk from the ring once (two 16-byte vectors per thread) and
//                    release the slot at once. Pass 1 (pass1_chunk): 2^(y - m) once per element (MUFU) with
//                    packed fp32x2 sums against a per-thread reference m set by the row's first chunk and
//                    raised only when a chunk's sums overflow; for the loss (BWD) e (bf16) and the chunk's
//                    reference m_c are parked in TENSOR MEMORY (9 columns per chunk in a 168-column window).
//                    Row total: warp shuffles + lane-parallel CTA combine + cluster exchange of 16-byte
//                    partials through DSMEM (st.async + mbarrier); K4-VPF adds the exchange with the other
//                    ranks over peer memory (epoch-tagged words). Pass 2 (pass2_row): softmax = e * 2^(m_c -
//                    lse) from tensor memory (no second read of the logits, no second exponential),
//                    dlogits = coef * (softmax - onehot) as bf16x2 products, 16-byte streaming stores.
//   warp 13        : BWD: zero-fills the dlogits of masked rows with bulk async stores; FWD / PARTIAL: the
//                    finalizer (row reduction, exchange and outputs off the consumers' critical path).
// k_rows_stream (mode BWD_PARTIALS, vocab shard): stats come from the all-gathered partials, so the
//   row is streamed once through the ring and written (one exponential per element).
// Rows with loss mask 0 are never read: their dlogits are zero-filled (write-only).
// All reductions run in a fixed order with explicitly rounded combine steps, so results are
// deterministic and bitwise identical between (3) and (4) and across the CTAs of a cluster.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "otk_internal.h"
#include "otk_ptx.cuh"


namespace otk {
using namespace ptx;

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kNCT = 32 * kConsumerWarps;
constexpr int kVPT = kChunkBytes / 16 / kNCT;  // 16-byte vectors per consumer thread per chunk (2)
static_assert(kVPT * kNCT * 16 == kChunkBytes, "chunk must split evenly over consumers");

// Running (max, sum 2^(y-m), sum 2^(y-m)(y-m)) in log2 units: y = log2(e) * s * x.
struct Stat {
  float m, s, t;
};

// combine / finalize use explicitly rounded ops (__fmul_rn / __fadd_rn are never contracted into
// FMAs), so every template instantiation and every CTA produces bitwise-identical row statistics.
__device__ __forceinline__ Stat combine(const Stat a, const Stat b) {
  const float M = fmaxf(a.m, b.m);
  if (M == -INFINITY) return a;
  float sa = 0.f, ta = 0.f, sb = 0.f, tb = 0.f;
  if (a.m != -INFINITY) {
    const float d = __fsub_rn(a.m, M), f = ex2(d);
    sa = __fmul_rn(a.s, f);
    ta = __fmul_rn(f, __fmaf_rn(d, a.s, a.t));
  }
  if (b.m != -INFINITY) {
    const float d = __fsub_rn(b.m, M), f = ex2(d);
    sb = __fmul_rn(b.s, f);
    tb = __fmul_rn(f, __fmaf_rn(d, b.s, b.t));
  }
  return Stat{M, __fadd_rn(sa, sb), __fadd_rn(ta, tb)};
}

struct RowStats {
  float L2;    // log2(e) * lse = m + lg2S (rounded: use m and lg2S separately where |m| is large)
  float m;     // the row total's reference (log2 units)
  float lg2S;  // log2 of the sum relative to m
  float logp;  // z_y - lse
  float H;     // entropy
  float lse;
};

// dy = log2(e) * s * x_y - t.m, formed with an FMA against the row reference (no cancellation between two
// large numbers, so logp keeps ~1e-6 absolute accuracy even for logits of magnitude 1e4).
__device__ __forceinline__ RowStats finalize(const Stat t, const float dy) {
  RowStats r;
  const float lg2S = lg2(t.s);
  r.m = t.m;
  r.lg2S = lg2S;
  r.L2 = __fadd_rn(t.m, lg2S);
  r.lse = __fmul_rn(r.L2, kLn2);
  r.logp = __fmul_rn(kLn2, __fsub_rn(dy, lg2S));
  r.H = __fmul_rn(kLn2, __fsub_rn(lg2S, __fdividef(t.t, t.s)));
  return r;
}

// Combine gathered vocab-shard partials (m, s, t, w) in rank order; w = s2*x_y - m of the shard holding the
// target (-inf on the others). Returns the row total and dy relative to its reference.
__device__ __forceinline__ Stat combine_partials(const float4* P, int64_t stride, int nshards, float& dy) {
  Stat tot{-INFINITY, 0.f, 0.f};
  for (int k = 0; k < nshards; ++k) {
    const float4 q = P[int64_t(k) * stride];
    tot = combine(tot, Stat{q.x, q.y, q.z});
  }
  dy = -INFINITY;
  for (int k = 0; k < nshards; ++k) {
    const float4 q = P[int64_t(k) * stride];
    if (q.w != -INFINITY) dy = __fadd_rn(q.w, __fsub_rn(q.x, tot.m));  // m_k - M is exact (Sterbenz)
  }
  return tot;
}

// ---- K4-VPF exchange buffer (one per rank, include/otk.h otk_vpf_peers): [2 parities][rows_cap][P] records of
// 32 bytes = four 64-bit words (value bits | epoch << 32) for m2, s, t2, w. Record (par, row, q) of rank p's
// buffer is written by rank q; a reader accepts it when all four words carry the call's epoch (each word is
// single-copy atomic, so a record is never half old, half new). Parity = epoch & 1: a rank can run at most
// one call ahead of a peer (it needs the peer's records of every row to finish a call), so the two record
// sets never collide.
__host__ __device__ __forceinline__ int64_t vpf_rec_index(int64_t cap, int nranks, uint32_t par, int64_t row, int q) {
  return (int64_t(par) * cap + row) * nranks + q;
}
constexpr uint64_t kVpfTimeoutNs = 20ull * 1000000000ull;
__device__ __forceinline__ uint64_t vpf_word(float v, uint32_t ep) {
  return uint64_t(__float_as_uint(v)) | (uint64_t(ep) << 32);
}

// The call's epoch: 1 + the calls completed on this buffer set, read from the device counter in the own buffer
// (the last CTA of the call bumps it), so a CUDA-graph replay gets a fresh epoch without host involvement.
__device__ __forceinline__ uint32_t vpf_epoch(const RowParams& p) {
  return *reinterpret_cast<volatile uint32_t*>(p.vpf_counter) + 1u;
}

// Push this rank's row partial `mine` = (m2, s, t2, w) into every peer's exchange buffer (one thread).
__device__ __forceinline__ void vpf_push(const RowParams& p, int64_t row, float4 mine, uint32_t ep) {
  const int P = p.vpf_nranks, me = p.vpf_rank;
  const uint32_t par = ep & 1u;
  const int64_t i = vpf_rec_index(p.vpf_rows_cap, P, par, row, me) * 32;
  const uint64_t w0 = vpf_word(mine.x, ep), w1 = vpf_word(mine.y, ep), w2 = vpf_word(mine.z, ep),
                 w3 = vpf_word(mine.w, ep);
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    char* b = reinterpret_cast<char*>(p.vpf_xchg[q]) + i;
    st_pair_sys(b, w0, w1);
    st_pair_sys(b + 16, w2, w3);
  }
}

// Collect the peers' records of `row` (waiting for this call's epoch) and combine all P partials in rank order
// exactly as combine_partials does (own = `mine`). Called by a whole warp: lane q waits for peer q's record, so
// the P - 1 round trips to peer memory overlap (the wait is the slowest peer's, not the sum); then every lane
// combines the P records in rank order (shuffles). Identical bits on every rank.
__device__ __forceinline__ Stat vpf_collect(const RowParams& p, int64_t row, float4 mine, float& dy, uint32_t ep,
                                            int lane) {
  const int P = p.vpf_nranks, me = p.vpf_rank;
  const uint32_t par = ep & 1u;
  const int64_t cap = p.vpf_rows_cap;
  const char* own = reinterpret_cast<const char*>(p.vpf_xchg[me]);
  float4 rec = make_float4(-INFINITY, 0.f, 0.f, -INFINITY);
  if (lane == me) {
    rec = mine;
  } else if (lane < P) {
    const char* r = own + vpf_rec_index(cap, P, par, row, lane) * 32;
    uint64_t a0, a1, a2, a3;
    auto ready = [&]() {
      ld_pair_sys(r, a0, a1);
      ld_pair_sys(r + 16, a2, a3);
      return uint32_t(a0 >> 32) == ep && uint32_t(a1 >> 32) == ep && uint32_t(a2 >> 32) == ep &&
             uint32_t(a3 >> 32) == ep;
    };
    bool ok = ready();
    if (!ok) {
      const uint64_t t0 = globaltimer_ns();
      while (!(ok = ready())) {
        // only a peer timeout of THIS call ends the wait early (a data error elsewhere never does: every
        // valid row still gets its peers' partials)
        if (*reinterpret_cast<volatile uint32_t*>(p.vpf_abort) == ep) break;
        if (globaltimer_ns() - t0 > kVpfTimeoutNs) {
          set_error(p.err, OTK_ERR_PEER_TIMEOUT);
          *reinterpret_cast<volatile uint32_t*>(p.vpf_abort) = ep;
          break;
        }
      }
    }
    if (ok)
      rec = make_float4(__uint_as_float(uint32_t(a0)), __uint_as_float(uint32_t(a1)), __uint_as_float(uint32_t(a2)),
                        __uint_as_float(uint32_t(a3)));
  }
  __syncwarp();
  Stat tot{-INFINITY, 0.f, 0.f};
  float wsel = -INFINITY, xsel = 0.f;
  for (int q = 0; q < P; ++q) {
    const float rx = __shfl_sync(0xffffffffu, rec.x, q), ry = __shfl_sync(0xffffffffu, rec.y, q),
                rz = __shfl_sync(0xffffffffu, rec.z, q), rw = __shfl_sync(0xffffffffu, rec.w, q);
    tot = combine(tot, Stat{rx, ry, rz});
    if (rw != -INFINITY) {  // the rank holding the target column (one)
      wsel = rw;
      xsel = rx;
    }
  }
  dy = wsel == -INFINITY ? -INFINITY : __fadd_rn(wsel, __fsub_rn(xsel, tot.m));  // m_k - M exact (Sterbenz)
  return tot;
}

// Before its first push a call (epoch ep) waits until every peer has completed call ep - 2: the records of call
// ep go to the parity buffer that call ep - 2 read. Normally the wait is immediate (finishing call ep - 1 needed
// the peers' records of ep - 1, so they were past ep - 2); it matters when call ep - 1 exchanged nothing (no
// active rows) and a fast rank would otherwise overwrite records a slow peer is still reading. One thread per CTA.
__device__ __forceinline__ void vpf_window(const RowParams& p, uint32_t ep) {
  if (ep <= 2u) return;
  const int64_t tail = int64_t(2) * p.vpf_rows_cap * p.vpf_nranks * 32;
  for (int q = 0; q < p.vpf_nranks; ++q) {
    if (q == p.vpf_rank) continue;
    const volatile uint32_t* c =
        reinterpret_cast<const volatile uint32_t*>(reinterpret_cast<const char*>(p.vpf_xchg[q]) + tail);
    if (*c + 2u >= ep) continue;
    const uint64_t t0 = globaltimer_ns();
    while (*c + 2u < ep) {
      if (*reinterpret_cast<volatile uint32_t*>(p.vpf_abort) == ep) return;
      if (globaltimer_ns() - t0 > kVpfTimeoutNs) {
        set_error(p.err, OTK_ERR_PEER_TIMEOUT);
        *reinterpret_cast<volatile uint32_t*>(p.vpf_abort) = ep;
        return;
      }
    }
  }
}

// Called by one warp per CTA after the CTA's (cluster's) row total: push (lane 0 of cluster rank 0), then collect
// and combine (the whole warp).
__device__ __forceinline__ Stat vpf_exchange(const RowParams& p, int64_t row, uint32_t crank, float4 mine, float& dy,
                                             uint32_t ep, int lane) {
  if (crank == 0 && lane == 0) vpf_push(p, row, mine, ep);
  __syncwarp();
  return vpf_collect(p, row, mine, dy, ep, lane);
}

// One element pair of pass 1: d = s2*x - m; e = 2^d; S += e; T += e*d (per-lane fp32 chains; kInit starts
// the chains instead of adding to them).
template <bool kInit>
__device__ __forceinline__ void pass1_pair(float xlo, float xhi, uint64_t s2x2, uint64_t negm2, uint64_t& accS,
                                           uint64_t& accT, float& e0, float& e1) {
  const uint64_t d2 = ffma2(f2(xlo, xhi), s2x2, negm2);
  float d0, d1;
  f2_split(d2, d0, d1);
  e0 = ex2(d0);
  e1 = ex2(d1);
  const uint64_t e2 = f2(e0, e1);
  if (kInit) {
    accS = e2;
    accT = fmul2(e2, d2);
  } else {
    accS = fadd2(accS, e2);
    accT = ffma2(e2, d2, accT);
  }
}

// ---- element-type traits ------------------------------------------------------------------------
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int EV = 4;
  __device__ static __forceinline__ void unpack(const uint4 v, float (&x)[4]) {
    x[0] = __uint_as_float(v.x);
    x[1] = __uint_as_float(v.y);
    x[2] = __uint_as_float(v.z);
    x[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float (&g)[4]) {
    return make_uint4(__float_as_uint(g[0]), __float_as_uint(g[1]), __float_as_uint(g[2]), __float_as_uint(g[3]));
  }
  // lanes >= nvalid become -1e30 (finite: e = 0 and e*d = 0, no NaN in the fast path)
  __device__ static __forceinline__ uint4 mask_tail(uint4 v, int nvalid) {
    constexpr uint32_t kLow = 0xf149f2cau;  // -1.0e30f
    return make_uint4(nvalid > 0 ? v.x : kLow, nvalid > 1 ? v.y : kLow, nvalid > 2 ? v.z : kLow,
                      nvalid > 3 ? v.w : kLow);
  }
  __device__ static __forceinline__ float vmax_acc(float acc, const uint4 v) {
    return fmaxf(acc, fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)),
                            fmaxf(__uint_as_float(v.z), __uint_as_float(v.w))));
  }
  using MaxAcc = float;
  __device__ static __forceinline__ float max_init() { return -INFINITY; }
  __device__ static __forceinline__ float max_acc(float acc, const uint4 v) { return vmax_acc(acc, v); }
  __device__ static __forceinline__ float max_final(float acc) { return acc; }
  __device__ static __forceinline__ float load1(const void* base, int64_t i) {
    return reinterpret_cast<const float*>(base)[i];
  }
  // pass 1 on one 16-byte vector (4 fp32 logits): e kept at full precision. kClamp maps -inf to -1e30.
  template <bool kKeepE, bool kClamp, bool kInit>
  __device__ static __forceinline__ uint4 pass1(const uint4 v, uint64_t s2x2, uint64_t negm2, uint64_t (&aS)[2],
                                                uint64_t (&aT)[2]) {
    float x[4], e[4];
    unpack(v, x);
    if (kClamp)
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = fmaxf(x[i], -1e30f);
    pass1_pair<kInit>(x[0], x[1], s2x2, negm2, aS[0], aT[0], e[0], e[1]);
    pass1_pair<kInit>(x[2], x[3], s2x2, negm2, aS[1], aT[1], e[2], e[3]);
    return kKeepE ? pack(e) : make_uint4(0, 0, 0, 0);
  }
  // e * 2^-64, exact (the underflow-safe split of pass2_row)
  __device__ static __forceinline__ uint4 scale_m64(const uint4 e) {
    const float k = 5.42101086242752217e-20f;  // 2^-64
    return make_uint4(__float_as_uint(__uint_as_float(e.x) * k), __float_as_uint(__uint_as_float(e.y) * k),
                      __float_as_uint(__uint_as_float(e.z) * k), __float_as_uint(__uint_as_float(e.w) * k));
  }
  // entropy-bonus variant: g = e (A + B log2 e)
  __device__ static __forceinline__ uint4 pass2_ent(const uint4 e, float A, float B) {
    float x[4], g[4];
    unpack(e, x);
#pragma unroll
    for (int i = 0; i < 4; ++i) g[i] = x[i] * fmaf(B, fmaxf(lg2(x[i]), -1e30f), A);
    return pack(g);
  }
  __device__ static __forceinline__ uint4 pass2(const uint4 e, float kt) {
    const uint64_t kt2 = f2(kt, kt);
    float g[4];
    f2_split(fmul2(f2(__uint_as_float(e.x), __uint_as_float(e.y)), kt2), g[0], g[1]);
    f2_split(fmul2(f2(__uint_as_float(e.z), __uint_as_float(e.w)), kt2), g[2], g[3]);
    return pack(g);
  }
  __device__ static __forceinline__ void store1(void* base, int64_t i, float v) {
    reinterpret_cast<float*>(base)[i] = v;
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int EV = 8;
  __device__ static __forceinline__ void unpack(const uint4 v, float (&x)[8]) {
    x[0] = bf_lo(v.x), x[1] = bf_hi(v.x), x[2] = bf_lo(v.y), x[3] = bf_hi(v.y);
    x[4] = bf_lo(v.z), x[5] = bf_hi(v.z), x[6] = bf_lo(v.w), x[7] = bf_hi(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float (&g)[8]) {
    return make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]), pack_bf16x2(g[4], g[5]),
                      pack_bf16x2(g[6], g[7]));
  }
  // lanes >= nvalid become -1e30 (bf16 0xf14a: finite, so e = 0 and e*d = 0 without NaN)
  __device__ static __forceinline__ uint32_t mask_word(uint32_t w, int lane0, int nvalid) {
    if (lane0 >= nvalid) return 0xf14af14au;
    if (lane0 + 1 >= nvalid) return (w & 0x0000ffffu) | 0xf14a0000u;
    return w;
  }
  __device__ static __forceinline__ uint4 mask_tail(uint4 v, int nvalid) {
    return make_uint4(mask_word(v.x, 0, nvalid), mask_word(v.y, 2, nvalid), mask_word(v.z, 4, nvalid),
                      mask_word(v.w, 6, nvalid));
  }
  using MaxAcc = uint32_t;  // packed bf16x2 running max
  __device__ static __forceinline__ uint32_t max_init() { return 0xff80ff80u; }
  __device__ static __forceinline__ uint32_t max_acc(uint32_t acc, const uint4 v) {
    return bmax2(acc, bmax2(bmax2(v.x, v.y), bmax2(v.z, v.w)));
  }
  __device__ static __forceinline__ float max_final(uint32_t acc) { return fmaxf(bf_lo(acc), bf_hi(acc)); }
  __device__ static __forceinline__ float load1(const void* base, int64_t i) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  }
  // pass 1 on one 16-byte vector (8 bf16 logits). kClamp (the exact path) maps -inf to -1e30 with one packed
  // max per pair, so e = 0 and e*d = 0. e = 2^(y - m) is kept as bf16 (relative error 2^-9).
  template <bool kClamp, bool kInit>
  __device__ static __forceinline__ uint32_t pass1_word(uint32_t w, uint64_t s2x2, uint64_t negm2, uint64_t& aS,
                                                        uint64_t& aT) {
    if (kClamp) w = bmax2(w, 0xf14af14au);  // bf16x2(-1.0e30)
    float e0, e1;
    pass1_pair<kInit>(bf_lo(w), bf_hi(w), s2x2, negm2, aS, aT, e0, e1);
    return pack_bf16x2(e0, e1);
  }
  template <bool kKeepE, bool kClamp, bool kInit>
  __device__ static __forceinline__ uint4 pass1(const uint4 v, uint64_t s2x2, uint64_t negm2, uint64_t (&aS)[2],
                                                uint64_t (&aT)[2]) {
    uint4 r;
    r.x = pass1_word<kClamp, kInit>(v.x, s2x2, negm2, aS[0], aT[0]);
    r.y = pass1_word<kClamp, kInit>(v.y, s2x2, negm2, aS[1], aT[1]);
    r.z = pass1_word<kClamp, false>(v.z, s2x2, negm2, aS[0], aT[0]);
    r.w = pass1_word<kClamp, false>(v.w, s2x2, negm2, aS[1], aT[1]);
    return r;
  }
  // g = e * kt directly in bf16x2: kt is split into kt_hi + kt_lo (both bf16), g = fma(e, kt_hi, e * kt_lo)
  // rounds once to bf16 (the kt split keeps 16 significant bits): 2 instructions per pair of elements.
  __device__ static __forceinline__ uint32_t pass2_word(uint32_t w, uint32_t hi2, uint32_t lo2) {
    uint32_t t, r;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(t) : "r"(w), "r"(lo2));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(hi2), "r"(t));
    return r;
  }
  // e * 2^-64, exact (bf16x2 multiply by a power of two; the underflow-safe split of pass2_row)
  __device__ static __forceinline__ uint32_t scale_m64_word(uint32_t w) {
    uint32_t r;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(0x1F801F80u));  // bf16x2(2^-64)
    return r;
  }
  __device__ static __forceinline__ uint4 scale_m64(const uint4 e) {
    return make_uint4(scale_m64_word(e.x), scale_m64_word(e.y), scale_m64_word(e.z), scale_m64_word(e.w));
  }
  // entropy-bonus variant: g = e (A + B log2 e) in fp32, rounded once to bf16
  __device__ static __forceinline__ uint4 pass2_ent(const uint4 e, float A, float B) {
    float x[8], g[8];
    unpack(e, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = x[i] * fmaf(B, fmaxf(lg2(x[i]), -1e30f), A);
    return pack(g);
  }
  __device__ static __forceinline__ uint4 pass2(const uint4 e, float kt) {
    const uint32_t hi2 = pack_bf16x2(kt, kt);
    const float khi = bf_lo(hi2);
    const uint32_t lo2 = pack_bf16x2(__fsub_rn(kt, khi), __fsub_rn(kt, khi));
    return make_uint4(pass2_word(e.x, hi2, lo2), pass2_word(e.y, hi2, lo2), pass2_word(e.z, hi2, lo2),
                      pass2_word(e.w, hi2, lo2));
  }
  __device__ static __forceinline__ void store1(void* base, int64_t i, float v) {
    reinterpret_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
  }
};

struct Smem {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t xbar[4];
  float4 xrecv[4][8];                 // peer partials, by active-row parity (pipelined loop: row index mod 4)
  float4 wred[2][kConsumerWarps];     // warp partials, double-buffered by active-row parity
  // FWD / PARTIAL: warp partials handed to the finalizer warp through a ring of kFinSlots rows
  uint64_t ffull[4];                  // all consumer warps wrote slot k (count kConsumerWarps)
  uint64_t fempty[4];                 // the finalizer has read slot k (count 1)
  float4 fred[4][kConsumerWarps];
  float4 rowbc[2];                    // (stream kernel) row broadcast
  float4 vbc[2];                      // (K4-VPF) the rank-order row total + dy, broadcast by thread 0
  struct Pend {                       // (pipelined loop) a row whose stage B is pending, by active-row index mod 4
    int64_t row, nb;                  // row < 0: end of this CTA's rows (K4-VPF collector)
    double A;
    float old_lp, ref_lp, rm, rs, rt, xy, dyl;
    int32_t y, ylc, owner, side_ok;
  } pend[4];
  uint64_t pfull[4];                  // (pipelined K4-VPF) pend[k] written (thread 0 -> collector warp)
  uint64_t cfull[4];                  // (pipelined K4-VPF) the rank-order total of row k is in ctot[k]
  float4 ctot[4];
  uint32_t tmem_base;
  long long load_row;                 // the loader's current row (zero-fill pacing; INT64_MAX when done)
};
constexpr int kZeroBytes = 4096;  // zero block: source of the bulk stores that zero-fill masked rows
constexpr size_t kRingBytes = size_t(kSlots) * kChunkBytes;
constexpr size_t kSmemBytes = kRingBytes + kZeroBytes + sizeof(Smem);
constexpr size_t smem_bytes_for(int ns) { return size_t(ns) * kChunkBytes + kZeroBytes + sizeof(Smem); }

__device__ __forceinline__ bool row_active(const RowParams& p, int32_t y, uint8_t m) {
  return m && y >= 0 && int64_t(y) < p.vocab_total;
}

// ---- loader (warp 0, one thread): bulk-TMA every active row's column segment, chunk by chunk, into the ring
template <typename T, int NS = kSlots>
__device__ __forceinline__ void load_rows(const RowParams& p, uint8_t* ring, Smem& S, int64_t group, int64_t ngroups,
                                          int64_t c0, uint32_t seg_bytes, int nch) {
  const uint64_t pol = policy_evict_first();
  const char* base = reinterpret_cast<const char*>(p.logits) + c0 * int64_t(sizeof(T));
  const int64_t row_bytes = p.ld * int64_t(sizeof(T));
  uint32_t slot = 0, phase = 0;
  int64_t row = group;
  int32_t y_n = row < p.num_rows ? p.targets[row] : 0;
  uint8_t m_n = (row < p.num_rows && p.mask) ? p.mask[row] : 1;
  for (; row < p.num_rows; row += ngroups) {
    const int32_t y = y_n;
    const uint8_t m = m_n;
    const int64_t nrow = row + ngroups;
    if (nrow < p.num_rows) {
      y_n = p.targets[nrow];
      m_n = p.mask ? p.mask[nrow] : 1;
    }
    if (!row_active(p, y, m)) continue;
#ifndef OTK_NO_ZERO_PACING
    *reinterpret_cast<volatile long long*>(&S.load_row) = row;  // masked rows before this one may be zero-filled
#endif
    const char* src = base + row * row_bytes;
    uint32_t off = 0;
    for (int c = 0; c < nch; ++c) {
      mbar_wait(&S.empty[slot], phase ^ 1u);
      const uint32_t bytes = min(uint32_t(kChunkBytes), seg_bytes - off);
      mbar_arrive_expect_tx(&S.full[slot], bytes);
      bulk_g2s(ring + size_t(slot) * kChunkBytes, src + off, bytes, &S.full[slot], pol);
      off += kChunkBytes;
      if (++slot == NS) {
        slot = 0;
        phase ^= 1u;
      }
    }
  }
  *reinterpret_cast<volatile long long*>(&S.load_row) = 0x7fffffffffffffffll;
}

// ---- zero-filler (warp 13, one thread): the dlogits segment of every inactive row is written with bulk
// async shared->global stores from a zeroed 4 KB block — never read, never touched by the consumers ----------
template <typename T>
__device__ __forceinline__ void zero_rows(const RowParams& p, const uint8_t* zero, Smem& S, int64_t group,
                                          int64_t ngroups, int64_t c0, int segn) {
  if (!p.zero_masked) return;
  const uint32_t zero_bytes = (uint32_t(segn) * uint32_t(sizeof(T))) & ~15u;  // 16-byte multiple part
  if (!zero_bytes) return;
  const uint64_t pol = policy_evict_first();
  char* dbase = reinterpret_cast<char*>(p.dlogits) + c0 * int64_t(sizeof(T));
  const int64_t row_bytes = p.ld * int64_t(sizeof(T));
  bool pending = false;
  for (int64_t row = group; row < p.num_rows; row += ngroups) {
    const int32_t y = p.targets[row];
    const uint8_t m = p.mask ? p.mask[row] : 1;
    if (row_active(p, y, m)) continue;
#ifndef OTK_NO_ZERO_PACING
    // paced by the loader: a masked row is zero-filled only once the loader has reached the rows around it, so
    // DRAM sees the write-only rows interleaved with the read+write rows instead of a write burst up front
    while (*reinterpret_cast<volatile long long*>(&S.load_row) < row) __nanosleep(128);
#endif
    char* dst = dbase + row * row_bytes;
    for (uint32_t off = 0; off < zero_bytes; off += kZeroBytes)
      bulk_s2g(dst + off, zero, min(uint32_t(kZeroBytes), zero_bytes - off), pol);
    bulk_commit();
    bulk_wait_read_8();
    pending = true;
  }
  if (pending) bulk_wait_all();
}

// ---- rows that are never read (R26): outputs 0; the dlogits zero-fill is the producer's bulk
// stores, except a sub-16-byte tail at the end of the vocabulary, written here ---------------------------
template <typename T, int MODE>
__device__ __forceinline__ void inactive_row(const RowParams& p, int64_t row, int ct, uint32_t crank, int64_t c0,
                                             int segn, bool bad_target) {
  if (bad_target && ct == 0 && crank == 0) set_error(p.err, OTK_ERR_TARGET_RANGE);
  if (ct != 0) return;
  if (MODE == kModeBwd || MODE == kModeBwdPartials || MODE == kModeBwdVpf) {
    if (p.zero_masked) {
      char* base = reinterpret_cast<char*>(p.dlogits) + (row * p.ld + c0) * int64_t(sizeof(T));
      const int done = int(((uint32_t(segn) * uint32_t(sizeof(T))) & ~15u) / sizeof(T));
      for (int k = done; k < segn; ++k) Vec<T>::store1(base, k, 0.f);
    }
    if (crank == 0) {
      if (p.logp) p.logp[row] = 0.f;
      if (p.entropy) p.entropy[row] = 0.f;
    }
  } else if (crank == 0) {
    if (MODE == kModeFwd) {
      p.logp[row] = 0.f;
      if (p.entropy) p.entropy[row] = 0.f;
      if (p.lse) p.lse[row] = 0.f;
    } else {
      p.partials_out[row] = make_float4(-INFINITY, 0.f, 0.f, -INFINITY);
    }
  }
}

// ---- per-token loss (north_star (4); same definition as oracle_ref.row_loss_terms), fp32 ---------------
struct LossOut {
  float L, kl;  // L = pg + beta*KL - c_H*H (unweighted)
  float w;      // row weight of the reduction (token mean: 1/N)
  float coef;   // -s * w * dL/dlogp
  float wcs;    // w * c_H * s: scale of the entropy-bonus gradient p (ln p + H)
  float gy;     // the target column's dlogit: coef (p_y - 1) + wcs p_y (logp + H)
  bool clipped;
};
struct RowSide {
  double A;
  float old_lp, ref_lp;
  int64_t nb;   // loss tokens of the row's trajectory (sequence-mean reductions)
};
// e^x via MUFU (relative error ~2^-22) and expm1 with a degree-5 Taylor branch near 0 (|x| < 1/4: relative
// error < 2e-6, no cancellation) — the per-row loss terms only need fp32-level accuracy.
__device__ __forceinline__ float exp_fast(float x) { return ex2(__fmul_rn(x, kLog2e)); }
__device__ __forceinline__ float expm1_fast(float x) {
  const float t = fmaf(x, fmaf(x, fmaf(x, fmaf(x, fmaf(x, 1.f / 120.f, 1.f / 24.f), 1.f / 6.f), 0.5f), 1.f), 0.f);
  return fabsf(x) < 0.25f ? t : exp_fast(x) - 1.f;
}

// Row weight w_j (R17, R29): token mean 1/N, seq-mean-token-mean 1/(n_b B), seq-mean-token-sum 1/B.
__device__ __forceinline__ float row_weight(const RowParams& p, float invN, int64_t nb, int64_t nact) {
  if (p.reduction == OTK_TOKEN_MEAN) return invN;
  if (nact <= 0) return 0.f;
  if (p.reduction == OTK_SEQ_MEAN_TOKEN_SUM) return float(1.0 / double(nact));
  return nb > 0 ? float(1.0 / (double(nb) * double(nact))) : 0.f;
}

// A_j and n_b of a trainable row. An index outside adv (row_traj[j] or adv_index[j] vs num_adv) or outside
// traj_tokens (sequence-mean reductions) is a data error: OTK_ERR_GROUP_RANGE (reported by `reporter`), and the
// row is treated as loss-masked (weight 0: zero gradient, no stats, logp / entropy 0) — never read out of bounds.
__device__ __forceinline__ bool row_side(const RowParams& p, int64_t row, int32_t rt, RowSide& sd, bool reporter) {
  const int64_t ai = p.adv_index ? int64_t(p.adv_index[row]) : int64_t(rt);
  const bool seq = p.reduction != OTK_TOKEN_MEAN;
  const bool ok = ai >= 0 && ai < p.num_adv && (!seq || (rt >= 0 && int64_t(rt) < p.num_traj));
  if (!ok) {
    if (reporter) set_error(p.err, OTK_ERR_GROUP_RANGE);
    sd.A = 0.0;
    sd.nb = 0;
    return false;
  }
  sd.A = p.adv[ai];
  if (seq) sd.nb = p.traj_tokens[rt];
  return true;
}

__device__ __forceinline__ LossOut loss_terms(const RowParams& p, float lp, float H, const RowSide& sd, float w) {
  const float C = float(p.clamp);
  bool clipped = false;
  float pg, G;
  if (p.sft) {  // supervised cross-entropy on the trainable tokens
    pg = -lp;
    G = -1.f;
  } else {
    const float A = float(sd.A);
    const float draw = lp - sd.old_lp;
    const float delta = fminf(fmaxf(draw, -C), C);
    const float r = exp_fast(delta);
    const float lo = float(1.0 - p.clip_low), hi = float(1.0 + p.clip_high);
    const float rbar = fminf(fmaxf(r, lo), hi);
    pg = fmaxf(-A * r, -A * rbar);
    clipped = (A > 0.f && r > hi) || (A < 0.f && r < lo);
    G = (clipped || fabsf(draw) > C) ? 0.f : -A * r;
    const float dc = float(p.dual_clip);
    if (dc > 0.f && A < 0.f && pg > -dc * A) {  // dual clip: cap at -c*A, zero gradient
      pg = -dc * A;
      G = 0.f;
    }
  }
  float kl = 0.f;
  const float beta = float(p.kl_beta);
  if (beta != 0.f) {
    float gk;
    if (p.kl_type == OTK_KL_K3) {
      const float dr = sd.ref_lp - lp;
      const float d = fminf(fmaxf(dr, -C), C);
      const float em1 = expm1_fast(d);
      kl = em1 - d;           // e^d - d - 1 without cancellation
      gk = fabsf(dr) > C ? 0.f : -em1;
    } else if (p.kl_type == OTK_KL_K1) {
      kl = lp - sd.ref_lp;
      gk = 1.f;
    } else {
      kl = 0.5f * (lp - sd.ref_lp) * (lp - sd.ref_lp);
      gk = lp - sd.ref_lp;
    }
    G = fmaf(beta, gk, G);
  }
  const float ce = float(p.ent_coef);
  LossOut o;
  o.L = fmaf(-ce, H, fmaf(beta, kl, pg));
  o.kl = kl;
  o.clipped = clipped;
  o.w = w;
  o.coef = -p.scale * w * G;
  o.wcs = w * ce * p.scale;
  o.gy = o.coef * expm1_fast(lp);  // coef * (p_y - 1), no cancellation when p_y -> 1
  if (ce != 0.f) o.gy = fmaf(o.wcs * exp_fast(lp), lp + H, o.gy);
  return o;
}

// vblock / vgrid: the CTA's index and count within this call (a grouped launch hosts several calls)
__device__ __forceinline__ void stats_epilogue(const RowParams& p, double acc_L, double acc_clip, double acc_kl,
                                               double acc_H, double acc_n, int64_t nl, unsigned vblock, unsigned vgrid,
                                               uint32_t vpf_ep = 0) {
  double* part = p.cta_partials + size_t(vblock) * kStatSlots;
  part[0] = acc_L;
  part[1] = acc_clip;
  part[2] = acc_kl;
  part[3] = acc_H;
  part[4] = acc_n;
  __threadfence();
  const unsigned int t = atomicAdd(p.ticket, 1u);
  if (t == vgrid - 1) {
    __threadfence();
    double tot[5] = {0, 0, 0, 0, 0};
    for (unsigned int b = 0; b < vgrid; ++b) {
      const volatile double* q2 = p.cta_partials + size_t(b) * kStatSlots;
      for (int k = 0; k < 5; ++k) tot[k] += q2[k];
    }
    (void)nl;
    otk_loss_stats* o = p.stats;
    if (p.accumulate) {
      o->loss += tot[0];
      o->n_clipped += tot[1];
      o->kl_sum += tot[2];
      o->entropy_sum += tot[3];
      o->n_tokens += tot[4];
    } else {
      o->loss = tot[0];
      o->n_clipped = tot[1];
      o->kl_sum = tot[2];
      o->entropy_sum = tot[3];
      o->n_tokens = tot[4];
    }
    if (p.vpf_counter) *p.vpf_counter = vpf_ep;  // K4-VPF: this call is complete on this rank
    *p.ticket = 0u;
  }
}

// Shared setup of both row kernels: barriers, zero block, optional TMEM allocation (warp 1).
template <bool kTmem>
__device__ __forceinline__ void row_kernel_setup(Smem& S, uint8_t* zero, int warp, int csize) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kConsumerWarps);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&S.xbar[i], 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&S.ffull[i], kConsumerWarps);
      mbar_init(&S.fempty[i], 1);
      mbar_init(&S.pfull[i], 1);
      mbar_init(&S.cfull[i], 1);
    }
    S.load_row = -1;
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < kZeroBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(zero)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();  // the bulk-store engine (async proxy) must see the zeros
  if (kTmem && warp == 1) {  // one warp owns the TMEM allocation (all 512 columns; 1 CTA per SM)
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  if (csize > 1)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
}

// Warp-wide (max, sum-exp, sum-exp*d): max first, one rescale per lane, then two butterfly sums. Every lane
// ends with the same bits (butterfly addition is commutative), so all warps agree without a broadcast.
__device__ __forceinline__ Stat warp_reduce(Stat st) {
  float M = st.m;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  float s = 0.f, t = 0.f;
  if (st.m != -INFINITY) {
    const float d = __fsub_rn(st.m, M), f = ex2(d);
    s = __fmul_rn(st.s, f);
    t = __fmul_rn(f, __fmaf_rn(d, st.s, st.t));
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, off));
  }
  return Stat{M, s, t};
}

// Row statistics after pass 1. Warp partials go through shared memory; every warp then reduces the 12
// partials lane-parallel (identical result in every thread, so no second barrier and no broadcast), and
// thread 0 exchanges the CTA total with the cluster peers through DSMEM (rank-order combine).
__device__ __forceinline__ void row_total(Smem& S, Stat st, int lane, int cw, int ct, int csize, uint32_t crank,
                                          uint32_t q, Stat& tot) {
  const uint32_t par = q & 1u;
  st = warp_reduce(st);
  if (lane == 0) S.wred[par][cw] = make_float4(st.m, st.s, st.t, 0.f);
  named_bar_sync(1, kNCT);
  Stat mine{-INFINITY, 0.f, 0.f};
  if (lane < kConsumerWarps) {
    const float4 w = S.wred[par][lane];
    mine = Stat{w.x, w.y, w.z};
  }
  const Stat r = warp_reduce(mine);
  if (csize > 1) {
    if (ct == 0) {
      for (int dst = 0; dst < csize; ++dst) {
        if (dst == int(crank)) continue;
        st_async_f4(mapa(smem_u32(&S.xrecv[par][crank]), dst), r.m, r.s, r.t, 0.f, mapa(smem_u32(&S.xbar[par]), dst));
      }
      mbar_arrive_expect_tx(&S.xbar[par], 16u * uint32_t(csize - 1));
    }
    mbar_wait(&S.xbar[par], (q >> 1) & 1u);
    if (csize == 2) {  // the common case (bf16 V = 151936): one combine, rank order
      const float4 P = S.xrecv[par][crank ^ 1u];
      const Stat peer{P.x, P.y, P.z};
      tot = crank == 0 ? combine(r, peer) : combine(peer, r);
    } else {
      tot = Stat{-INFINITY, 0.f, 0.f};
      for (int k = 0; k < csize; ++k) {
        const float4 P = (k == int(crank)) ? make_float4(r.m, r.s, r.t, 0.f) : S.xrecv[par][k];
        tot = combine(tot, Stat{P.x, P.y, P.z});
      }
    }
  } else {
    tot = r;
  }
}

// FWD / PARTIAL finalizer (warp kConsumerWarps + 1, idle in these modes otherwise): takes each active row's 12
// warp partials from the fred ring, reduces them exactly as row_total does (same order, same rounded ops, so
// logp is bitwise equal to the BWD kernel's), exchanges with the cluster peers and writes the row's outputs.
// The consumer warps therefore never wait for a row's reduction: they hand off their partial and stream on.
template <typename T, int MODE>
__device__ __forceinline__ void finalize_rows(const RowParams& p, Smem& S, int lane, int csize, uint32_t crank,
                                              int64_t group, int64_t ngroups) {
  using VT = Vec<T>;
  const float s2 = __fmul_rn(p.scale, kLog2e);
  uint32_t fs = 0, fph = 0, q = 0;
  int64_t row = group;
  int32_t y_n = 0;
  uint8_t m_n = 0;
  if (row < p.num_rows) {
    y_n = p.targets[row];
    m_n = p.mask ? p.mask[row] : 1;
  }
  auto xy_of = [&](int64_t r, int32_t yy) -> float {
    const int64_t g = int64_t(yy) - p.vocab_start;
    return (g >= 0 && g < p.vocab) ? VT::load1(p.logits, r * p.ld + g) : 0.f;
  };
  float xy_n = (row < p.num_rows && row_active(p, y_n, m_n)) ? xy_of(row, y_n) : 0.f;
  for (; row < p.num_rows; row += ngroups) {
    const int32_t y = y_n;
    const uint8_t m = m_n;
    const float xy = xy_n;
    const int64_t nrow = row + ngroups;
    if (nrow < p.num_rows) {
      y_n = p.targets[nrow];
      m_n = p.mask ? p.mask[nrow] : 1;
    }
    if (!row_active(p, y, m)) {  // the consumers wrote this row's zeros
      if (nrow < p.num_rows && row_active(p, y_n, m_n)) xy_n = xy_of(nrow, y_n);
      continue;
    }
    mbar_wait(&S.ffull[fs], fph);
    Stat mine{-INFINITY, 0.f, 0.f};
    if (lane < kConsumerWarps) {
      const float4 w = S.fred[fs][lane];
      mine = Stat{w.x, w.y, w.z};
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.fempty[fs]);
    if (++fs == 4) {
      fs = 0;
      fph ^= 1u;
    }
    if (nrow < p.num_rows && row_active(p, y_n, m_n)) xy_n = xy_of(nrow, y_n);
    const Stat r = warp_reduce(mine);
    Stat tot;
    const uint32_t par = q & 1u;
    if (csize > 1) {
      if (lane == 0) {
        for (int dst = 0; dst < csize; ++dst) {
          if (dst == int(crank)) continue;
          st_async_f4(mapa(smem_u32(&S.xrecv[par][crank]), dst), r.m, r.s, r.t, 0.f, mapa(smem_u32(&S.xbar[par]), dst));
        }
        mbar_arrive_expect_tx(&S.xbar[par], 16u * uint32_t(csize - 1));
      }
      mbar_wait(&S.xbar[par], (q >> 1) & 1u);
      if (csize == 2) {
        const float4 P = S.xrecv[par][crank ^ 1u];
        const Stat peer{P.x, P.y, P.z};
        tot = crank == 0 ? combine(r, peer) : combine(peer, r);
      } else {
        tot = Stat{-INFINITY, 0.f, 0.f};
        for (int k = 0; k < csize; ++k) {
          const float4 P = (k == int(crank)) ? make_float4(r.m, r.s, r.t, 0.f) : S.xrecv[par][k];
          tot = combine(tot, Stat{P.x, P.y, P.z});
        }
      }
    } else {
      tot = r;
    }
    const int64_t yg = int64_t(y) - p.vocab_start;
    const float dy = (yg >= 0 && yg < p.vocab) ? __fmaf_rn(xy, s2, -tot.m) : -INFINITY;
    if (lane == 0 && crank == 0) {
      if (MODE == kModePartial) {
        p.partials_out[row] = make_float4(tot.m, tot.s, tot.t, dy);
      } else {
        const RowStats rs = finalize(tot, dy);
        p.logp[row] = rs.logp;
        if (p.entropy) p.entropy[row] = rs.H;
        if (p.lse) p.lse[row] = rs.lse;
      }
    }
    ++q;
  }
}

#ifdef OTK_PHASE_TIMING
__device__ unsigned long long g_phase[8];  // experiments only: clock64 sums per phase (warp lane 0 of consumers)
#endif

// Pass 2 of one row segment, shared by the row loops: dlogits = e * (coef * 2^(m_c - lse)) from tensor memory (e of
// chunk c at columns tm + 8c, its reference m_c at tm + kColM + c). The TMEM load of chunk c+1 is in flight while
// chunk c is scaled and stored (two register sets, ping-pong, no copies). The entropy-bonus form (one extra MUFU,
// log2 e, per element) is selected once per row. The caller then stores the target column.
template <typename T, int kColM>
__device__ __forceinline__ void pass2_row(char* drow, uint32_t tm, int ct, int nch, int segn, const RowStats& rs,
                                          const LossOut& lo) {
  using VT = Vec<T>;
  constexpr int EV = VT::EV;
  constexpr int CE = kChunkBytes / int(sizeof(T));
  char* tp = drow + ct * 16;
  auto chunk2 = [&](int c, const uint4& e0, const uint4& e1, uint32_t mw, auto entf) {
    constexpr bool kEnt = decltype(entf)::value;
    // m_c - lse (log2 units) as (m_c - m) - lg2S: the difference of the two references first (exact when they are
    // close), so rows of large-magnitude logits (|m| ~ 1e4: fp32 ulp 2^-10) keep full relative accuracy in p
    float dm = __fsub_rn(__fsub_rn(__uint_as_float(mw), rs.m), rs.lg2S);
    uint4 e0s = e0, e1s = e1;
    if (dm < -64.f) {  // 2^dm would flush to 0 while e (up to 2^64) times it need not: move 2^-64 into e (exact)
      e0s = VT::scale_m64(e0);
      e1s = VT::scale_m64(e1);
      dm = __fadd_rn(dm, 64.f);
    }
    const float qc = ex2(dm);
    uint4 g0, g1;
    if constexpr (!kEnt) {
      const float kt = __fmul_rn(lo.coef, qc);
      g0 = VT::pass2(e0s, kt);
      g1 = VT::pass2(e1s, kt);
    } else {  // g = e q (coef + wcs (ln2 (log2 e + m_c - lse) + H))
      const float Ac = qc * fmaf(lo.wcs, fmaf(kLn2, dm, rs.H), lo.coef);
      const float Bc = qc * lo.wcs * kLn2;
      g0 = VT::pass2_ent(e0s, Ac, Bc);
      g1 = VT::pass2_ent(e1s, Ac, Bc);
    }
    char* q0 = tp + size_t(c) * kChunkBytes;
    if (c < nch - 1 || (c + 1) * CE <= segn) {
      stg_cs_v4(q0, g0);
      stg_cs_v4(q0 + kNCT * 16, g1);
    } else {  // last, partial chunk
      const uint4 gg[2] = {g0, g1};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int lc = c * CE + (ct + k * kNCT) * EV;
        if (lc + EV <= segn) {
          stg_cs_v4(q0 + k * kNCT * 16, gg[k]);
        } else if (lc < segn) {
          float g[EV];
          VT::unpack(gg[k], g);
          for (int i = 0; i < EV && lc + i < segn; ++i) VT::store1(drow, lc + i, g[i]);
        }
      }
    }
  };
  auto pass2 = [&](auto entf) {
    uint4 a0, a1, b0, b1;
    uint32_t am, bm;
    tmem_ld8_1_issue(tm, tm + uint32_t(kColM), a0, a1, am);
    tmem_wait_ld_dep(a0, a1, am);
    for (int c = 0;;) {
      if (c + 1 < nch) tmem_ld8_1_issue(tm + uint32_t(8 * (c + 1)), tm + uint32_t(kColM + c + 1), b0, b1, bm);
      chunk2(c, a0, a1, am, entf);
      if (++c >= nch) break;
      tmem_wait_ld_dep(b0, b1, bm);
      if (c + 1 < nch) tmem_ld8_1_issue(tm + uint32_t(8 * (c + 1)), tm + uint32_t(kColM + c + 1), a0, a1, am);
      chunk2(c, b0, b1, bm, entf);
      if (++c >= nch) break;
      tmem_wait_ld_dep(a0, a1, am);
    }
  };
  if (lo.wcs == 0.f)
    pass2(std::false_type{});
  else
    pass2(std::true_type{});
}

// One chunk of pass 1, shared by the row loops: wait for the ring slot, read this thread's two 16-byte vectors,
// release the slot at once, and add (sum e, sum e*d) of the chunk to the row accumulators (rS, rT) against the row
// reference mref. mref is set by the row's first chunk (exact path) and raised only when a chunk's partial sums
// overflow 2^64 or turn NaN (a -inf logit) — then the chunk is redone on the exact path (clamp, packed max,
// rescale) — so the common chunk needs neither a max reduction nor a rescale. kTail: the segment's last chunk
// (lanes past segn become -1e30). e0 / e1: the chunk's exponentials (kKeepE: for the tensor-memory copy).
template <typename T, bool kKeepE, bool kTail, int NS>
__device__ __forceinline__ void pass1_chunk(Smem& S, const uint8_t* ring, uint32_t& slot, uint32_t& phase, int ct,
                                            int lane, int c, int segn, float s2, uint64_t s2x2, float& mref,
                                            uint64_t& rS, uint64_t& rT, uint4& e0, uint4& e1) {
  using VT = Vec<T>;
  constexpr int EV = VT::EV;
  constexpr int CE = kChunkBytes / int(sizeof(T));
  mbar_wait(&S.full[slot], phase);
  const uint8_t* buf = ring + size_t(slot) * kChunkBytes;
  uint4 v0 = *reinterpret_cast<const uint4*>(buf + ct * 16);
  uint4 v1 = *reinterpret_cast<const uint4*>(buf + (ct + kNCT) * 16);
  if constexpr (kTail) {
    const int lc0 = c * CE + ct * EV, lc1 = lc0 + kNCT * EV;
    if (lc0 + EV > segn) v0 = VT::mask_tail(v0, segn - lc0);
    if (lc1 + EV > segn) v1 = VT::mask_tail(v1, segn - lc1);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&S.empty[slot]);
  if (++slot == NS) {
    slot = 0;
    phase ^= 1u;
  }
  uint64_t cS[2], cT[2];
  bool ok = false;
  if (mref != -INFINITY) {  // fast path: fixed reference, no clamp
    const uint64_t negm2 = f2(-mref, -mref);
    e0 = VT::template pass1<kKeepE, false, true>(v0, s2x2, negm2, cS, cT);
    e1 = VT::template pass1<kKeepE, false, false>(v1, s2x2, negm2, cS, cT);
    const uint64_t sS = fadd2(cS[0], cS[1]), sT = fadd2(cT[0], cT[1]);
    float s0, s1, t0, t1;
    f2_split(sS, s0, s1);
    f2_split(sT, t0, t1);
    ok = fmaxf(s0, s1) <= 0x1p64f && !isnan(t0 + t1);  // also false for inf / NaN sums
    cS[0] = sS;
    cT[0] = sT;
  }
  if (!ok) {  // exact path: the row's first chunk, an overflow, or -inf logits
    // lanes at or below -1e30 (masked tails, clamped -inf) never set the reference: with a reference that
    // large, s2*x - m would be dominated by the rounding residual of the product
    const float mx = VT::max_final(VT::max_acc(VT::max_acc(VT::max_init(), v0), v1));
    if (mx > -1e30f) {
      const float mn = fmaxf(mref, __fmul_rn(mx, s2));
      if (mn > mref) {
        if (mref != -INFINITY) {
          const float d = __fsub_rn(mref, mn), f = ex2(d);
          const uint64_t f2x = f2(f, f);
          rT = fmul2(f2x, ffma2(f2(d, d), rS, rT));
          rS = fmul2(rS, f2x);
        }
        mref = mn;
      }
    }
    const float mr = (mref == -INFINITY) ? 0.f : mref;
    const uint64_t negm2 = f2(-mr, -mr);
    e0 = VT::template pass1<kKeepE, true, true>(v0, s2x2, negm2, cS, cT);
    e1 = VT::template pass1<kKeepE, true, false>(v1, s2x2, negm2, cS, cT);
    cS[0] = fadd2(cS[0], cS[1]);
    cT[0] = fadd2(cT[0], cT[1]);
  }
  rS = fadd2(rS, cS[0]);
  rT = fadd2(rT, cT[0]);
}

// =====================================================================================================
// Pipelined K4-VPF consumer (kPipe; segments of <= kPipeChunks chunks, so TWO rows fit a warp's TMEM window).
// Stage A(r): pass 1 of row r into TMEM half (q & 1), CTA reduction, then the row partial is SENT (cluster
// peers through DSMEM; K4-VPF csize 1: the peer ranks) but not awaited. Stage B(r-1): wait for the previous
// row's partials, loss terms, pass 2 from the other TMEM half. Order A(r), B(r-1), A(r+1), B(r), ...: the
// exchange latency of a row (and the skew between the CTAs / ranks sharing it) is hidden behind a whole
// pass 1. Cluster mailboxes are indexed by active-row index mod 4: a peer can be at most 3 rows ahead of the
// row being read (its A(r+4) needs our A(r+2), which follows our B(r)).
// =====================================================================================================
// Generalised to a lag of L rows (template kLag): L + 1 row slots in the warp's TMEM window, stage B(r - L) after
// stage A(r), so L whole passes 1 hide a row's exchange and the skew between the ranks sharing it. Lag 1: slots
// of 64 columns (segments <= 7 chunks: K4-VPF P = 4 at V = 151936); lag 3: four slots of 42 columns (<= 4 chunks:
// P >= 8).
template <int kLag>
struct PipeCfg {
  static constexpr int kSlotCols = kLag == 1 ? 64 : kTmemWindow / 4;   // TMEM columns per row slot
  static constexpr int kMaxCh = kLag == 1 ? kPipeChunks : kLag3Chunks;  // chunks per row segment
  static constexpr int kColM = 8 * kMaxCh;                        // [0, kColM) e, then one m_c column per chunk
  static_assert((kLag + 1) * kSlotCols <= kTmemWindow && kColM + kMaxCh <= kSlotCols, "TMEM slots");
  static_assert(kLag == 1 || kLag == 3, "lag 1 or 3 (slot index = q & kLag)");
};

struct PipeRow {
  int64_t row;
  RowSide sd;
  Stat r;          // this CTA's partial (cluster rank order combine in stage B)
  float xy;
  int32_t y;
  int ylc, owner;
  uint32_t q;
  bool side_ok;
};

template <typename T, int MODE, int kLag>
__device__ __forceinline__ void consumer_pipe(const RowParams& p, Smem& S, uint8_t* ring, int warp, int lane,
                                              int csize, uint32_t crank, int64_t group, int64_t ngroups, int64_t c0,
                                              int segn, int nch, unsigned vblock, unsigned vgrid) {
  constexpr bool kVpf = (MODE == kModeBwdVpf);
  using VT = Vec<T>;
  constexpr int EV = VT::EV;
  constexpr int CE = kChunkBytes / int(sizeof(T));
  constexpr int kColM = PipeCfg<kLag>::kColM;
  constexpr int kSlotCols = PipeCfg<kLag>::kSlotCols;
  const int ct = threadIdx.x - 32;
  const int cw = warp - 1;
  const uint32_t tm0 = S.tmem_base + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(kTmemWindow * (cw >> 2));
  const float s2 = __fmul_rn(p.scale, kLog2e);
  const uint64_t s2x2 = f2(s2, s2);
  double acc_L = 0.0, acc_clip = 0.0, acc_kl = 0.0, acc_H = 0.0, acc_n = 0.0;
  const int64_t nl = *p.n_loss;
  const float invN = nl > 0 ? float(1.0 / double(nl)) : 0.f;
  const int64_t nact = p.reduction != OTK_TOKEN_MEAN ? *p.n_active : 0;
  uint32_t slot = 0, phase = 0, q = 0;
  const uint32_t vep = (kVpf && ct < 32) ? vpf_epoch(p) : 0u;  // the collecting warp, before the ticket
  if (kVpf && ct == 0) vpf_window(p, vep);

  // ---- stage B: a pending row's statistics, loss and pass 2 (its record in S.pend, written by thread 0 in its
  // stage A, kLag rows ago — named barriers in between; the slot is rewritten only after every thread has passed
  // the next stage A's barrier, i.e. left this stage B)
  auto stage_b = [&](uint32_t qb) {
    const Smem::Pend& pe = S.pend[qb & 3u];
    PipeRow pr;
    pr.row = pe.row;
    pr.sd = RowSide{pe.A, pe.old_lp, pe.ref_lp, pe.nb};
    pr.r = Stat{pe.rm, pe.rs, pe.rt};
    pr.xy = pe.xy;
    pr.y = pe.y;
    pr.ylc = pe.ylc;
    pr.owner = pe.owner;
    pr.q = qb;
    pr.side_ok = pe.side_ok != 0;
    const uint32_t k = pr.q & 3u;
    Stat tot;
    if (csize > 1) {
      mbar_wait(&S.xbar[k], (pr.q >> 2) & 1u);
      tot = Stat{-INFINITY, 0.f, 0.f};
      for (int c = 0; c < csize; ++c) {
        const float4 P = (c == int(crank)) ? make_float4(pr.r.m, pr.r.s, pr.r.t, 0.f) : S.xrecv[k][c];
        tot = combine(tot, Stat{P.x, P.y, P.z});
      }
    } else {
      tot = pr.r;
    }
    const int64_t yg = int64_t(pr.y) - p.vocab_start;
    float dy = (yg >= 0 && yg < p.vocab) ? __fmaf_rn(pr.xy, s2, -tot.m) : -INFINITY;
    if constexpr (kVpf) {  // csize 1 here: pushed in stage A, collected by the collector warp meanwhile
      mbar_wait(&S.cfull[k], (pr.q >> 2) & 1u);
      const float4 b = S.ctot[k];
      tot = Stat{b.x, b.y, b.z};
      dy = b.w;
    }
    const RowStats rs = finalize(tot, dy);
    const LossOut lo = loss_terms(p, rs.logp, rs.H, pr.sd, pr.side_ok ? row_weight(p, invN, pr.sd.nb, nact) : 0.f);
    if (ct == 0 && crank == 0) {
      if (pr.side_ok) {
        acc_L += double(lo.w) * double(lo.L);
        acc_clip += lo.clipped ? 1.0 : 0.0;
        acc_kl += double(lo.kl);
        acc_H += double(rs.H);
        acc_n += 1.0;
      }
      if (p.logp) p.logp[pr.row] = pr.side_ok ? rs.logp : 0.f;
      if (p.entropy) p.entropy[pr.row] = pr.side_ok ? rs.H : 0.f;
    }
    const uint32_t tm = tm0 + (pr.q & uint32_t(kLag)) * kSlotCols;
    char* drow = reinterpret_cast<char*>(p.dlogits) + (pr.row * p.ld + c0) * int64_t(sizeof(T));
    pass2_row<T, kColM>(drow, tm, ct, nch, segn, rs, lo);
    if (ct == pr.owner) VT::store1(drow, pr.ylc, lo.gy);
  };

  int64_t row = group;
  int32_t y_n = 0, rt_n = 0;
  uint8_t m_n = 1;
  float old_n = 0.f, ref_n = 0.f;
  if (row < p.num_rows) {
    y_n = p.targets[row];
    m_n = p.mask ? p.mask[row] : 1;
    rt_n = p.row_traj[row];
    old_n = p.old_logp[row];
    if (p.ref_logp) ref_n = p.ref_logp[row];
  }
  auto xy_of = [&](int64_t r, int32_t yy) -> float {
    const int64_t g = int64_t(yy) - p.vocab_start;
    return (g >= 0 && g < p.vocab) ? VT::load1(p.logits, r * p.ld + g) : 0.f;
  };
  float xy_n = (row < p.num_rows && row_active(p, y_n, m_n)) ? xy_of(row, y_n) : 0.f;
  int npend = 0;  // rows whose stage B is pending: active-row indices q - npend .. q - 1
  for (; row < p.num_rows; row += ngroups) {
    const int32_t y = y_n;
    const uint8_t m = m_n;
    const float xy = xy_n;
    RowSide sd{0.0, old_n, ref_n, 0};
    const int32_t rt = rt_n;
    const int64_t nrow = row + ngroups;
    if (nrow < p.num_rows) {
      y_n = p.targets[nrow];
      m_n = p.mask ? p.mask[nrow] : 1;
      rt_n = p.row_traj[nrow];
      old_n = p.old_logp[nrow];
      if (p.ref_logp) ref_n = p.ref_logp[nrow];
    }
    if (!row_active(p, y, m)) {
      inactive_row<T, MODE>(p, row, ct, crank, c0, segn, m != 0);
      if (nrow < p.num_rows && row_active(p, y_n, m_n)) xy_n = xy_of(nrow, y_n);
      continue;
    }
    const int64_t ylc64 = int64_t(y) - p.vocab_start - c0;
    const int ylc = (ylc64 >= 0 && ylc64 < segn) ? int(ylc64) : -1;
    const bool side_ok = row_side(p, row, rt, sd, ct == 0 && crank == 0);
    const uint32_t tm = tm0 + (q & uint32_t(kLag)) * kSlotCols;

    // ---------------- stage A: pass 1 into TMEM half (q & 1) (same arithmetic as the unpipelined loop)
    uint64_t rS = 0ull, rT = 0ull;
    float mref = -INFINITY;
    auto chunk1 = [&](int c, auto tail) {
      uint4 e0, e1;
      pass1_chunk<T, true, decltype(tail)::value, kSlots>(S, ring, slot, phase, ct, lane, c, segn, s2, s2x2, mref, rS,
                                                          rT, e0, e1);
      tmem_st8(tm + uint32_t(8 * c), e0, e1);
      tmem_st1(tm + uint32_t(kColM + c), __float_as_uint(mref == -INFINITY ? 0.f : mref));
    };
    for (int c = 0; c < nch - 1; ++c) chunk1(c, std::false_type{});
    if (nch > 0) chunk1(nch - 1, std::true_type{});
    if (nrow < p.num_rows && row_active(p, y_n, m_n)) xy_n = xy_of(nrow, y_n);
    tmem_wait_st();
    // CTA reduction (as row_total), then send without waiting
    const uint32_t par = q & 1u, k = q & 3u;
    const Stat wst = warp_reduce(Stat{mref, f2_sum(rS), f2_sum(rT)});
    if (lane == 0) S.wred[par][cw] = make_float4(wst.m, wst.s, wst.t, 0.f);
    named_bar_sync(1, kNCT);
    Stat mine{-INFINITY, 0.f, 0.f};
    if (lane < kConsumerWarps) {
      const float4 w = S.wred[par][lane];
      mine = Stat{w.x, w.y, w.z};
    }
    const Stat r = warp_reduce(mine);
    if (ct == 0) {
      if (csize > 1) {
        for (int dst = 0; dst < csize; ++dst) {
          if (dst == int(crank)) continue;
          st_async_f4(mapa(smem_u32(&S.xrecv[k][crank]), dst), r.m, r.s, r.t, 0.f, mapa(smem_u32(&S.xbar[k]), dst));
        }
        mbar_arrive_expect_tx(&S.xbar[k], 16u * uint32_t(csize - 1));
      }
      if constexpr (kVpf) {  // csize 1: this CTA's partial is the rank's
        const int64_t yg = int64_t(y) - p.vocab_start;
        const float dyl = (yg >= 0 && yg < p.vocab) ? __fmaf_rn(xy, s2, -r.m) : -INFINITY;
        vpf_push(p, row, make_float4(r.m, r.s, r.t, dyl), vep);
        S.pend[q & 3u].dyl = dyl;
      }
    }
    if (ct == 0) {
      Smem::Pend& pe = S.pend[q & 3u];
      pe.row = row;
      pe.nb = sd.nb;
      pe.A = sd.A;
      pe.old_lp = sd.old_lp;
      pe.ref_lp = sd.ref_lp;
      pe.rm = r.m;
      pe.rs = r.s;
      pe.rt = r.t;
      pe.xy = xy;
      pe.y = y;
      pe.ylc = ylc;
      pe.owner = ylc >= 0 ? ((ylc % CE) / EV) % kNCT : -1;
      pe.side_ok = side_ok ? 1 : 0;
      if constexpr (kVpf) mbar_arrive(&S.pfull[q & 3u]);  // the collector may start on this row
    }
    // ---------------- stage B of the row kLag rows back (its partials have had kLag passes 1 to arrive)
    if (npend == kLag) {
      stage_b(q - uint32_t(kLag));
      --npend;
    }
    ++npend;
    ++q;
  }
  // thread 0 wrote the last pending record after the last stage A's barrier: one more barrier before reading it
  named_bar_sync(1, kNCT);
  if constexpr (kVpf) {
    if (ct == 0) {  // end of rows for the collector (slot q & 3 was last read in stage B(q - 4), before the barrier)
      S.pend[q & 3u].row = -1;
      mbar_arrive(&S.pfull[q & 3u]);
    }
  }
  for (; npend > 0; --npend) stage_b(q - uint32_t(npend));
  if (ct == 0) stats_epilogue(p, acc_L, acc_clip, acc_kl, acc_H, acc_n, nl, vblock, vgrid, vep);
}

// =====================================================================================================
// k_rows_tm: FWD / PARTIAL / BWD. Pass 1 streams each chunk from the ring exactly once (slot released
// right away); for BWD the exponentials e = 2^(y - m_c) (bf16 for bf16 input, with m_c the thread's
// running max after chunk c) and m_c are parked in TENSOR MEMORY, so pass 2 needs no second read of the
// logits and no second exponential: softmax = e * 2^(m_c - lse).
// =====================================================================================================
// Pipelined K4-VPF collector (warp kConsumerWarps + 2): for each active row in order, once thread 0 has pushed
// the row's partial and recorded it in S.pend, wait for the P - 1 peer records (lane q: peer q), combine them in
// rank order and hand the total to stage B through S.ctot / S.cfull — the round trips to peer memory run beside
// the consumers' passes instead of in front of every stage B.
__device__ __forceinline__ void vpf_collector(const RowParams& p, Smem& S, int lane) {
  const uint32_t ep = vpf_epoch(p);  // before this CTA's ticket (taken by thread 0 of the consumers at the end)
  for (uint32_t k = 0;; ++k) {
    mbar_wait(&S.pfull[k & 3u], (k >> 2) & 1u);
    const Smem::Pend& pe = S.pend[k & 3u];
    const int64_t row = pe.row;
    if (row < 0) break;
    float gdy;
    const Stat g = vpf_collect(p, row, make_float4(pe.rm, pe.rs, pe.rt, pe.dyl), gdy, ep, lane);
    if (lane == 0) {
      S.ctot[k & 3u] = make_float4(g.m, g.s, g.t, gdy);
      mbar_arrive(&S.cfull[k & 3u]);
    }
    __syncwarp();
  }
}

template <typename T, int MODE, int kPipe>
__device__ __forceinline__ void rows_tm_body(const RowParams& p, unsigned vblock, unsigned vgrid) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr bool kVpf = (MODE == kModeBwdVpf);  // BWD with the vocab-shard exchange fused in
  constexpr bool kBwd = (MODE == kModeBwd) || kVpf;
  constexpr int NS = kBwd ? kSlots : kSlotsFwd;  // ring slots (FWD / PARTIAL: two CTAs per SM)
  uint8_t* ring = smem;
  uint8_t* zero = smem + size_t(NS) * kChunkBytes;
  Smem& S = *reinterpret_cast<Smem*>(smem + size_t(NS) * kChunkBytes + kZeroBytes);
  using VT = Vec<T>;
  constexpr int EV = VT::EV;
  constexpr int CE = kChunkBytes / int(sizeof(T));
  constexpr int kColM = 8 * kMaxChunks;  // per-thread TMEM columns: [0, 8*kMaxChunks) e, then m_c
  static_assert(kColM + kMaxChunks <= kTmemWindow, "TMEM window too small");
  static_assert(kConsumerWarps / 4 * kTmemWindow <= 512, "TMEM has 512 columns");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int csize = p.csize;
  const uint32_t crank = csize > 1 ? cluster_ctarank() : 0u;
  const int64_t group = vblock / csize;
  const int64_t ngroups = vgrid / csize;
  const int64_t c0 = int64_t(crank) * p.seg_elems;
  const int64_t c1 = min(p.vocab, c0 + int64_t(p.seg_elems));
  const int segn = c1 > c0 ? int(c1 - c0) : 0;
  const uint32_t seg_bytes = (uint32_t(segn) * uint32_t(sizeof(T)) + 15u) & ~15u;
  const int nch = int((seg_bytes + kChunkBytes - 1) / kChunkBytes);  // <= kMaxChunks (host-checked)

  row_kernel_setup<kBwd>(S, zero, warp, csize);

  if (warp == 0) {
    if (lane == 0 && nch > 0) load_rows<T, NS>(p, ring, S, group, ngroups, c0, seg_bytes, nch);
    __syncwarp();
  } else if (warp == kConsumerWarps + 1) {
    if (kBwd) {
      if (lane == 0) zero_rows<T>(p, zero, S, group, ngroups, c0, segn);
    } else {
      finalize_rows<T, MODE>(p, S, lane, csize, crank, group, ngroups);
    }
    __syncwarp();
  } else if (warp == kConsumerWarps + 2) {
    if constexpr (kVpf && kPipe > 0) vpf_collector(p, S, lane);  // the 15th warp exists for these kernels only
  } else if constexpr (kPipe > 0) {
    consumer_pipe<T, MODE, kPipe>(p, S, ring, warp, lane, csize, crank, group, ngroups, c0, segn, nch, vblock, vgrid);
  } else {
    const int ct = threadIdx.x - 32;
    const int cw = warp - 1;
    // this warp's TMEM window: its lane quadrant (warp % 4) and one of three 128-column windows
    const uint32_t tm = kBwd ? S.tmem_base + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(kTmemWindow * (cw >> 2)) : 0u;
    const float s2 = __fmul_rn(p.scale, kLog2e);
    const uint64_t s2x2 = f2(s2, s2);
    double acc_L = 0.0, acc_clip = 0.0, acc_kl = 0.0, acc_H = 0.0, acc_n = 0.0;
    int64_t nl = 0;
    float invN = 0.f;
    int64_t nact = 0;
    if (kBwd) {
      nl = *p.n_loss;
      invN = nl > 0 ? float(1.0 / double(nl)) : 0.f;
      if (p.reduction != OTK_TOKEN_MEAN) nact = *p.n_active;
    }
    uint32_t slot = 0, phase = 0, q = 0;
    uint32_t fs = 0, fph = 0;  // FWD / PARTIAL: hand-off ring to the finalizer warp
    const uint32_t vep = (kVpf && ct < 32) ? vpf_epoch(p) : 0u;  // the collecting warp, before the ticket
    if (kVpf && ct == 0) vpf_window(p, vep);

    int64_t row = group;
    int32_t y_n = 0, rt_n = 0;
    uint8_t m_n = 1;
    float old_n = 0.f, ref_n = 0.f;
    if (row < p.num_rows) {
      y_n = p.targets[row];
      m_n = p.mask ? p.mask[row] : 1;
      if (kBwd) {
        rt_n = p.row_traj[row];
        old_n = p.old_logp[row];
        if (p.ref_logp) ref_n = p.ref_logp[row];
      }
    }
    // the target logit, read straight from HBM (one sector per row), one row ahead: issued once the next
    // row's target has arrived (after this row's pass 1), consumed by the next row's finalize
    auto xy_of = [&](int64_t r, int32_t yy) -> float {
      const int64_t g = int64_t(yy) - p.vocab_start;
      return (g >= 0 && g < p.vocab) ? VT::load1(p.logits, r * p.ld + g) : 0.f;
    };
    float xy_n = (row < p.num_rows && row_active(p, y_n, m_n)) ? xy_of(row, y_n) : 0.f;
#ifdef OTK_PHASE_TIMING
    unsigned long long ph_a = 0, ph_b = 0, ph_c = 0, ph_d = 0, ph_in = 0;
    long long t_prev = clock64();
#endif
    for (; row < p.num_rows; row += ngroups) {
      const int32_t y = y_n;
      const uint8_t m = m_n;
      const float xy = xy_n;
      RowSide sd{0.0, old_n, ref_n, 0};
      const int32_t rt = rt_n;
      const int64_t nrow = row + ngroups;
      if (nrow < p.num_rows) {  // side data of the next row: in flight while this row is computed
        y_n = p.targets[nrow];
        m_n = p.mask ? p.mask[nrow] : 1;
        if (kBwd) {
          rt_n = p.row_traj[nrow];
          old_n = p.old_logp[nrow];
          if (p.ref_logp) ref_n = p.ref_logp[nrow];
        }
      }
      if (!row_active(p, y, m)) {
        inactive_row<T, MODE>(p, row, ct, crank, c0, segn, m != 0);
        if (nrow < p.num_rows && row_active(p, y_n, m_n)) xy_n = xy_of(nrow, y_n);
#ifdef OTK_PHASE_TIMING
        t_prev = clock64();
#endif
        continue;
      }
      const int64_t ylc64 = int64_t(y) - p.vocab_start - c0;  // target column local to this CTA's segment
      const int ylc = (ylc64 >= 0 && ylc64 < segn) ? int(ylc64) : -1;
      bool side_ok = true;
      if (kBwd) side_ok = row_side(p, row, rt, sd, ct == 0 && crank == 0);  // consumed after pass 1
      const int64_t yg = int64_t(y) - p.vocab_start;

      // ---------------- pass 1: online max / sum 2^(y-m) / sum 2^(y-m)(y-m), one exponential per element
      const int owner_ct = ylc >= 0 ? ((ylc % CE) / EV) % kNCT : -1;  // thread that stores the target column
      // Row-level pair accumulators of (sum e, sum e*d). The reference max mref is set by the row's first
      // chunk (exact path) and raised only when a chunk's values overflow 2^64 or hold -inf — detected from
      // the chunk's partial sums — so the common chunk needs neither a max reduction nor a rescale.
      uint64_t rS = 0ull, rT = 0ull;
      float mref = -INFINITY;
      // one chunk of pass 1; kTail only for the segment's last chunk (lanes past segn become -1e30)
      auto chunk1 = [&](int c, auto tail) {
        uint4 e0, e1;
        pass1_chunk<T, kBwd, decltype(tail)::value, NS>(S, ring, slot, phase, ct, lane, c, segn, s2, s2x2, mref, rS,
                                                        rT, e0, e1);
        if (kBwd) {
          tmem_st8(tm + uint32_t(8 * c), e0, e1);
          tmem_st1(tm + uint32_t(kColM + c), __float_as_uint(mref == -INFINITY ? 0.f : mref));
        }
      };
      for (int c = 0; c < nch - 1; ++c) chunk1(c, std::false_type{});
      if (nch > 0) chunk1(nch - 1, std::true_type{});
      if (nrow < p.num_rows && row_active(p, y_n, m_n)) xy_n = xy_of(nrow, y_n);
      const Stat st{mref, f2_sum(rS), f2_sum(rT)};
      if (!kBwd) {  // hand the warp partial to the finalizer and stream on (no per-row barrier)
        const Stat wst = warp_reduce(st);
        if (lane == 0) {
          mbar_wait(&S.fempty[fs], fph ^ 1u);
          S.fred[fs][cw] = make_float4(wst.m, wst.s, wst.t, 0.f);
          mbar_arrive(&S.ffull[fs]);
        }
        if (++fs == 4) {
          fs = 0;
          fph ^= 1u;
        }
        continue;
      }
      if (kBwd) tmem_wait_st();
#ifdef OTK_PHASE_TIMING
      const long long t_b = clock64();
      ph_a += t_b - t_prev;
#endif

      Stat tot;
      row_total(S, st, lane, cw, ct, csize, crank, q, tot);
#ifdef OTK_PHASE_TIMING
      const long long t_c = clock64();
      ph_b += t_c - t_b;
#endif
      float dy = (yg >= 0 && yg < p.vocab) ? __fmaf_rn(xy, s2, -tot.m) : -INFINITY;
      if constexpr (kVpf) {  // this rank's partial -> peers; peers' partials -> rank-order total (global row)
        if (ct < 32) {
          float gdy;
          const Stat g = vpf_exchange(p, row, crank, make_float4(tot.m, tot.s, tot.t, dy), gdy, vep, lane);
          if (ct == 0) S.vbc[q & 1u] = make_float4(g.m, g.s, g.t, gdy);
        }
        named_bar_sync(2, kNCT);
        const float4 b = S.vbc[q & 1u];
        tot = Stat{b.x, b.y, b.z};
        dy = b.w;
      }
      if (MODE == kModePartial) {
        if (ct == 0 && crank == 0) p.partials_out[row] = make_float4(tot.m, tot.s, tot.t, dy);
      } else {
        const RowStats rs = finalize(tot, dy);
        if (MODE == kModeFwd) {
          if (ct == 0 && crank == 0) {
            p.logp[row] = rs.logp;
            if (p.entropy) p.entropy[row] = rs.H;
            if (p.lse) p.lse[row] = rs.lse;
          }
        } else {
          const LossOut lo = loss_terms(p, rs.logp, rs.H, sd, side_ok ? row_weight(p, invN, sd.nb, nact) : 0.f);
          if (ct == 0 && crank == 0) {
            if (side_ok) {
              acc_L += double(lo.w) * double(lo.L);
              acc_clip += lo.clipped ? 1.0 : 0.0;
              acc_kl += double(lo.kl);
              acc_H += double(rs.H);
              acc_n += 1.0;
            }
            if (p.logp) p.logp[row] = side_ok ? rs.logp : 0.f;
            if (p.entropy) p.entropy[row] = side_ok ? rs.H : 0.f;
          }
          // ---------------- pass 2: dlogits = e * (coef * 2^(m_c - lse)) from TMEM; the TMEM load of chunk
          // c+1 is in flight while chunk c is scaled and stored (two register sets, ping-pong, no copies)
          char* drow = reinterpret_cast<char*>(p.dlogits) + (row * p.ld + c0) * int64_t(sizeof(T));
          pass2_row<T, kColM>(drow, tm, ct, nch, segn, rs, lo);
          // target column: coef * (p_y - 1), overwriting this thread's own vector store (program order)
          if (ct == owner_ct) VT::store1(drow, ylc, lo.gy);
#ifdef OTK_PHASE_TIMING
          ph_c += clock64() - t_c;
#endif
        }
      }
      ++q;
#ifdef OTK_PHASE_TIMING
      t_prev = clock64();
#endif
    }
#ifdef OTK_PHASE_TIMING
    if (kBwd && lane == 0) {
      atomicAdd(&g_phase[0], ph_a);
      atomicAdd(&g_phase[1], ph_b);
      atomicAdd(&g_phase[2], ph_c);
      atomicAdd(&g_phase[3], 1ull);
    }
#endif
    if (kBwd && ct == 0) stats_epilogue(p, acc_L, acc_clip, acc_kl, acc_H, acc_n, nl, vblock, vgrid, vep);
  }
  tc_fence_before();
  if (csize > 1)
    cluster_sync_all();
  else
    __syncthreads();
  if (kBwd && warp == 1) {  // (kBwd includes K4-VPF)
    tc_fence_after();
    tmem_dealloc(S.tmem_base, 512);
  }
}

template <typename T, int MODE, int kPipe = 0>
__global__ void __launch_bounds__(kThreads + (kPipe > 0 ? 32 : 0), 1) k_rows_tm(const RowParams p) {
  rows_tm_body<T, MODE, kPipe>(p, blockIdx.x, gridDim.x);
}

// K4-VPF ranks emulated on ONE GPU in ONE launch (otk_policy_loss_fwd_bwd_vpf_group): CTA block b runs call
// b / blocks_per_set as its CTA b % blocks_per_set. Every rank's CTAs are resident together by construction
// (cooperative launch, or a checked resident-cluster count), so the in-kernel exchange never waits on a rank
// the hardware has not scheduled — unlike separate launches on separate streams, which CUDA does not co-schedule.
struct RowParamsSet {
  RowParams p[OTK_VPF_MAX_RANKS];
  int nsets;
  int blocks_per_set;
};
template <typename T, int kPipe>
__global__ void __launch_bounds__(kThreads + (kPipe > 0 ? 32 : 0), 1) k_rows_vpf_group(const __grid_constant__ RowParamsSet ps) {
  const unsigned set = blockIdx.x / unsigned(ps.blocks_per_set);
  rows_tm_body<T, kModeBwdVpf, kPipe>(ps.p[set], blockIdx.x - set * unsigned(ps.blocks_per_set),
                                       unsigned(ps.blocks_per_set));
}

// =====================================================================================================
// k_rows_stream: BWD on a vocab shard from all-gathered partials (no pass 1): stream, write, release
// =====================================================================================================
template <typename T>
__global__ void __launch_bounds__(kThreads, 1) k_rows_stream(const RowParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint8_t* zero = smem + kRingBytes;
  Smem& S = *reinterpret_cast<Smem*>(smem + kRingBytes + kZeroBytes);
  using VT = Vec<T>;
  constexpr int EV = VT::EV;
  constexpr int CE = kChunkBytes / int(sizeof(T));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int csize = p.csize;
  const uint32_t crank = csize > 1 ? cluster_ctarank() : 0u;
  const int64_t group = blockIdx.x / csize;
  const int64_t ngroups = gridDim.x / csize;
  const int64_t c0 = int64_t(crank) * p.seg_elems;
  const int64_t c1 = min(p.vocab, c0 + int64_t(p.seg_elems));
  const int segn = c1 > c0 ? int(c1 - c0) : 0;
  const uint32_t seg_bytes = (uint32_t(segn) * uint32_t(sizeof(T)) + 15u) & ~15u;
  const int nch = int((seg_bytes + kChunkBytes - 1) / kChunkBytes);

  row_kernel_setup<false>(S, zero, warp, csize);

  if (warp == 0) {
    if (lane == 0 && nch > 0) load_rows<T>(p, ring, S, group, ngroups, c0, seg_bytes, nch);
    __syncwarp();
  } else if (warp == kConsumerWarps + 1) {
    if (lane == 0) zero_rows<T>(p, zero, S, group, ngroups, c0, segn);
    __syncwarp();
  } else {
    const int ct = threadIdx.x - 32;
    const float s2 = __fmul_rn(p.scale, kLog2e);
    double acc_L = 0.0, acc_clip = 0.0, acc_kl = 0.0, acc_H = 0.0, acc_n = 0.0;
    const int64_t nl = *p.n_loss;
    const float invN = nl > 0 ? float(1.0 / double(nl)) : 0.f;
    const int64_t nact = p.reduction != OTK_TOKEN_MEAN ? *p.n_active : 0;
    uint32_t slot = 0, phase = 0, q = 0;
    int64_t row = group;
    int32_t y_n = row < p.num_rows ? p.targets[row] : 0;
    uint8_t m_n = (row < p.num_rows && p.mask) ? p.mask[row] : 1;
    for (; row < p.num_rows; row += ngroups) {
      const int32_t y = y_n;
      const uint8_t m = m_n;
      const int64_t nrow = row + ngroups;
      if (nrow < p.num_rows) {
        y_n = p.targets[nrow];
        m_n = p.mask ? p.mask[nrow] : 1;
      }
      if (!row_active(p, y, m)) {
        inactive_row<T, kModeBwdPartials>(p, row, ct, crank, c0, segn, m != 0);
        continue;
      }
      const int64_t ylc64 = int64_t(y) - p.vocab_start - c0;
      const int ylc = (ylc64 >= 0 && ylc64 < segn) ? int(ylc64) : -1;
      // every thread combines the gathered partials (rank order) and evaluates the loss terms
      float dy;
      const Stat tot = combine_partials(p.partials_in + row, p.num_rows, p.nshards, dy);
      const RowStats rs = finalize(tot, dy);
      const int32_t rt = p.row_traj[row];
      RowSide sd{0.0, p.old_logp[row], p.ref_logp ? p.ref_logp[row] : 0.f, 0};
      const bool side_ok = row_side(p, row, rt, sd, ct == 0 && crank == 0);
      const LossOut lo = loss_terms(p, rs.logp, rs.H, sd, side_ok ? row_weight(p, invN, sd.nb, nact) : 0.f);
      if (ct == 0 && crank == 0) {
        if (side_ok) {
          acc_L += double(lo.w) * double(lo.L);
          acc_clip += lo.clipped ? 1.0 : 0.0;
          acc_kl += double(lo.kl);
          acc_H += double(rs.H);
          acc_n += 1.0;
        }
        if (p.logp) p.logp[row] = side_ok ? rs.logp : 0.f;
        if (p.entropy) p.entropy[row] = side_ok ? rs.H : 0.f;
      }
      const float mr = rs.m, lg2S = rs.lg2S, coef = lo.coef;
      char* drow = reinterpret_cast<char*>(p.dlogits) + (row * p.ld + c0) * int64_t(sizeof(T));
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&S.full[slot], phase);
        const uint8_t* buf = ring + size_t(slot) * kChunkBytes;
#pragma unroll
        for (int k = 0; k < kVPT; ++k) {
          const int vi = ct + k * kNCT;
          const int lc = c * CE + vi * EV;
          if (lc >= segn) continue;
          const uint4 w = *reinterpret_cast<const uint4*>(buf + vi * 16);
          float x[EV], g[EV];
          VT::unpack(w, x);
#pragma unroll
          for (int i = 0; i < EV; ++i) {
            const float d = __fsub_rn(__fmaf_rn(x[i], s2, -mr), lg2S);   // log2 p (reference first: see pass2_row)
            const float pv = ex2(d);
            // coef p + wcs p (ln p + H): the entropy-bonus term costs two FMAs, no extra exponential
            g[i] = lo.wcs == 0.f ? __fmul_rn(coef, pv) : pv * fmaf(lo.wcs, fmaf(kLn2, fmaxf(d, -1e30f), rs.H), coef);
          }
          if (unsigned(ylc - lc) < unsigned(EV)) {
#pragma unroll
            for (int i = 0; i < EV; ++i)
              if (lc + i == ylc) g[i] = lo.gy;
          }
          if (lc + EV <= segn) {
            stg_cs_v4(drow + size_t(lc) * sizeof(T), VT::pack(g));
          } else {
#pragma unroll
            for (int i = 0; i < EV; ++i)
              if (lc + i < segn) VT::store1(drow, lc + i, g[i]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[slot]);
        if (++slot == kSlots) {
          slot = 0;
          phase ^= 1u;
        }
      }
      ++q;
    }
    if (ct == 0) stats_epilogue(p, acc_L, acc_clip, acc_kl, acc_H, acc_n, nl, blockIdx.x, gridDim.x);
  }
  if (csize > 1) cluster_sync_all();
}

// ---- vocab-shard combine (otk_logprob_entropy_combine): same combine / finalize as the row kernels -----
__global__ void k_combine(int64_t num_rows, int nshards, const float4* __restrict__ partials,
                          const uint8_t* __restrict__ row_mask, float* logp, float* entropy, float* lse) {
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < num_rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    if (row_mask && !row_mask[row]) {
      logp[row] = 0.f;
      if (entropy) entropy[row] = 0.f;
      if (lse) lse[row] = 0.f;
      continue;
    }
    float dy;
    const Stat tot = combine_partials(partials + row, num_rows, nshards, dy);
    const RowStats rs = finalize(tot, dy);
    logp[row] = rs.logp;
    if (entropy) entropy[row] = rs.H;
    if (lse) lse[row] = rs.lse;
  }
}

// ---- launchers ---------------------------------------------------------------------------------------
// Clusters of csize CTAs must fit inside one GPC, so fewer than num_sms / csize of them can be resident at once
// (GPCs whose SM count is not a multiple of csize leave SMs over). A persistent grid larger than that runs in
// two waves — half the throughput (measured for 4-CTA rows) — so the grid is capped at the resident count
// (cudaOccupancyMaxActiveClusters; cached per (kernel, device, cluster size, smem, CTAs per SM)).
struct ClusterCap {
  const void* kern;
  int dev, csize, per_sm;
  size_t smem;
  int clusters;
};
static std::mutex g_cap_mu;
static ClusterCap g_cap[64];
static int g_ncap = 0;

template <typename KernelT>
static int max_resident_clusters(KernelT kern, int dev, int csize, size_t smem, int per_sm, cudaLaunchConfig_t cfg) {
  std::lock_guard<std::mutex> lk(g_cap_mu);
  for (int i = 0; i < g_ncap; ++i)
    if (g_cap[i].kern == (const void*)kern && g_cap[i].dev == dev && g_cap[i].csize == csize &&
        g_cap[i].smem == smem && g_cap[i].per_sm == per_sm)
      return g_cap[i].clusters;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;  // unknown: no cap
  }
  if (g_ncap < 64) g_cap[g_ncap++] = ClusterCap{(const void*)kern, dev, csize, per_sm, smem, n};
  return n;
}

template <typename KernelT>
static cudaError_t launch_row_kernel(KernelT kern, const otk_ctx* ctx, const RowParams& p, cudaStream_t s,
                                     int* grid_out, size_t smem_bytes = kSmemBytes, int ctas_per_sm = 1,
                                     int max_ctas = 0, int threads = kThreads) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes));
  if (e != cudaSuccess) return e;
  int64_t groups = int64_t(ctx->num_sms) * ctas_per_sm / p.csize;
  if (max_ctas > 0 && groups > max_ctas / p.csize) groups = max_ctas / p.csize;  // ranks sharing a GPU
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.csize > 1 ? 1 : 0;
  if (p.csize > 1) {
    cfg.gridDim = dim3(unsigned(groups * p.csize));
    const int cap = max_resident_clusters(kern, ctx->device, p.csize, smem_bytes, ctas_per_sm, cfg);
    if (cap > 0 && groups > cap) groups = cap;
  }
  if (groups > p.num_rows) groups = p.num_rows;
  if (groups < 1) groups = 1;
  const int grid = int(groups * p.csize);
  if (grid > kMaxCtas) return cudaErrorInvalidConfiguration;
  cfg.gridDim = dim3(grid);
  if (grid_out) *grid_out = grid;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_rows(const otk_ctx* ctx, RowMode mode, otk_dtype dtype, const RowParams& p, cudaStream_t s,
                        int* grid_out, int max_ctas) {
  constexpr size_t kFwdSmem = smem_bytes_for(kSlotsFwd);  // ~104 KB: two CTAs per SM
  if (dtype == OTK_BF16) {
    using B = __nv_bfloat16;
    switch (mode) {
      case kModeFwd: return launch_row_kernel(k_rows_tm<B, kModeFwd>, ctx, p, s, grid_out, kFwdSmem, 2);
      case kModePartial: return launch_row_kernel(k_rows_tm<B, kModePartial>, ctx, p, s, grid_out, kFwdSmem, 2);
      case kModeBwd: return launch_row_kernel(k_rows_tm<B, kModeBwd>, ctx, p, s, grid_out);
      case kModeBwdPartials: return launch_row_kernel(k_rows_stream<B>, ctx, p, s, grid_out);
      case kModeBwdVpf:
        if (p.pipe == 3)
          return launch_row_kernel(k_rows_tm<B, kModeBwdVpf, 3>, ctx, p, s, grid_out, kSmemBytes, 1, max_ctas,
                                   kThreads + 32);
        if (p.pipe)
          return launch_row_kernel(k_rows_tm<B, kModeBwdVpf, 1>, ctx, p, s, grid_out, kSmemBytes, 1, max_ctas,
                                   kThreads + 32);
        return launch_row_kernel(k_rows_tm<B, kModeBwdVpf>, ctx, p, s, grid_out, kSmemBytes, 1, max_ctas);
    }
  } else {
    switch (mode) {
      case kModeFwd: return launch_row_kernel(k_rows_tm<float, kModeFwd>, ctx, p, s, grid_out, kFwdSmem, 2);
      case kModePartial: return launch_row_kernel(k_rows_tm<float, kModePartial>, ctx, p, s, grid_out, kFwdSmem, 2);
      case kModeBwd: return launch_row_kernel(k_rows_tm<float, kModeBwd>, ctx, p, s, grid_out);
      case kModeBwdPartials: return launch_row_kernel(k_rows_stream<float>, ctx, p, s, grid_out);
      case kModeBwdVpf:
        if (p.pipe == 3)
          return launch_row_kernel(k_rows_tm<float, kModeBwdVpf, 3>, ctx, p, s, grid_out, kSmemBytes, 1, max_ctas,
                                   kThreads + 32);
        if (p.pipe)
          return launch_row_kernel(k_rows_tm<float, kModeBwdVpf, 1>, ctx, p, s, grid_out, kSmemBytes, 1, max_ctas,
                                   kThreads + 32);
        return launch_row_kernel(k_rows_tm<float, kModeBwdVpf>, ctx, p, s, grid_out, kSmemBytes, 1, max_ctas);
    }
  }
  return cudaErrorInvalidValue;
}

// K4-VPF ranks emulated in one launch: blocks_per_set = the SMs / nsets (one CTA per SM, a multiple of the cluster
// size), so the whole grid is one resident wave; csize 1 launches cooperatively (the driver refuses a grid that
// cannot be co-resident), csize > 1 checks the resident-cluster count.
cudaError_t launch_rows_vpf_group(const otk_ctx* ctx, otk_dtype dtype, const RowParams* ps, int nsets, int pipe,
                                  cudaStream_t s, int* grid_out) {
  RowParamsSet set;
  std::memset(&set, 0, sizeof(set));
  if (nsets < 1 || nsets > OTK_VPF_MAX_RANKS) return cudaErrorInvalidValue;
  for (int k = 0; k < nsets; ++k) set.p[k] = ps[k];
  const int csize = ps[0].csize;
  int64_t groups = int64_t(ctx->num_sms) / nsets / csize;
  if (groups > ps[0].num_rows) groups = ps[0].num_rows;
  if (groups < 1) groups = 1;
  set.nsets = nsets;
  set.blocks_per_set = int(groups * csize);
  const int grid = set.blocks_per_set * nsets;
  if (grid > ctx->num_sms) return cudaErrorCooperativeLaunchTooLarge;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(kThreads + (pipe ? 32 : 0));  // + the collector warp of the pipelined loop
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (csize > 1) {
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(grid);
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const int cap = max_resident_clusters(kern, ctx->device, csize, kSmemBytes, 1, cfg);
      if (cap > 0 && grid / csize > cap) return cudaErrorCooperativeLaunchTooLarge;
    } else {
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    cfg.gridDim = dim3(grid);
    if (grid_out) *grid_out = grid;
    return cudaLaunchKernelEx(&cfg, kern, set);
  };
  if (dtype == OTK_BF16) {
    using B = __nv_bfloat16;
    return pipe == 3 ? go(k_rows_vpf_group<B, 3>) : pipe ? go(k_rows_vpf_group<B, 1>) : go(k_rows_vpf_group<B, 0>);
  }
  return pipe == 3 ? go(k_rows_vpf_group<float, 3>) : pipe ? go(k_rows_vpf_group<float, 1>)
                                                       : go(k_rows_vpf_group<float, 0>);
}

// several partials of one row (e.g. the vocab chunks of the fused LM head on one rank) -> one partial of the
// same form, for a vocab-sharded caller to all-gather (same combine as above, rank order)
__global__ void k_combine_to_partial(int64_t num_rows, int nparts, const float4* __restrict__ partials,
                                     const uint8_t* __restrict__ row_mask, float4* out) {
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < num_rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    if (row_mask && !row_mask[row]) {
      out[row] = make_float4(-INFINITY, 0.f, 0.f, -INFINITY);
      continue;
    }
    float dy;
    const Stat tot = combine_partials(partials + row, num_rows, nparts, dy);
    out[row] = make_float4(tot.m, tot.s, tot.t, dy);
  }
}

cudaError_t launch_combine_to_partial(const otk_ctx* ctx, int64_t num_rows, int nparts, const float4* partials,
                                      const uint8_t* row_mask, float4* out, cudaStream_t s) {
  int64_t blocks = (num_rows + 255) / 256;
  if (blocks > int64_t(ctx->num_sms) * 8) blocks = int64_t(ctx->num_sms) * 8;
  if (blocks < 1) blocks = 1;
  k_combine_to_partial<<<int(blocks), 256, 0, s>>>(num_rows, nparts, partials, row_mask, out);
  return cudaGetLastError();
}

cudaError_t launch_combine(const otk_ctx* ctx, int64_t num_rows, int nshards, const float4* partials,
                           const uint8_t* row_mask, float* logp, float* entropy, float* lse, cudaStream_t s) {
  int64_t blocks = (num_rows + 255) / 256;
  if (blocks > int64_t(ctx->num_sms) * 8) blocks = int64_t(ctx->num_sms) * 8;
  if (blocks < 1) blocks = 1;
  k_combine<<<int(blocks), 256, 0, s>>>(num_rows, nshards, partials, row_mask, logp, entropy, lse);
  return cudaGetLastError();
}


// ---- NEXT-1 backward: per-row loss terms from the fused LM head's chunk partials ------------------------
// One thread per row: combine the row's vocab-chunk partials (chunk order, as k_combine), finalize, evaluate the
// loss terms of (4) (same loss_terms / row_side / row_weight as the row kernels), accumulate the stats, and write
// the constants the backward GEMMs form dx from (k_lmhead_bwd.cu):
//   dx_v = 2^d (alpha' + beta' d),  d = s log2(e) x_v - m,  alpha' = (coef + wcs H - wcs ln2 lg2S) 2^-lg2S,
//   beta' = wcs ln2 2^-lg2S  (so dx_v = coef p_v + wcs p_v (ln p_v + H), the (4) gradient incl. the entropy bonus),
// and gy = the target column's value (coef expm1(logp) + bonus). Inactive rows get m = 1e30 (2^d = 0), 0, 0, 0.
// The loss partials are reduced per CTA in a fixed order and by the last CTA (ticket): deterministic.
__global__ void __launch_bounds__(256) k_lmhead_loss_rows(const RowParams p, float4* __restrict__ rowc) {
  __shared__ double red[8][5];
  double acc[5] = {0, 0, 0, 0, 0};
  const int64_t nl = *p.n_loss;
  const float invN = nl > 0 ? float(1.0 / double(nl)) : 0.f;
  const int64_t nact = p.reduction != OTK_TOKEN_MEAN ? *p.n_active : 0;
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < p.num_rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int32_t y = p.targets[row];
    const uint8_t m = p.mask[row];
    float4 rc = make_float4(1e30f, 0.f, 0.f, 0.f);
    float lp_out = 0.f, H_out = 0.f;
    if (row_active(p, y, m)) {
      float dy;
      const Stat tot = combine_partials(p.partials_in + row, p.num_rows, p.nshards, dy);
      const RowStats rs = finalize(tot, dy);
      RowSide sd{0.0, p.old_logp[row], p.ref_logp ? p.ref_logp[row] : 0.f, 0};
      const bool side_ok = row_side(p, row, p.row_traj[row], sd, true);
      const LossOut lo = loss_terms(p, rs.logp, rs.H, sd, side_ok ? row_weight(p, invN, sd.nb, nact) : 0.f);
      if (side_ok) {
        acc[0] += double(lo.w) * double(lo.L);
        acc[1] += lo.clipped ? 1.0 : 0.0;
        acc[2] += double(lo.kl);
        acc[3] += double(rs.H);
        acc[4] += 1.0;
        lp_out = rs.logp;
        H_out = rs.H;
        const float sc = ex2(-rs.lg2S);
        const float alpha = fmaf(lo.wcs, rs.H, lo.coef), beta = lo.wcs * kLn2;
        rc = make_float4(rs.m, fmaf(-beta, rs.lg2S, alpha) * sc, beta * sc, lo.gy);
      }
    }
    rowc[row] = rc;
    if (p.logp) p.logp[row] = lp_out;
    if (p.entropy) p.entropy[row] = H_out;
  }
  // CTA reduction in a fixed order: warp shuffles, then warp 0 over the warps
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[w][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < int(blockDim.x >> 5); ++i)
      for (int k = 0; k < 5; ++k) t[k] += red[i][k];
    stats_epilogue(p, t[0], t[1], t[2], t[3], t[4], nl, blockIdx.x, gridDim.x);
  }
}

cudaError_t launch_lmhead_loss_rows(const otk_ctx* ctx, const RowParams& p, float4* rowc, cudaStream_t s) {
  int64_t blocks = (p.num_rows + 255) / 256;
  if (blocks > int64_t(ctx->num_sms) * 4) blocks = int64_t(ctx->num_sms) * 4;  // <= kMaxCtas stat slots
  if (blocks < 1) blocks = 1;
  k_lmhead_loss_rows<<<int(blocks), 256, 0, s>>>(p, rowc);
  return cudaGetLastError();
}

}  // namespace otk

#ifdef OTK_PHASE_TIMING
extern "C" void otk_debug_phase(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, otk::g_phase, sizeof(unsigned long long) * 8);
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(otk::g_phase, z, sizeof(z));
}
#endif
