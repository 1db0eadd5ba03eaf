// k_sample_tm.cu — otk_sample_tokens, sampled draws on large decode batches (one CTA per row): the row streamed
// once through a bulk-TMA shared-memory ring, the inverse-transform search done by a dedicated warp off the
// streaming path. Same contract as k_sample.cu (R32; PAPER.md:170-171;
// SPEC.md:300-306): t = min{t : sum_{v <= t} p_v > u},  p = softmax(s x). (Greedy argmax stays on k_sample.cu,
// whose lane-strided pass measured faster for it.)
//
// Two CTAs per SM, 14 warps each:
//   warp 0 (one thread)  loader: 12 KB chunks of the row into an 8-slot ring (cp.async.bulk + mbarrier).
//   warps 1-12           consumers: thread ct reads the ADJACENT 16-byte vectors 2ct, 2ct+1 of a chunk, so a warp
//                        covers one contiguous 1 KB column segment per chunk. Per chunk and warp: a reference r
//                        (set by the first finite values, raised warp-uniformly only when a chunk sum overflows
//                        2^64 — no max in the common chunk), the segment's sum of
//                        e = 2^(x k2 - r) (one MUFU per element), reduced over the warp and stored with r.
//                        No per-row barrier: the segment sums go to the
//                        search warp through a 2-row mbarrier hand-off and the consumers stream on.
//   warp 13              search: R = max r, S = sum of the segment sums at R, T = u S; the crossing segment in
//                        column order (chunk-major, warp-minor); re-reads that 1 KB segment (L2), recomputes the
//                        same e values, a warp scan finds the crossing lane, which walks its 16 elements.
// fp32 rounding can put T an ulp outside the located range: the last column with non-zero mass is then taken
// (the draw is within rounding of a cdf boundary, where both neighbours are correct — DESIGN.md R32).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "otk_internal.h"
#include "otk_ptx.cuh"

namespace otk {
using namespace ptx;

namespace {
constexpr int kSWarps = 12;                      // consumer warps
constexpr int kSThreads = 32 * (kSWarps + 2);    // + loader warp 0 + search warp 13
constexpr int kSNct = 32 * kSWarps;
constexpr int kSSlots = 8;                       // 96 KB ring: two CTAs per SM
constexpr int kSChunk = 12288;                   // = kSNct * 32 bytes: two adjacent vectors per consumer thread
constexpr float kSNoRef = -1e30f;                // reference before the first finite logit
static_assert(kSChunk == kSNct * 32, "chunk = two 16-byte vectors per consumer thread");

struct SampSmem {
  uint64_t full[kSSlots], empty[kSSlots];
  uint64_t hfull[2], hempty[2];                  // consumer -> search hand-off, by row parity
  float2 part[2][kSampleTmMaxChunks][kSWarps];   // (sum of e at r, r) per (chunk, warp)
};
constexpr size_t kSSmemBytes = size_t(kSSlots) * kSChunk + sizeof(SampSmem);

template <typename T>
struct SV2;
template <>
struct SV2<__nv_bfloat16> {
  static constexpr int EV = 8;
  __device__ static float vmax(const uint4& q) {
    const uint32_t a = bmax2(bmax2(q.x, q.y), bmax2(q.z, q.w));
    return fmaxf(bf_lo(a), bf_hi(a));
  }
  __device__ static float elem(const uint4& q, int i) {
    const uint32_t w = i < 2 ? q.x : i < 4 ? q.y : i < 6 ? q.z : q.w;
    return (i & 1) ? bf_hi(w) : bf_lo(w);
  }
  __device__ static void mask_tail(uint4& q, int n_valid) {  // columns >= n_valid -> -inf
    uint32_t* w = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (2 * k >= n_valid) w[k] = 0xff80ff80u;
      else if (2 * k + 1 >= n_valid) w[k] = (w[k] & 0xffffu) | 0xff800000u;
    }
  }
  // sum of 2^(x k2 + rk) over the vector, pairwise in column order (the search re-uses it bit for bit)
  __device__ static float esum(const uint4& q, uint64_t k2x2, uint64_t rk2) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint64_t a = f2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float d0, d1;
      f2_split(ffma2(f2(bf_lo(w[k]), bf_hi(w[k])), k2x2, rk2), d0, d1);
      a = fadd2(a, f2(ex2(d0), ex2(d1)));
    }
    return f2_sum(a);
  }
};
template <>
struct SV2<float> {
  static constexpr int EV = 4;
  __device__ static float vmax(const uint4& q) {
    return fmaxf(fmaxf(__uint_as_float(q.x), __uint_as_float(q.y)), fmaxf(__uint_as_float(q.z), __uint_as_float(q.w)));
  }
  __device__ static float elem(const uint4& q, int i) {
    return __uint_as_float(i == 0 ? q.x : i == 1 ? q.y : i == 2 ? q.z : q.w);
  }
  __device__ static void mask_tail(uint4& q, int n_valid) {
    uint32_t* w = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k >= n_valid) w[k] = 0xff800000u;
  }
  __device__ static float esum(const uint4& q, uint64_t k2x2, uint64_t rk2) {
    float d0, d1, d2, d3;
    f2_split(ffma2(f2(__uint_as_float(q.x), __uint_as_float(q.y)), k2x2, rk2), d0, d1);
    f2_split(ffma2(f2(__uint_as_float(q.z), __uint_as_float(q.w)), k2x2, rk2), d2, d3);
    uint64_t a = f2(ex2(d0), ex2(d1));
    a = fadd2(a, f2(ex2(d2), ex2(d3)));
    return f2_sum(a);
  }
};

// element i of a vector: its e at reference rk (same formula as esum, element by element)
template <typename T>
__device__ __forceinline__ float e_elem(const uint4& q, int i, float k2, float rk) {
  return ex2(fmaf(SV2<T>::elem(q, i), k2, rk));
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(kSThreads, 2) k_sample_tm(const SampleParams p) {
  using SV = SV2<T>;
  constexpr int EV = SV::EV;
  constexpr int CE = kSChunk / int(sizeof(T));   // columns per chunk
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  SampSmem& S = *reinterpret_cast<SampSmem*>(smem + size_t(kSSlots) * kSChunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row_bytes_v = p.vocab * int64_t(sizeof(T));
  const uint32_t rb16 = uint32_t((row_bytes_v + 15) & ~int64_t(15));
  const int nch = int((rb16 + kSChunk - 1) / kSChunk);
  const int nvec = int((p.vocab + EV - 1) / EV);
  const int tail_valid = int(p.vocab - int64_t(nvec - 1) * EV);
  const float k2 = p.scale * 1.4426950408889634f;
  const uint64_t k2x2 = f2(k2, k2);
  const uint4 ninf = sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                                    : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSSlots; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kSWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.hfull[i], kSWarps);
      mbar_init(&S.hempty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- loader: every row, chunk by chunk
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t slot = 0, phase = 0;
      for (int64_t row = blockIdx.x; row < p.num_rows; row += gridDim.x) {
        const char* src = reinterpret_cast<const char*>(p.logits) + row * p.ld * int64_t(sizeof(T));
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&S.empty[slot], phase ^ 1u);
          const uint32_t off = uint32_t(c) * kSChunk;
          const uint32_t bytes = min(uint32_t(kSChunk), rb16 - off);
          mbar_arrive_expect_tx(&S.full[slot], bytes);
          bulk_g2s(ring + size_t(slot) * kSChunk, src + off, bytes, &S.full[slot], pol);
          if (++slot == kSSlots) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp <= kSWarps) {
    // ---------------- consumers
    const int ct = threadIdx.x - 32, cw = warp - 1;
    uint32_t slot = 0, phase = 0, par = 0, hph = 0;
    for (int64_t row = blockIdx.x; row < p.num_rows; row += gridDim.x) {
      mbar_wait(&S.hempty[par], hph ^ 1u);   // the search warp has read this parity's previous row
      float r = kSNoRef;                      // warp-uniform reference (k2 units)
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&S.full[slot], phase);
        const uint8_t* buf = ring + size_t(slot) * kSChunk + ct * 32;
        uint4 q0 = *reinterpret_cast<const uint4*>(buf);
        uint4 q1 = *reinterpret_cast<const uint4*>(buf + 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[slot]);
        if (++slot == kSSlots) {
          slot = 0;
          phase ^= 1u;
        }
        const int v0 = c * (CE / EV) + 2 * ct;   // vector index of q0 in the row
        // vectors past the row (stale ring bytes) -> -inf; the row's partial last vector -> -inf past vocab
        if (v0 >= nvec) q0 = ninf;
        else if (v0 == nvec - 1 && tail_valid < EV) SV::mask_tail(q0, tail_valid);
        if (v0 + 1 >= nvec) q1 = ninf;
        else if (v0 + 1 == nvec - 1 && tail_valid < EV) SV::mask_tail(q1, tail_valid);
        // the warp's reference r: set from the warp maximum when there is none yet, and raised to the chunk's
        // warp maximum only when a thread's chunk sum leaves [0, 2^64] (overflow; NaN from +inf) — detected from
        // the sums, so the common chunk needs no max at all. Each chunk's sum is stored with its own r.
        float cs = 0.f;
        bool redo = !(r > kSNoRef);
        if (!redo) {
          const float rk = -r;
          const uint64_t rk2 = f2(rk, rk);
          cs = __fadd_rn(SV::esum(q0, k2x2, rk2), SV::esum(q1, k2x2, rk2));
          redo = __any_sync(0xffffffffu, !(cs <= 0x1p64f));
        } else {
          redo = true;
        }
        if (redo) {  // warp-uniform: the first chunk with a finite value, or an overflow
          float wm = fmaxf(SV::vmax(q0), SV::vmax(q1));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
          if (wm * k2 > r) r = wm * k2;
          cs = 0.f;
          if (r > kSNoRef) {
            const float rk = -r;
            const uint64_t rk2 = f2(rk, rk);
            cs = __fadd_rn(SV::esum(q0, k2x2, rk2), SV::esum(q1, k2x2, rk2));
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cs = __fadd_rn(cs, __shfl_xor_sync(0xffffffffu, cs, o));
        if (lane == 0) S.part[par][c][cw] = make_float2(cs, r);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.hfull[par]);
      par ^= 1u;
      if (par == 0) hph ^= 1u;
    }
  } else {
    // ---------------- search warp
    uint32_t par = 0, hph = 0;
    for (int64_t row = blockIdx.x; row < p.num_rows; row += gridDim.x) {
      mbar_wait(&S.hfull[par], hph);
      // row reference R and total S (fixed order: chunk-major, warp-minor, lane-strided then butterfly)
      const int nseg = nch * kSWarps;
      float R = kSNoRef;
      for (int i = lane; i < nseg; i += 32) R = fmaxf(R, S.part[par][i / kSWarps][i % kSWarps].y);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) R = fmaxf(R, __shfl_xor_sync(0xffffffffu, R, o));
      float Sl = 0.f;
      for (int i = lane; i < nseg; i += 32) {
        const float2 v = S.part[par][i / kSWarps][i % kSWarps];
        if (v.x > 0.f) Sl = __fadd_rn(Sl, __fmul_rn(v.x, ex2(v.y - R)));
      }
      float Sw = Sl;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Sw = __fadd_rn(Sw, __shfl_xor_sync(0xffffffffu, Sw, o));
      const bool degenerate = !(R > kSNoRef) || !(Sw > 0.f);
      const T* rbase = reinterpret_cast<const T*>(p.logits) + row * p.ld;
      if (degenerate) {  // no finite logit: token 0, logp -inf (as k_sample.cu)
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&S.hempty[par]);
          p.tokens[row] = 0;
          if (p.logp) p.logp[row] = -INFINITY;
        }
      } else {
        float u = p.u[row];
        if (!(u >= 0.f && u < 1.f)) {
          if (lane == 0) set_error(p.err, OTK_ERR_INVALID_ARG);
          u = fminf(fmaxf(u, 0.f), 0.99999994f);
        }
        float Tt = u * Sw;
        if (!(Tt < Sw)) Tt = Sw * 0.99999976f;
        // crossing segment, in column order; 32 segments per step: lane prefix sums, ballot of the first crossing
        int seg = -1, seglast = -1;
        float P = 0.f, Pseg = 0.f, Plast = 0.f, fseg = 0.f, flast = 0.f;
        for (int base = 0; base < nseg && seg < 0; base += 32) {
          const int i = base + lane;
          float c = 0.f, f = 0.f;
          if (i < nseg) {
            const float2 v = S.part[par][i / kSWarps][i % kSWarps];
            f = ex2(v.y - R);
            c = v.x > 0.f ? __fmul_rn(v.x, f) : 0.f;
          }
          float incl = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = __fadd_rn(incl, y);
          }
          const unsigned cross = __ballot_sync(0xffffffffu, i < nseg && __fadd_rn(P, incl) > Tt);
          const unsigned nz = __ballot_sync(0xffffffffu, c > 0.f);
          if (nz) {  // last segment with mass so far (fallback)
            const int l = 31 - __clz(nz);
            seglast = base + l;
            Plast = __fadd_rn(P, __shfl_sync(0xffffffffu, incl - c, l));
            flast = __shfl_sync(0xffffffffu, f, l);
          }
          if (cross) {
            const int l = __ffs(cross) - 1;
            seg = base + l;
            Pseg = __fadd_rn(P, __shfl_sync(0xffffffffu, incl - c, l));
            fseg = __shfl_sync(0xffffffffu, f, l);
          }
          P = __fadd_rn(P, __shfl_sync(0xffffffffu, incl, 31));
        }
        if (seg < 0) {
          seg = seglast;
          Pseg = Plast;
          fseg = flast;
        }
        const int cstar = seg / kSWarps, wstar = seg % kSWarps;
        const float rseg = S.part[par][cstar][wstar].y;
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.hempty[par]);   // the hand-off buffer is no longer read
        // re-read the 1 KB segment (L2): lane l holds its vectors 2l, 2l+1 of thread-range (wstar, lane l)
        const int v0 = cstar * (CE / EV) + 2 * (32 * wstar + lane);
        const uint4* rp = reinterpret_cast<const uint4*>(rbase);
        uint4 q[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int v = v0 + k;
          q[k] = v < nvec ? __ldg(rp + v) : ninf;
          if (v == nvec - 1 && tail_valid < EV) SV::mask_tail(q[k], tail_valid);
        }
        const float rk = -rseg;
        const uint64_t rk2 = f2(rk, rk);
        const float ls = __fadd_rn(SV::esum(q[0], k2x2, rk2), SV::esum(q[1], k2x2, rk2));
        float incl = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl = __fadd_rn(incl, y);
        }
        const unsigned cross = __ballot_sync(0xffffffffu, __fadd_rn(Pseg, __fmul_rn(incl, fseg)) > Tt);
        const unsigned nz = __ballot_sync(0xffffffffu, ls > 0.f);
        const int lw = cross ? __ffs(cross) - 1 : (nz ? 31 - __clz(nz) : 0);
        // lane lw's 2 EV elements, one per lane (column order), scanned across the warp
        const float base = __shfl_sync(0xffffffffu, __fadd_rn(Pseg, __fmul_rn(incl - ls, fseg)), lw);
        uint4 qq[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          qq[k].x = __shfl_sync(0xffffffffu, q[k].x, lw);
          qq[k].y = __shfl_sync(0xffffffffu, q[k].y, lw);
          qq[k].z = __shfl_sync(0xffffffffu, q[k].z, lw);
          qq[k].w = __shfl_sync(0xffffffffu, q[k].w, lw);
        }
        const int vl = __shfl_sync(0xffffffffu, v0, lw);
        const int ke = lane / EV, ie = lane % EV;   // this lane's element (lanes >= 2 EV: none)
        float x = -INFINITY, e = 0.f;
        if (lane < 2 * EV) {
          const uint4 qk = ke == 0 ? qq[0] : qq[1];
          x = SV::elem(qk, ie);
          e = __fmul_rn(e_elem<T>(qk, ie, k2, rk), fseg);
        }
        float acc = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, acc, o);
          if (lane >= o) acc = __fadd_rn(acc, y);
        }
        const unsigned hit = __ballot_sync(0xffffffffu, lane < 2 * EV && __fadd_rn(base, acc) > Tt);
        const unsigned enz = __ballot_sync(0xffffffffu, e > 0.f);
        const int li = hit ? __ffs(hit) - 1 : (enz ? 31 - __clz(enz) : 0);  // fallback: the last column with mass
        const float xt = __shfl_sync(0xffffffffu, x, li);
        if (lane == 0) {
          p.tokens[row] = vl * EV + li;
          if (p.logp) p.logp[row] = (xt * k2 - R - log2f(Sw)) * 0.6931471805599453f;
        }
      }
      par ^= 1u;
      if (par == 0) hph ^= 1u;
    }
  }
}

// =====================================================================================================
// k_sample_dec — decode-sized batches (a few to ~70 rows): ONE row per thread-block cluster of C CTAs, each CTA
// holding its whole column range in shared memory (bulk TMA, 4 barriers: compute starts on the first quarter),
// so the row is read from HBM once, in one round of latency, and the search never re-reads it from L2. Per CTA:
// 16 warps over 1 KB segments (lane l: vectors 2l, 2l+1), a warp-uniform reference per warp (k_sample_tm's
// scheme), one (sum of e, reference) per segment and a running per-warp total; per CTA (R_c, S_c) and the greedy
// (max, first index); ONE cluster barrier, then a split arrive / wait so that only the crossing CTA's search is left
// on the critical path; every CTA combines the C partials in rank order (lane r reads CTA r over DSMEM); the
// crossing CTA's warp 0 finds the crossing segment (ballot scan), then from shared memory the crossing lane and,
// one element per lane, the crossing column. Same contract and rounding fallback as the other samplers.
// =====================================================================================================
constexpr int kDecWarps = 16;
constexpr int kDecThreads = 32 * kDecWarps;
constexpr int kDecSeg = 1024;                        // bytes per segment (64 vectors: 2 per lane)
constexpr int kDecMaxSegs = 200;                     // 200 KB of row per CTA
#ifndef OTK_SDEC_PARTS
#define OTK_SDEC_PARTS 4
#endif
constexpr int kDecParts = OTK_SDEC_PARTS;            // bulk copies (and barriers) the range is loaded in
constexpr size_t kDecSmemBase = 2048 + 512;          // part[] (float2 x kDecMaxSegs) + barriers, ahead of the data

struct DecSmem {
  float2 part[kDecMaxSegs];                          // (sum of e at r, r) per segment
  uint64_t full[16];
  float4 cta;                                        // (R_c, S_c, greedy max, greedy first index) — read over DSMEM
  float wb[kDecWarps];
  int wi[kDecWarps];
  float2 wr[kDecWarps];                              // per warp (reference, sum of its segments at it)
};
static_assert(sizeof(DecSmem) <= kDecSmemBase, "decode sampler header");

#ifdef OTK_SDEC_TIMING  // experiments only: globaltimer stamps of CTA 0 (ns)
__device__ unsigned long long g_sdec_t[8];
#define SDEC_T(i) if (blockIdx.x == 0 && threadIdx.x == 0) g_sdec_t[i] = globaltimer_ns()
#else
#define SDEC_T(i)
#endif
template <typename T, bool kCl>
__global__ void __launch_bounds__(kDecThreads, 1) k_sample_dec(const SampleParams p, int nseg_c) {
  using SV = SV2<T>;
  constexpr int EV = SV::EV;
  constexpr int VPS = kDecSeg / 16;                  // vectors per segment (64)
  extern __shared__ __align__(1024) uint8_t smem[];
  DecSmem& S = *reinterpret_cast<DecSmem*>(smem);
  uint8_t* data = smem + kDecSmemBase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = kCl ? p.csize : 1;
  const int rank = kCl ? int(cluster_ctarank()) : 0;
  const int64_t row = kCl ? int64_t(cluster_id_x()) : int64_t(blockIdx.x);
  const int nvec = int((p.vocab + EV - 1) / EV);
  const int tail_valid = int(p.vocab - int64_t(nvec - 1) * EV);
  const int v_begin = rank * nseg_c * VPS;           // first vector of this CTA's range
  const int nv_c = max(0, min(nseg_c * VPS, nvec - v_begin));
  const int nseg = (nv_c + VPS - 1) / VPS;           // segments with data
  const float k2 = p.scale * 1.4426950408889634f;
  const uint64_t k2x2 = f2(k2, k2);
  const bool greedy = p.greedy != 0;
  const bool need_sum = !(greedy && p.logp == nullptr);
  const uint4 ninf = sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                                    : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
  const T* rbase = reinterpret_cast<const T*>(p.logits) + row * p.ld;
  // quarters of the range: part q covers segments [q0(q), q0(q+1))
  auto q0 = [&](int q) { return (nseg * q + kDecParts - 1) / kDecParts; };
  SDEC_T(0);

  if (threadIdx.x == 0) {
    for (int q = 0; q < kDecParts; ++q) mbar_init(&S.full[q], 1);
    fence_mbar_init();
    const uint64_t pol = policy_evict_first();
    const char* src = reinterpret_cast<const char*>(rbase) + int64_t(v_begin) * 16;
    for (int q = 0; q < kDecParts; ++q) {
      const int s0 = q0(q), s1 = q0(q + 1);
      const uint32_t b0 = uint32_t(s0) * kDecSeg, b1 = uint32_t(min(s1 * VPS, nv_c)) * 16u;
      if (b1 > b0) {
        mbar_arrive_expect_tx(&S.full[q], b1 - b0);
        bulk_g2s(data + b0, src + b0, b1 - b0, &S.full[q], pol);
      } else {
        mbar_arrive(&S.full[q]);
      }
    }
  }
  __syncthreads();

  // ---------------- segments: warp w takes segments w, w + 8, ... (in order: waits the quarters in order)
  float r = kSNoRef;                                 // warp-uniform reference (k2 units)
  float racc = kSNoRef, sacc = 0.f;                  // this warp's running total of its segments, at racc
  float best = -INFINITY;
  int bidx = INT_MAX;
  int qw = 0;
  for (int sg = warp; sg < nseg; sg += kDecWarps) {
    while (qw < kDecParts && q0(qw + 1) <= sg) ++qw;
    mbar_wait(&S.full[qw], 0);
    const int v0 = v_begin + sg * VPS + 2 * lane;    // row vector index of q[0]
    uint4 q[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int v = v0 + k;
      q[k] = v < nvec ? *reinterpret_cast<const uint4*>(data + size_t(v - v_begin) * 16) : ninf;
      if (v == nvec - 1 && tail_valid < EV) SV::mask_tail(q[k], tail_valid);
    }
    if (greedy) {  // the lane's first maximum (column order: vector 0 before vector 1, element order inside)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < EV; ++i) {
          const float x = SV::elem(q[k], i);
          if (x > best) {
            best = x;
            bidx = (v0 + k) * EV + i;
          }
        }
    }
    if (need_sum) {
      float cs = 0.f;
      bool redo = !(r > kSNoRef);
      if (!redo) {
        const float rk = -r;
        const uint64_t rk2 = f2(rk, rk);
        cs = __fadd_rn(SV::esum(q[0], k2x2, rk2), SV::esum(q[1], k2x2, rk2));
        redo = __any_sync(0xffffffffu, !(cs <= 0x1p64f));
      }
      if (redo) {
        float wm = fmaxf(SV::vmax(q[0]), SV::vmax(q[1]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        if (wm * k2 > r) r = wm * k2;
        cs = 0.f;
        if (r > kSNoRef) {
          const float rk = -r;
          const uint64_t rk2 = f2(rk, rk);
          cs = __fadd_rn(SV::esum(q[0], k2x2, rk2), SV::esum(q[1], k2x2, rk2));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cs = __fadd_rn(cs, __shfl_xor_sync(0xffffffffu, cs, o));
      if (lane == 0) S.part[sg] = make_float2(cs, r);
      if (r > racc) {  // the reference was raised: move the running total to it
        sacc = racc > kSNoRef ? __fmul_rn(sacc, ex2(racc - r)) : 0.f;
        racc = r;
      }
      sacc = __fadd_rn(sacc, cs);
    }
  }
  if (lane == 0) S.wr[warp] = make_float2(racc, sacc);
  SDEC_T(1);
  if (greedy) {  // warp: max, then the first column holding it
    float bw = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bw = fmaxf(bw, __shfl_xor_sync(0xffffffffu, bw, o));
    int iw = best == bw ? bidx : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) iw = min(iw, __shfl_xor_sync(0xffffffffu, iw, o));
    if (lane == 0) {
      S.wb[warp] = bw;
      S.wi[warp] = iw;
    }
  }
  __syncthreads();
  // ---------------- CTA partial (warp 0; fixed order: lane-strided over segments, then butterfly)
  if (warp == 0) {  // CTA partial from the warp totals (lane w: warp w; butterfly order)
    float R = kSNoRef, Sl = 0.f;
    if (need_sum) {
      const float2 wv = lane < kDecWarps ? S.wr[lane] : make_float2(kSNoRef, 0.f);
      R = wv.x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) R = fmaxf(R, __shfl_xor_sync(0xffffffffu, R, o));
      Sl = wv.y > 0.f ? __fmul_rn(wv.y, ex2(wv.x - R)) : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Sl = __fadd_rn(Sl, __shfl_xor_sync(0xffffffffu, Sl, o));
    }
    if (lane == 0) {
      float B = -INFINITY;
      int I = INT_MAX;
      if (greedy)
        for (int w = 0; w < kDecWarps; ++w) {
          if (S.wb[w] > B) {
            B = S.wb[w];
            I = S.wi[w];
          } else if (S.wb[w] == B) {
            I = min(I, S.wi[w]);
          }
        }
      S.cta = make_float4(R, Sl, B, __int_as_float(I));
    }
  }
  SDEC_T(2);
  if (kCl) cluster_sync_all(); else __syncthreads();
  SDEC_T(3);
  // every CTA's partial is final: the exit barrier's arrive now (warp 0 after its DSMEM reads, below), its wait at
  // the end — a CTA never exits while a peer may still read its partial, and only the search stays on the path
  if (kCl && warp != 0) asm volatile("barrier.cluster.arrive.release;" ::: "memory");
  // ---------------- row combine (rank order, identical in every CTA) and the crossing CTA
  if (warp == 0) {
    // lane rr reads CTA rr's partial (the C DSMEM round trips overlap); the rank-order loops below take them by
    // shuffles
    float4 mine4 = S.cta;
    if (kCl && lane < C && lane != rank) {
      const uint32_t ra = mapa(smem_u32(&S.cta), uint32_t(lane));
      asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(mine4.x), "=f"(mine4.y), "=f"(mine4.z), "=f"(mine4.w)
                   : "r"(ra)
                   : "memory");
    }
    if (kCl) asm volatile("barrier.cluster.arrive.release;" ::: "memory");
    auto part_of = [&](int rr) -> float4 {
      return make_float4(__shfl_sync(0xffffffffu, mine4.x, rr), __shfl_sync(0xffffffffu, mine4.y, rr),
                         __shfl_sync(0xffffffffu, mine4.z, rr), __shfl_sync(0xffffffffu, mine4.w, rr));
    };
    float R = kSNoRef, B = -INFINITY;
    int I = INT_MAX;
    for (int rr = 0; rr < C; ++rr) {
      const float4 v = part_of(rr);
      R = fmaxf(R, v.x);
      if (greedy) {
        const int ir = __float_as_int(v.w);
        if (v.z > B) {
          B = v.z;
          I = ir;
        } else if (v.z == B) {
          I = min(I, ir);
        }
      }
    }
    float Sw = 0.f;
    for (int rr = 0; rr < C; ++rr) {
      const float4 v = part_of(rr);
      if (v.y > 0.f) Sw = __fadd_rn(Sw, __fmul_rn(v.y, ex2(v.x - R)));
    }
    // as the other samplers (R32): logits <= -1e30 carry no mass, a row without any larger one is degenerate
    const bool degenerate = greedy ? !(B > -1e30f) || (need_sum && !(Sw > 0.f))
                                   : (!(R > kSNoRef) || !(Sw > 0.f));
    if (greedy || degenerate) {
      if (rank == 0 && lane == 0) {
        p.tokens[row] = degenerate ? 0 : I;
        if (p.logp) p.logp[row] = degenerate ? -INFINITY : (B * k2 - R - log2f(Sw)) * 0.6931471805599453f;
      }
    } else {
      float u = p.u[row];
      if (!(u >= 0.f && u < 1.f)) {
        if (lane == 0 && rank == 0) set_error(p.err, OTK_ERR_INVALID_ARG);
        u = fminf(fmaxf(u, 0.f), 0.99999994f);
      }
      float Tt = u * Sw;
      if (!(Tt < Sw)) Tt = Sw * 0.99999976f;
      // crossing CTA (rank order), fallback: the last CTA with mass
      int rs = -1, rlast = 0;
      float P = 0.f, Pc = 0.f, Plast = 0.f;
      for (int rr = 0; rr < C; ++rr) {
        const float4 v = part_of(rr);
        const float c = v.y > 0.f ? __fmul_rn(v.y, ex2(v.x - R)) : 0.f;
        if (c > 0.f) {
          rlast = rr;
          Plast = P;
        }
        const float Pn = __fadd_rn(P, c);
        if (Pn > Tt) {
          rs = rr;
          Pc = P;
          break;
        }
        P = Pn;
      }
      if (rs < 0) {
        rs = rlast;
        Pc = Plast;
      }
      if (rank == rs) {
        // crossing segment (column order), 32 per step: lane prefix sums, ballot of the first crossing
        int seg = -1, seglast = -1;
        float Pseg = 0.f, Pl = 0.f, fseg = 0.f, flast = 0.f;
        P = Pc;
        for (int base = 0; base < nseg && seg < 0; base += 32) {
          const int i = base + lane;
          float c = 0.f, f = 0.f;
          if (i < nseg) {
            const float2 v = S.part[i];
            f = ex2(v.y - R);
            c = v.x > 0.f ? __fmul_rn(v.x, f) : 0.f;
          }
          float incl = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = __fadd_rn(incl, y);
          }
          const unsigned cross = __ballot_sync(0xffffffffu, i < nseg && __fadd_rn(P, incl) > Tt);
          const unsigned nz = __ballot_sync(0xffffffffu, c > 0.f);
          if (nz) {
            const int l = 31 - __clz(nz);
            seglast = base + l;
            Pl = __fadd_rn(P, __shfl_sync(0xffffffffu, incl - c, l));
            flast = __shfl_sync(0xffffffffu, f, l);
          }
          if (cross) {
            const int l = __ffs(cross) - 1;
            seg = base + l;
            Pseg = __fadd_rn(P, __shfl_sync(0xffffffffu, incl - c, l));
            fseg = __shfl_sync(0xffffffffu, f, l);
          }
          P = __fadd_rn(P, __shfl_sync(0xffffffffu, incl, 31));
        }
        if (seg < 0) {
          seg = max(seglast, 0);
          Pseg = Pl;
          fseg = flast;
        }
        // the segment from SHARED memory: lane l's vectors 2l, 2l+1 (the e values of the segment pass, bit for bit)
        const float rseg = S.part[seg].y;
        const int v0 = v_begin + seg * VPS + 2 * lane;
        uint4 q[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int v = v0 + k;
          q[k] = v < nvec ? *reinterpret_cast<const uint4*>(data + size_t(v - v_begin) * 16) : ninf;
          if (v == nvec - 1 && tail_valid < EV) SV::mask_tail(q[k], tail_valid);
        }
        const float rk = -rseg;
        const uint64_t rk2 = f2(rk, rk);
        const float ls = __fadd_rn(SV::esum(q[0], k2x2, rk2), SV::esum(q[1], k2x2, rk2));
        float incl = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl = __fadd_rn(incl, y);
        }
        const unsigned cross = __ballot_sync(0xffffffffu, __fadd_rn(Pseg, __fmul_rn(incl, fseg)) > Tt);
        const unsigned nz = __ballot_sync(0xffffffffu, ls > 0.f);
        const int lw = cross ? __ffs(cross) - 1 : (nz ? 31 - __clz(nz) : 0);
        // lane lw's 2 EV elements, one per lane (column order), scanned across the warp
        const float base = __shfl_sync(0xffffffffu, __fadd_rn(Pseg, __fmul_rn(incl - ls, fseg)), lw);
        uint4 qq[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          qq[k].x = __shfl_sync(0xffffffffu, q[k].x, lw);
          qq[k].y = __shfl_sync(0xffffffffu, q[k].y, lw);
          qq[k].z = __shfl_sync(0xffffffffu, q[k].z, lw);
          qq[k].w = __shfl_sync(0xffffffffu, q[k].w, lw);
        }
        const int vl = __shfl_sync(0xffffffffu, v0, lw);
        const int ke = lane / EV, ie = lane % EV;   // this lane's element (lanes >= 2 EV: none)
        float x = -INFINITY, e = 0.f;
        if (lane < 2 * EV) {
          const uint4 qk = ke == 0 ? qq[0] : qq[1];
          x = SV::elem(qk, ie);
          e = __fmul_rn(e_elem<T>(qk, ie, k2, rk), fseg);
        }
        float acc = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, acc, o);
          if (lane >= o) acc = __fadd_rn(acc, y);
        }
        const unsigned hit = __ballot_sync(0xffffffffu, lane < 2 * EV && __fadd_rn(base, acc) > Tt);
        const unsigned enz = __ballot_sync(0xffffffffu, e > 0.f);
        const int li = hit ? __ffs(hit) - 1 : (enz ? 31 - __clz(enz) : 0);  // fallback: the last column with mass
        const float xt = __shfl_sync(0xffffffffu, x, li);
        if (lane == 0) {
          p.tokens[row] = vl * EV + li;
          if (p.logp) p.logp[row] = (xt * k2 - R - log2f(Sw)) * 0.6931471805599453f;
        }
      }
    }
  }
  SDEC_T(4);
  if (kCl) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");  // no CTA exits while a peer reads its partial
  SDEC_T(5);
}
#ifdef OTK_SDEC_TIMING
extern "C" void otk_debug_sdec(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_sdec_t, sizeof(g_sdec_t)); }
#endif

// the decode kernel's shape for this batch, or false: C >= 4 CTAs per row with C * rows <= SMs and a range of at
// most kDecMaxSegs segments per CTA
bool sample_dec_shape(int64_t num_rows, int64_t vocab, int dtype, int num_sms, int* csize, int* nseg_c) {
  const int64_t nvec = (vocab * (dtype == OTK_BF16 ? 2 : 4) + 15) / 16;
  const int64_t nsegs = (nvec + 63) / 64;
  if (num_rows < 1 || num_rows > num_sms) return false;
  // at least 4 CTAs per row (<= 37 rows on 148 SMs): measured faster than the lane-strided kernel there (16 rows
  // 7.8 vs 8.4 us), slower with 2 (64 rows 13.0 vs 12.3 us: a 152 KB range per CTA is one SM's bandwidth share)
#ifndef OTK_SDEC_MINC
#define OTK_SDEC_MINC 4
#endif
  const int64_t c = std::min<int64_t>(8, num_sms / num_rows);
  if (c < OTK_SDEC_MINC) return false;
  const int64_t per = (nsegs + c - 1) / c;
  if (per > kDecMaxSegs) return false;
  *csize = int(c);
  *nseg_c = int(per);
  return true;
}

cudaError_t launch_sample_dec(otk_ctx* ctx, SampleParams p, int dtype, int csize, int nseg_c, cudaStream_t s) {
  p.csize = csize;
  const size_t smem = kDecSmemBase + size_t(nseg_c) * kDecSeg;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(p.num_rows * csize), 1, 1);
  cfg.blockDim = dim3(kDecThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(csize);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = csize > 1 ? 1 : 0;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, kern, p, nseg_c);
    return e != cudaSuccess ? e : cudaGetLastError();
  };
  if (dtype == OTK_BF16)
    return csize > 1 ? go(k_sample_dec<__nv_bfloat16, true>) : go(k_sample_dec<__nv_bfloat16, false>);
  return csize > 1 ? go(k_sample_dec<float, true>) : go(k_sample_dec<float, false>);
}

bool sample_tm_fits(int64_t vocab, int dtype) {
  const int64_t rb = (vocab * (dtype == OTK_BF16 ? 2 : 4) + 15) / 16 * 16;
  return (rb + kSChunk - 1) / kSChunk <= kSampleTmMaxChunks;
}

cudaError_t launch_sample_tm(otk_ctx* ctx, const SampleParams& p, int dtype, cudaStream_t s) {
  const int grid = int(std::min<int64_t>(p.num_rows, int64_t(ctx->num_sms) * 2));
  if (dtype == OTK_BF16) {
    cudaError_t e = cudaFuncSetAttribute(k_sample_tm<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSSmemBytes));
    if (e != cudaSuccess) return e;
    k_sample_tm<__nv_bfloat16><<<grid, kSThreads, kSSmemBytes, s>>>(p);
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_sample_tm<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSSmemBytes));
    if (e != cudaSuccess) return e;
    k_sample_tm<float><<<grid, kSThreads, kSSmemBytes, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace otk
