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
        if (lane == lw) {
          float acc = __fadd_rn(Pseg, __fmul_rn(incl - ls, fseg));
          int t = -1, tnz = -1;
          float xt = 0.f, xnz = 0.f;
          for (int k = 0; k < 2 && t < 0; ++k) {
#pragma unroll
            for (int i = 0; i < EV; ++i) {
              const float e = e_elem<T>(q[k], i, k2, rk);
              const int col = (v0 + k) * EV + i;
              acc = __fadd_rn(acc, __fmul_rn(e, fseg));
              if (e > 0.f) {
                tnz = col;
                xnz = SV::elem(q[k], i);
              }
              if (t < 0 && acc > Tt) {
                t = col;
                xt = SV::elem(q[k], i);
              }
            }
          }
          if (t < 0) {
            t = tnz >= 0 ? tnz : 0;
            xt = tnz >= 0 ? xnz : SV::elem(q[0], 0);
          }
          p.tokens[row] = t;
          if (p.logp) p.logp[row] = (xt * k2 - R - log2f(Sw)) * 0.6931471805599453f;
        }
      }
      par ^= 1u;
      if (par == 0) hph ^= 1u;
    }
  }
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
