// k_sample_tm.cu — otk_sample_tokens, sampled draws on batches above the decode kernel's range (one CTA per row, or
// for up to two rows per SM a cluster of 2-8 CTAs per row): the row streamed once through a bulk-TMA shared-memory
// ring, the inverse-transform search done by a dedicated warp off the streaming path. Also k_sample_dec (decode
// batches, below). Same contract as k_sample.cu (R32; PAPER.md:170-171;
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
  float4 peer[8];                                // cluster split: the CTAs' (R_c, S_c) pushed by rank
  uint64_t xbar;
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

__device__ __forceinline__ float redux_max_f32(float v) {   // warp max (sm_100a: one CREDUX)
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ int redux_min_s32(int v) {
  int r;
  asm volatile("redux.sync.min.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
// element i of a vector: its e at reference rk (same formula as esum, element by element)
template <typename T>
__device__ __forceinline__ float e_elem(const uint4& q, int i, float k2, float rk) {
  return ex2(fmaf(SV2<T>::elem(q, i), k2, rk));
}
}  // namespace

#ifdef OTK_STM_TIMING  // experiments only: [cta][0] globaltimer at the start (ns), [cta][1..] clock64 stamps of the
// first row: 1 start, 2 consumer warp 1 has chunk 0, 3 it has finished the row, 4 search warp has the row, 5 done
__device__ unsigned long long g_stm_t[256 * 8];
#define STM_T(i, who)                                                                 \
  if ((who) && blockIdx.x < 256 && row == blockIdx.x) {                               \
    if ((i) == 1) g_stm_t[blockIdx.x * 8] = globaltimer_ns();                         \
    g_stm_t[blockIdx.x * 8 + (i)] = clock64();                                        \
  }
extern "C" void otk_debug_stm(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_stm_t, sizeof(g_stm_t)); }
#else
#define STM_T(i, who)
#endif
// kCl: one row per thread-block cluster of p.csize CTAs (batches of up to ~2 rows per SM): CTA `rank` streams the
// row's chunks [rank nchc, (rank + 1) nchc), its search warp pushes the CTA's (R_c, S_c) to every CTA of the cluster
// (st.async + mbarrier, as k_sample_dec) and the crossing CTA's search warp finishes the draw on its own segments.
template <typename T, bool kCl>
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
  const int C = kCl ? p.csize : 1;
  const int crank = kCl ? int(cluster_ctarank()) : 0;
  const int64_t row0 = kCl ? int64_t(cluster_id_x()) : int64_t(blockIdx.x);
  const int64_t rstride = kCl ? int64_t(nclusters_x()) : int64_t(gridDim.x);
  const int nchc = (nch + C - 1) / C;
  const int ch0 = min(nch, crank * nchc);                 // this CTA's chunks [ch0, ch0 + nloc) of every row
  const int nloc = max(0, min(nch, ch0 + nchc) - ch0);

#ifdef OTK_STM_TIMING
  {
    const int64_t row = blockIdx.x;
    STM_T(1, threadIdx.x == 0);
  }
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSSlots; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kSWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.hfull[i], kSWarps);
      mbar_init(&S.hempty[i], 1);
    }
    if (kCl) mbar_init(&S.xbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // kCl: publishes xbar's initialisation to the cluster; every thread waits once before its CTA's first push (the
  // loader at its end, long complete by then)
  if (kCl) asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
  if (kCl && warp != 0) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");

  if (warp == 0) {
    // ---------------- loader: every row, chunk by chunk
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t slot = 0, phase = 0;
      for (int64_t row = row0; row < p.num_rows; row += rstride) {
        const char* src = reinterpret_cast<const char*>(p.logits) + row * p.ld * int64_t(sizeof(T));
        for (int c = ch0; c < ch0 + nloc; ++c) {
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
    if (kCl) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
  } else if (warp <= kSWarps) {
    // ---------------- consumers
    const int ct = threadIdx.x - 32, cw = warp - 1;
    uint32_t slot = 0, phase = 0, par = 0, hph = 0;
    for (int64_t row = row0; row < p.num_rows; row += rstride) {
      mbar_wait(&S.hempty[par], hph ^ 1u);   // the search warp has read this parity's previous row
      float r = kSNoRef;                      // warp-uniform reference (k2 units)
      for (int lc = 0; lc < nloc; ++lc) {
        const int c = ch0 + lc;                  // the chunk's index in the row
        mbar_wait(&S.full[slot], phase);
        STM_T(2, c == 0 && ct == 0);
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
        if (lane == 0) S.part[par][lc][cw] = make_float2(cs, r);
      }
      __syncwarp();
      STM_T(3, ct == 0);
      if (lane == 0) mbar_arrive(&S.hfull[par]);
      par ^= 1u;
      if (par == 0) hph ^= 1u;
    }
  } else {
    // ---------------- search warp
    uint32_t par = 0, hph = 0;
    for (int64_t row = row0; row < p.num_rows; row += rstride) {
      mbar_wait(&S.hfull[par], hph);
      STM_T(4, lane == 0);
      // row reference R and total S: lane l takes the B contiguous segments [l B, (l + 1) B) (column order:
      // chunk-major, warp-minor), then one 32-lane scan of the lane totals
      const int nseg = nloc * kSWarps;
      const int B = (nseg + 31) / 32;
      const int i0 = min(lane * B, nseg), i1 = min(i0 + B, nseg);
      auto part_at = [&](int i) { return S.part[par][i / kSWarps][i % kSWarps]; };
      float rl = kSNoRef;
      for (int i = i0; i < i1; ++i) rl = fmaxf(rl, part_at(i).y);
      const float Rc = redux_max_f32(rl);                // this CTA's reference and sum (the row's unless kCl)
      float lt = 0.f;
      for (int i = i0; i < i1; ++i) {
        const float2 v = part_at(i);
        if (v.x > 0.f) lt = __fadd_rn(lt, __fmul_rn(v.x, ex2(v.y - Rc)));
      }
      float incl = lt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = __fadd_rn(incl, y);
      }
      const float Sc = __shfl_sync(0xffffffffu, incl, 31);
      float R = Rc, Sw = Sc, Pc = 0.f, fc = 1.f;        // row reference / sum; mass before this CTA; its scale
      float crr = 0.f, cir = 0.f, cer = 0.f;             // kCl: lane rr's CTA mass, inclusive / exclusive prefix
      if (kCl) {   // the C partials of the row (lane rr: CTA rr), identical in every CTA
        if (lane < C)
          st_async_f4(mapa(smem_u32(&S.peer[crank]), uint32_t(lane)), Rc, Sc, 0.f, 0.f,
                      mapa(smem_u32(&S.xbar), uint32_t(lane)));
        if (lane == 0) mbar_arrive_expect_tx(&S.xbar, 16u * uint32_t(C));
        mbar_wait_cluster(&S.xbar, 0);                   // one row per cluster: one phase
        const float4 pv = lane < C ? S.peer[lane] : make_float4(kSNoRef, 0.f, 0.f, 0.f);
        R = redux_max_f32(pv.x);
        crr = pv.y > 0.f ? __fmul_rn(pv.y, ex2(pv.x - R)) : 0.f;
        cir = crr;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, cir, o);
          if (lane >= o) cir = __fadd_rn(cir, y);
        }
        Sw = __shfl_sync(0xffffffffu, cir, 31);
        fc = ex2(Rc - R);
        const float up = __shfl_up_sync(0xffffffffu, cir, 1);
        cer = lane == 0 ? 0.f : up;
      }
      const bool degenerate = !(R > kSNoRef) || !(Sw > 0.f);
      const T* rbase = reinterpret_cast<const T*>(p.logits) + row * p.ld;
      int rs = 0;                                        // the crossing CTA (kCl)
      float u = 0.f, Tt = 0.f;
      if (!degenerate) {
        u = p.u[row];
        if (!(u >= 0.f && u < 1.f)) {
          if (lane == 0 && crank == 0) set_error(p.err, OTK_ERR_INVALID_ARG);
          u = fminf(fmaxf(u, 0.f), 0.99999994f);
        }
        Tt = u * Sw;
        if (!(Tt < Sw)) Tt = Sw * 0.99999976f;
        if (kCl) {   // rank order; fallback: the last CTA with mass
          const unsigned cr = __ballot_sync(0xffffffffu, lane < C && cir > Tt);
          const unsigned nzr = __ballot_sync(0xffffffffu, lane < C && crr > 0.f);
          rs = cr ? __ffs(cr) - 1 : 31 - __clz(nzr);
          Pc = __shfl_sync(0xffffffffu, cer, rs);
        }
      }
      if (degenerate || rs != crank) {   // no finite logit: token 0, logp -inf (as k_sample.cu); or not this CTA
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&S.hempty[par]);
          if (degenerate && crank == 0) {
            p.tokens[row] = 0;
            if (p.logp) p.logp[row] = -INFINITY;
          }
        }
      } else {
        // the crossing lane's range (fallback: the last lane with mass), then its segments one per lane, scanned;
        // masses in the row's units: P = Pc + fc x (this CTA's prefix at Rc)
        const unsigned cl = __ballot_sync(0xffffffffu, __fadd_rn(Pc, __fmul_rn(incl, fc)) > Tt);
        const unsigned nzl = __ballot_sync(0xffffffffu, lt > 0.f);
        const int L = cl ? __ffs(cl) - 1 : 31 - __clz(nzl);
        const float excl = __shfl_up_sync(0xffffffffu, incl, 1);
        const float Pb = L == 0 ? Pc : __fadd_rn(Pc, __fmul_rn(__shfl_sync(0xffffffffu, excl, L), fc));
        const int j0 = min(L * B, nseg), j1 = min(j0 + B, nseg);
        const int i = j0 + lane;
        float c = 0.f, f = 0.f;
        if (i < j1) {
          const float2 v = part_at(i);
          f = ex2(v.y - R);
          c = v.x > 0.f ? __fmul_rn(v.x, f) : 0.f;
        }
        float ic = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, ic, o);
          if (lane >= o) ic = __fadd_rn(ic, y);
        }
        const unsigned crs = __ballot_sync(0xffffffffu, i < j1 && __fadd_rn(Pb, ic) > Tt);
        const unsigned nzs = __ballot_sync(0xffffffffu, c > 0.f);
        const int l = crs ? __ffs(crs) - 1 : (nzs ? 31 - __clz(nzs) : 0);   // fallback: the last with mass
        const int seg = j0 + l;
        const float Pseg = __fadd_rn(Pb, __shfl_sync(0xffffffffu, ic - c, l));
        const float fseg = __shfl_sync(0xffffffffu, f, l);
        const int cstar = seg / kSWarps, wstar = seg % kSWarps;
        const float rseg = S.part[par][cstar][wstar].y;
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.hempty[par]);   // the hand-off buffer is no longer read
        // re-read the 1 KB segment (L2): lane l holds its vectors 2l, 2l+1 of thread-range (wstar, lane l)
        const int v0 = (ch0 + cstar) * (CE / EV) + 2 * (32 * wstar + lane);
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
      STM_T(5, lane == 0);
      par ^= 1u;
      if (par == 0) hph ^= 1u;
    }
  }
}

// =====================================================================================================
// k_sample_dec — decode-sized batches (a few to ~37 rows): ONE row per thread-block cluster of C CTAs. Each CTA's
// column range is loaded straight into registers (LDG.128, every load issued before any is used: the row is read
// once, in one round of memory latency, and never re-read), and the pass has no __syncthreads and no cluster
// barrier on its critical path:
//   warp w of a CTA owns K = ceil(segments / 16) CONTIGUOUS 1 KB segments (lane l: vectors 2l, 2l+1 of each); per
//     segment the sum of e = 2^(x k2 - r) at a warp-uniform reference r (k_sample_tm's scheme) and a running warp
//     total (R_w, S_w) in column order, plus the greedy (max, first column);
//   every warp PUSHES its partial to every CTA of the cluster (st.async + mbarrier complete_tx) and waits for the
//     16 C partials of the row: a CTA never reads a peer's shared memory and leaves only after every push to it has
//     landed, so there is no exit barrier;
//   every warp combines the 16 C partials in column order (rank-major, warp-minor; lane l takes 16 C / 32 of them):
//     max, scale, inclusive scan -> S, T = u S and the crossing warp of the row; that warp alone finds the
//     crossing segment (its K segment sums, sequentially), lane (warp scan) and column (one element per lane) from
//     its registers.
// The mbarrier's initialisation is published by a split cluster arrive (kernel start) / wait (after the segment
// pass, long complete). Same contract and rounding fallback as the other samplers (R32).
// =====================================================================================================
constexpr int kDecWarps = 16;
constexpr int kDecThreads = 32 * kDecWarps;
constexpr int kDecSeg = 1024;                        // bytes per segment (64 vectors: 2 per lane)
constexpr int kDecMaxK = 8;                          // segments per warp held in registers (64 registers of data)
constexpr int kDecMaxSegs = kDecWarps * kDecMaxK;    // 128 KB of row per CTA
constexpr int kDecMaxC = 8;

struct DecSmem {
  float4 peer[kDecMaxC * kDecWarps];                 // pushed warp partials (R_w, S_w, greedy max, first column),
  uint64_t xbar;                                     //   by rank * 16 + warp (column order)
};

#ifdef OTK_SDEC_TIMING  // experiments only, thread 0 of every CTA (<= 256 CTAs): [0] globaltimer (ns) at the start,
// [1 + i] clock64 at stamp i (SM cycles; reading the global timer costs far more than a clock read)
__device__ unsigned long long g_sdec_t[256 * 8];
#define SDEC_T(i)                                                                     \
  if (threadIdx.x == 0 && blockIdx.x < 256) {                                         \
    if ((i) == 0) g_sdec_t[blockIdx.x * 8] = globaltimer_ns();                        \
    g_sdec_t[blockIdx.x * 8 + 1 + (i)] = clock64();                                   \
  }
#else
#define SDEC_T(i)
#endif

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

#ifndef OTK_SDEC_MINB
#define OTK_SDEC_MINB 1   // resident CTAs per SM asked of the 4-segment variant
#endif
template <typename T, int KMAX>
__global__ void __launch_bounds__(kDecThreads, KMAX <= 4 ? OTK_SDEC_MINB : 1) k_sample_dec(const SampleParams p, int nseg_c) {
  using SV = SV2<T>;
  constexpr int EV = SV::EV;
  constexpr int VPS = kDecSeg / 16;                  // vectors per segment (64)
  __shared__ DecSmem S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.csize;
  const int rank = int(cluster_ctarank());
  const int64_t row = int64_t(cluster_id_x());
  const int nvec = int((p.vocab + EV - 1) / EV);
  const int tail_valid = int(p.vocab - int64_t(nvec - 1) * EV);
  const int K = (nseg_c + kDecWarps - 1) / kDecWarps;          // segments per warp (<= KMAX)
  const int sg0 = rank * nseg_c + warp * K;                    // this warp's first segment in the row
  const int sg1 = min(rank * nseg_c + min((warp + 1) * K, nseg_c), (nvec + VPS - 1) / VPS);
  const float k2 = p.scale * 1.4426950408889634f;
  const uint64_t k2x2 = f2(k2, k2);
  const bool greedy = p.greedy != 0;
  const bool need_sum = !(greedy && p.logp == nullptr);
  const uint4 ninf = sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                                    : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
  const uint8_t* rbase = reinterpret_cast<const uint8_t*>(p.logits) + row * p.ld * int64_t(sizeof(T));
  SDEC_T(0);

  // ---------------- the warp's segments into registers: every load issued before any is used
  uint4 q[KMAX][2];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int v = (sg0 + k) * VPS + 2 * lane + j;
      q[k][j] = (sg0 + k < sg1 && v < nvec) ? ldg_nc_v4(rbase + size_t(v) * 16) : ninf;
    }
  const float u_in = greedy ? 0.f : p.u[row];
  if (threadIdx.x == 0) {
    mbar_init(&S.xbar, 1);
    fence_mbar_init();
  }
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");   // publishes xbar's init (waited below)

  // ---------------- segments (column order): the warp's maximum is the reference of all its segments, so no sum
  // can overflow (e <= 1, <= 512 per segment) and the segments' warp sums are independent of one another
  float lm = -INFINITY;                              // the lane's maximum (raw logits)
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int v = (sg0 + k) * VPS + 2 * lane + j;
      if (v == nvec - 1 && tail_valid < EV) SV::mask_tail(q[k][j], tail_valid);
      lm = fmaxf(lm, SV::vmax(q[k][j]));            // ninf outside the range
    }
  const float wmax = redux_max_f32(lm);
  const float r = wmax * k2;                         // warp-uniform reference (k2 units); <= kSNoRef: no mass
  const bool has_mass = need_sum && r > kSNoRef;
  float cs_l[KMAX], cs_k[KMAX];                      // per segment: the lane's / the warp's sum of e at r
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    cs_l[k] = 0.f;
    if (has_mass && sg0 + k < sg1) {
      const float rk = -r;
      const uint64_t rk2 = f2(rk, rk);
      cs_l[k] = __fadd_rn(SV::esum(q[k][0], k2x2, rk2), SV::esum(q[k][1], k2x2, rk2));
    }
    cs_k[k] = cs_l[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < KMAX; ++k) cs_k[k] = __fadd_rn(cs_k[k], __shfl_xor_sync(0xffffffffu, cs_k[k], o));
  float sacc = 0.f;                                  // the warp's total at r (column order)
#pragma unroll
  for (int k = 0; k < KMAX; ++k) sacc = __fadd_rn(sacc, cs_k[k]);
  const float racc = has_mass ? r : kSNoRef;
  float best = -INFINITY;
  int bidx = INT_MAX;
  if (greedy) {  // the first column holding the warp's maximum
    int li = INT_MAX;
    if (lm == wmax && wmax > -INFINITY) {
#pragma unroll
      for (int k = KMAX - 1; k >= 0; --k)
#pragma unroll
        for (int j = 1; j >= 0; --j)
#pragma unroll
          for (int i = EV - 1; i >= 0; --i)
            if (SV::elem(q[k][j], i) == lm) li = ((sg0 + k) * VPS + 2 * lane + j) * EV + i;
    }
    best = wmax;
    bidx = redux_min_s32(li);
  }
  SDEC_T(1);
  // ---------------- push the warp partial to every CTA of the cluster (lane rr -> rank rr)
  asm volatile("barrier.cluster.wait.acquire;" ::: "memory");   // every CTA's xbar is initialised
  if (lane < C)
    st_async_f4(mapa(smem_u32(&S.peer[rank * kDecWarps + warp]), uint32_t(lane)), racc, sacc, best,
                __int_as_float(bidx), mapa(smem_u32(&S.xbar), uint32_t(lane)));
  if (threadIdx.x == 0) mbar_arrive_expect_tx(&S.xbar, 16u * kDecWarps * uint32_t(C));
  mbar_wait_cluster(&S.xbar, 0);
  SDEC_T(2);

  // ---------------- the 16 C warp partials in column order, identical in every warp of every CTA:
  // lane l holds partials [l NP, (l + 1) NP)
  const int NP = (kDecWarps * C + 31) / 32;          // <= 4
  float4 pv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = lane * NP + i;
    pv[i] = (i < NP && idx < kDecWarps * C) ? S.peer[idx]
                                            : make_float4(kSNoRef, 0.f, -INFINITY, __int_as_float(INT_MAX));
  }
  const float R = redux_max_f32(fmaxf(fmaxf(pv[0].x, pv[1].x), fmaxf(pv[2].x, pv[3].x)));
  SDEC_T(3);
  float B = -INFINITY;
  int I = INT_MAX;
  if (greedy) {
    B = redux_max_f32(fmaxf(fmaxf(pv[0].z, pv[1].z), fmaxf(pv[2].z, pv[3].z)));
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (pv[i].z == B) I = min(I, __float_as_int(pv[i].w));
    I = redux_min_s32(I);
  }
  float c[4], lt = 0.f;                              // masses at R, the lane's total
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    c[i] = pv[i].y > 0.f ? __fmul_rn(pv[i].y, ex2(pv[i].x - R)) : 0.f;
    lt = __fadd_rn(lt, c[i]);
  }
  float incl = lt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = __fadd_rn(incl, y);
  }
  const float Sw = __shfl_sync(0xffffffffu, incl, 31);
  SDEC_T(4);
  // as the other samplers (R32): logits <= -1e30 carry no mass, a row without any larger one is degenerate
  const bool degenerate = greedy ? !(B > -1e30f) || (need_sum && !(Sw > 0.f)) : (!(R > kSNoRef) || !(Sw > 0.f));
  if (greedy || degenerate) {
    if (rank == 0 && threadIdx.x == 0) {
      p.tokens[row] = degenerate ? 0 : I;
      if (p.logp) p.logp[row] = degenerate ? -INFINITY : (B * k2 - R - log2f(Sw)) * 0.6931471805599453f;
    }
  } else {
    float u = u_in;
    if (!(u >= 0.f && u < 1.f)) {
      if (threadIdx.x == 0 && rank == 0) set_error(p.err, OTK_ERR_INVALID_ARG);
      u = fminf(fmaxf(u, 0.f), 0.99999994f);
    }
    float Tt = u * Sw;
    if (!(Tt < Sw)) Tt = Sw * 0.99999976f;
    // crossing lane, then its crossing partial (column order); fallback: the last partial with mass
    const unsigned cl = __ballot_sync(0xffffffffu, incl > Tt);
    const unsigned nzl = __ballot_sync(0xffffffffu, lt > 0.f);
    const int L = cl ? __ffs(cl) - 1 : 31 - __clz(nzl);
    float P = __shfl_sync(0xffffffffu, __fadd_rn(incl, -lt), L);   // mass before lane L's partials
    int X = -1, Xl = -1;
    float Px = 0.f, Pl = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float ci = __shfl_sync(0xffffffffu, c[i], L);
      if (i < NP) {
        const float Pn = __fadd_rn(P, ci);
        if (ci > 0.f) {
          Xl = L * NP + i;
          Pl = P;
        }
        if (X < 0 && Pn > Tt) {
          X = L * NP + i;
          Px = P;
        }
        P = Pn;
      }
    }
    if (X < 0) {
      X = Xl;
      Px = Pl;
    }
    SDEC_T(5);
    if (X == rank * kDecWarps + warp) {
      // this warp holds the crossing: segment (sequential over its K), lane (warp scan), column (one per lane);
      // every segment of the warp is at its reference racc
      const float fseg = ex2(racc - R);
      int ks = -1, kl = 0;
      float Pseg = Px, Plast = Px, Pk = Px;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (sg0 + k < sg1) {
          const float ck = __fmul_rn(cs_k[k], fseg);
          const float Pn = __fadd_rn(Pk, ck);
          if (ck > 0.f) {
            kl = k;
            Plast = Pk;
          }
          if (ks < 0 && Pn > Tt) {
            ks = k;
            Pseg = Pk;
          }
          Pk = Pn;
        }
      }
      if (ks < 0) {
        ks = kl;
        Pseg = Plast;
      }
      uint4 qa = ninf, qb = ninf;
      float ls = 0.f;                                // the lane's sum of the segment (the pass's value, bit for bit)
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k == ks) {
          qa = q[k][0];
          qb = q[k][1];
          ls = cs_l[k];
        }
      const int v0 = (sg0 + ks) * VPS + 2 * lane;
      const float rk = -racc;
      float li = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, li, o);
        if (lane >= o) li = __fadd_rn(li, y);
      }
      const unsigned cross = __ballot_sync(0xffffffffu, __fadd_rn(Pseg, __fmul_rn(li, fseg)) > Tt);
      const unsigned nz = __ballot_sync(0xffffffffu, ls > 0.f);
      const int lw = cross ? __ffs(cross) - 1 : (nz ? 31 - __clz(nz) : 0);
      // lane lw's 2 EV elements, one per lane (column order), scanned across the warp
      const float base = __shfl_sync(0xffffffffu, __fadd_rn(Pseg, __fmul_rn(li - ls, fseg)), lw);
      uint4 qq[2];
      qq[0].x = __shfl_sync(0xffffffffu, qa.x, lw);
      qq[0].y = __shfl_sync(0xffffffffu, qa.y, lw);
      qq[0].z = __shfl_sync(0xffffffffu, qa.z, lw);
      qq[0].w = __shfl_sync(0xffffffffu, qa.w, lw);
      qq[1].x = __shfl_sync(0xffffffffu, qb.x, lw);
      qq[1].y = __shfl_sync(0xffffffffu, qb.y, lw);
      qq[1].z = __shfl_sync(0xffffffffu, qb.z, lw);
      qq[1].w = __shfl_sync(0xffffffffu, qb.w, lw);
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
      const int le = hit ? __ffs(hit) - 1 : (enz ? 31 - __clz(enz) : 0);  // fallback: the last column with mass
      const float xt = __shfl_sync(0xffffffffu, x, le);
      if (lane == 0) {
        p.tokens[row] = vl * EV + le;
        if (p.logp) p.logp[row] = (xt * k2 - R - log2f(Sw)) * 0.6931471805599453f;
      }
    }
  }
  SDEC_T(6);
}
#ifdef OTK_SDEC_TIMING
extern "C" void otk_debug_sdec(unsigned long long* out) {  // out: [256][8]
  cudaMemcpyFromSymbol(out, g_sdec_t, sizeof(g_sdec_t));
}
#endif

namespace {
template <int KMAX>
const void* dec_kernel(int dtype) {
  return dtype == OTK_BF16 ? reinterpret_cast<const void*>(k_sample_dec<__nv_bfloat16, KMAX>)
                           : reinterpret_cast<const void*>(k_sample_dec<float, KMAX>);
}
const void* dec_kernel(int dtype, int nseg_c) {
  return nseg_c <= kDecWarps * 4 ? dec_kernel<4>(dtype) : dec_kernel<8>(dtype);
}
// clusters of c CTAs of this kernel that can be resident at once (cached; the same for every B200)
int dec_max_clusters(int dtype, int nseg_c, int c) {
  static int cache[2][2][kDecMaxC + 1];
  static bool init = false;
  if (!init) {
    for (auto& a : cache)
      for (auto& b : a)
        for (int& v : b) v = -1;
    init = true;
  }
  int& slot = cache[dtype == OTK_BF16][nseg_c > kDecWarps * 4][c];
  if (slot < 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(c), 1, 1);
    cfg.blockDim = dim3(kDecThreads, 1, 1);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(c);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, dec_kernel(dtype, nseg_c), &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    slot = n;
  }
  return slot;
}
}  // namespace

// the decode kernel's shape for this batch, or false: the largest C <= 8 CTAs per row (>= 4) whose clusters are
// all resident at once (one wave), with at most kDecMaxSegs segments per CTA
bool sample_dec_shape(int64_t num_rows, int64_t vocab, int dtype, int num_sms, int* csize, int* nseg_c) {
  const int64_t nvec = (vocab * (dtype == OTK_BF16 ? 2 : 4) + 15) / 16;
  const int64_t nsegs = (nvec + 63) / 64;
  if (num_rows < 1 || num_rows > num_sms) return false;
  // at least 3 CTAs per row (<= 49 rows on 148 SMs), the whole range in registers
#ifndef OTK_SDEC_MINC
#define OTK_SDEC_MINC 3
#endif
  for (int64_t c = std::min<int64_t>(kDecMaxC, num_sms / num_rows); c >= OTK_SDEC_MINC; --c) {
    const int64_t per = (nsegs + c - 1) / c;
    if (per > kDecMaxSegs) return false;
    if (dec_max_clusters(dtype, int(per), int(c)) < num_rows) continue;
    *csize = int(c);
    *nseg_c = int(per);
    return true;
  }
  return false;
}

cudaError_t launch_sample_dec(otk_ctx* ctx, SampleParams p, int dtype, int csize, int nseg_c, cudaStream_t s) {
  p.csize = csize;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(p.num_rows * csize), 1, 1);
  cfg.blockDim = dim3(kDecThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(csize);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) -> cudaError_t {
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, nseg_c);
    return e != cudaSuccess ? e : cudaGetLastError();
  };
  const bool small = nseg_c <= kDecWarps * 4;   // <= 4 segments per warp: half the registers of data
  if (dtype == OTK_BF16) return small ? go(k_sample_dec<__nv_bfloat16, 4>) : go(k_sample_dec<__nv_bfloat16, 8>);
  return small ? go(k_sample_dec<float, 4>) : go(k_sample_dec<float, 8>);
}

bool sample_tm_fits(int64_t vocab, int dtype) {
  const int64_t rb = (vocab * (dtype == OTK_BF16 ? 2 : 4) + 15) / 16 * 16;
  return (rb + kSChunk - 1) / kSChunk <= kSampleTmMaxChunks;
}

namespace {
// resident clusters of c CTAs of k_sample_tm<T, true> (cached; the same on every B200)
template <typename T>
int stm_max_clusters(int c) {
  static int cache[9] = {};
  int& slot = cache[c];
  if (slot == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(c), 1, 1);
    cfg.blockDim = dim3(kSThreads, 1, 1);
    cfg.dynamicSmemBytes = kSSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(c);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_sample_tm<T, true>, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    slot = n > 0 ? n : -1;
  }
  return slot;
}

template <typename T>
cudaError_t launch_stm(otk_ctx* ctx, SampleParams p, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_sample_tm<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSSmemBytes));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_sample_tm<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSSmemBytes));
  if (e != cudaSuccess) return e;
  // up to two rows per SM: split each row over a cluster of C CTAs (C = the largest <= 8 with C x rows <= the
  // resident-CTA slots whose clusters all fit at once); more rows: one CTA per row, two per SM, persistent
#ifndef OTK_STM_NO_CLUSTER
  for (int c = int(std::min<int64_t>(8, 2 * int64_t(ctx->num_sms) / p.num_rows)); c >= 2; --c) {
    if (stm_max_clusters<T>(c) < p.num_rows) continue;
    p.csize = c;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(p.num_rows * c), 1, 1);
    cfg.blockDim = dim3(kSThreads, 1, 1);
    cfg.dynamicSmemBytes = kSSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(c);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_sample_tm<T, true>, p);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
#endif
  p.csize = 1;
  const int grid = int(std::min<int64_t>(p.num_rows, int64_t(ctx->num_sms) * 2));
  k_sample_tm<T, false><<<grid, kSThreads, kSSmemBytes, s>>>(p);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_sample_tm(otk_ctx* ctx, const SampleParams& p, int dtype, cudaStream_t s) {
  return dtype == OTK_BF16 ? launch_stm<__nv_bfloat16>(ctx, p, s) : launch_stm<float>(ctx, p, s);
}

}  // namespace otk
