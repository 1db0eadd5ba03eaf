// k_sample.cu — otk_sample_tokens (rollout-side sampling; R32).
// PAPER.md:170-171 (GENERATING: "the agent model generates tokens autoregressively")
// sample_token (softmax(logits / temperature), returns token and its probability) and greedy_token
// (argmax, ties to the lowest token id).
//
// A row is split over a thread-block cluster of C CTAs (C chosen per launch so that rows x C fills the
// GPU; C = 1 for large batches), each CTA over 8 warps, each warp over a contiguous column range read
// lane-strided (16-byte vectors, 4 in flight per lane). ONE read of the row from HBM:
//   main pass: per lane an online (max m, sum 2^{(x-m) s log2 e}) with a rescale when the max grows,
//              plus (greedy) the vector holding the lane's first maximum; warp / CTA / cluster combine
//              in a fixed order (DSMEM reads of the CTA partials after one cluster barrier per row).
//   sample:    T = u S; the crossing CTA r* and, inside it, the crossing warp w* follow from the
//              prefix sums of the partials in column order; then ALL threads of CTA r* re-read warp
//              w*'s range (1/(8C) of the row, L2-resident), each a contiguous slice, a CTA scan of the
//              slice sums finds the crossing thread and that thread's elements, in column order, give
//              t = min{t : cdf_t > T}.
// fp32 rounding of the prefix sums can place T an ulp outside the located range; the last column with
// non-zero mass is then taken (the draw is within rounding of a cdf boundary, where both neighbours
// are correct — DESIGN.md R32).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "otk_internal.h"
#include "otk_ptx.cuh"

namespace otk {

using namespace ptx;

constexpr int kSampleThreads = 256;
constexpr int kSampleWarps = kSampleThreads / 32;
constexpr int kSampleMaxCluster = 8;
#ifndef OTK_SAMPLE_MINB
#define OTK_SAMPLE_MINB 4  // resident CTAs per SM the register budget is sized for
#endif

template <typename T>
struct SVec;
template <>
struct SVec<__nv_bfloat16> {
  static constexpr int EV = 8;
  static constexpr uint32_t kNegInf = 0xff80ff80u;  // two bf16 -inf
  __device__ static float vmax(const uint4& q) {
    const uint32_t a = bmax2(bmax2(q.x, q.y), bmax2(q.z, q.w));
    return fmaxf(bf_lo(a), bf_hi(a));
  }
  __device__ static float elem(const uint4& q, int i) {
    const uint32_t w = i < 2 ? q.x : i < 4 ? q.y : i < 6 ? q.z : q.w;
    return (i & 1) ? bf_hi(w) : bf_lo(w);
  }
  // columns >= n_valid of this vector -> -inf
  __device__ static void mask_tail(uint4& q, int n_valid) {
    uint32_t* w = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (2 * k >= n_valid) w[k] = kNegInf;
      else if (2 * k + 1 >= n_valid) w[k] = (w[k] & 0xffffu) | 0xff800000u;
    }
  }
  // acc += (2^{x k2 + mk} for the 8 elements), pairwise in column order
  __device__ static uint64_t acc(const uint4& q, uint64_t k2x2, uint64_t mkx2, uint64_t a) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float d0, d1;
      f2_split(ffma2(f2(bf_lo(w[k]), bf_hi(w[k])), k2x2, mkx2), d0, d1);
      a = fadd2(a, f2(ex2(d0), ex2(d1)));
    }
    return a;
  }
  __device__ static float load1(const void* base, int64_t i) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  }
};
template <>
struct SVec<float> {
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
  __device__ static uint64_t acc(const uint4& q, uint64_t k2x2, uint64_t mkx2, uint64_t a) {
    float d0, d1, d2, d3;
    f2_split(ffma2(f2(__uint_as_float(q.x), __uint_as_float(q.y)), k2x2, mkx2), d0, d1);
    f2_split(ffma2(f2(__uint_as_float(q.z), __uint_as_float(q.w)), k2x2, mkx2), d2, d3);
    a = fadd2(a, f2(ex2(d0), ex2(d1)));
    return fadd2(a, f2(ex2(d2), ex2(d3)));
  }
  __device__ static float load1(const void* base, int64_t i) { return reinterpret_cast<const float*>(base)[i]; }
};

// 2^{(m_from - m_to) k2}: moves a partial sum from reference m_from to m_to (the -1e30 "no finite
// logit yet" reference gives 0)
__device__ __forceinline__ float rescale(float m_from, float m_to, float k2) { return ex2((m_from - m_to) * k2); }

__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

constexpr float kNoRef = -1e30f;  // reference before the first finite logit (logits <= -1e30 carry no mass)

template <typename T, bool kCl, int kMinB = OTK_SAMPLE_MINB>
__global__ void __launch_bounds__(kSampleThreads, kMinB) k_sample(const SampleParams p) {
  using SV = SVec<T>;
  constexpr int EV = SV::EV;
#ifndef OTK_SAMPLE_U
#define OTK_SAMPLE_U 4
#endif
  constexpr int U = OTK_SAMPLE_U;  // vectors in flight per lane
  __shared__ float s_wm[kSampleWarps], s_ws[kSampleWarps], s_wb[kSampleWarps];
  __shared__ int s_wi[kSampleWarps];
  __shared__ __align__(16) float s_cta[2][4];  // this CTA's (M, S, argmax, max) by row parity, read over DSMEM
  __shared__ float s_scan[kSampleWarps];
  __shared__ int s_first, s_lastnz;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int C = kCl ? p.csize : 1;
  const int rank = kCl ? int(cluster_ctarank()) : 0;
  const int64_t group = kCl ? int64_t(cluster_id_x()) : int64_t(blockIdx.x);
  const int64_t ngroups = kCl ? int64_t(nclusters_x()) : int64_t(gridDim.x);
  const int nvec = int((p.vocab + EV - 1) / EV);
  const int tail_valid = int(p.vocab - int64_t(nvec - 1) * EV);  // columns of the last vector
  const int nvc = (nvec + C - 1) / C;
  const int c_v0 = min(rank * nvc, nvec), c_v1 = min(c_v0 + nvc, nvec);
  const int nvw = (c_v1 - c_v0 + kSampleWarps - 1) / kSampleWarps;
  const int w_v0 = min(c_v0 + warp * nvw, c_v1), w_v1 = min(w_v0 + nvw, c_v1);
  // the partial last vector of the row (if any) is peeled out of the main loop
  const bool has_tail = tail_valid < EV && w_v1 == nvec && w_v0 < w_v1;
  const int w_main1 = has_tail ? nvec - 1 : w_v1;
  const bool tail_lane = has_tail && ((nvec - 1 - w_v0) & 31) == lane;
  const float k2 = p.scale * 1.4426950408889634f;
  const float thr = 32.f / k2;  // raise the reference only when values would pass 2^32
  const uint64_t k2x2 = f2(k2, k2);
  const bool greedy = p.greedy != 0;
  const bool need_sum = !(greedy && p.logp == nullptr);  // greedy without logp: the argmax needs no exponentials

  int parity = 0;
  for (int64_t row = group; row < p.num_rows; row += ngroups, parity ^= 1) {
    const T* rbase = reinterpret_cast<const T*>(p.logits) + row * p.ld;
    const uint4* rp = reinterpret_cast<const uint4*>(rbase);

    // ---------------- main pass. Per lane: a reference m, raised only when a vector's max exceeds it by
    // more than 32 binades of 2^{x k2} (so the common vector needs no rescale), and the pair sum of
    // 2^{x k2 - m k2}; greedy also keeps the lane's first maximum (value, vector index).
    float m = kNoRef;
    uint64_t a2 = f2(0.f, 0.f), mk2 = f2(-kNoRef * k2, -kNoRef * k2);
    float best = -INFINITY;
    int bv = -1;
    auto consume = [&](const uint4& q, int vk) {
      const float vm = SV::vmax(q);
      if (vm > m + thr) {
        const float r = rescale(m, vm, k2);
        a2 = fmul2(a2, f2(r, r));
        m = vm;
        const float mk = -vm * k2;
        mk2 = f2(mk, mk);
      }
      if (need_sum) a2 = SV::acc(q, k2x2, mk2, a2);
      if (greedy && vm > best) {
        best = vm;
        bv = vk;
      }
    };
    {
      const uint4* end = rp + w_main1;
      for (const uint4* ptr = rp + w_v0 + lane; ptr < end; ptr += 32 * U) {
        uint4 q[U];
#pragma unroll
        for (int k = 0; k < U; ++k)
          if (ptr + 32 * k < end) q[k] = __ldg(ptr + 32 * k);
#pragma unroll
        for (int k = 0; k < U; ++k)
          if (ptr + 32 * k < end) consume(q[k], int(ptr - rp) + 32 * k);
      }
      if (tail_lane) {
        uint4 q = __ldg(rp + nvec - 1);
        SV::mask_tail(q, tail_valid);
        consume(q, nvec - 1);
      }
    }
    // ---------------- warp combine: reference M_w, S_w; greedy: max B_w and its first index
    float Mw = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
    float sl = f2_sum(a2) * rescale(m, Mw, k2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
    float Bw = best;
    int idx = INT_MAX;
    if (greedy) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Bw = fmaxf(Bw, __shfl_xor_sync(0xffffffffu, Bw, o));
      if (bv >= 0 && best == Bw) {
        uint4 q = __ldg(rp + bv);
        if (bv == nvec - 1) SV::mask_tail(q, tail_valid);
        for (int i = EV - 1; i >= 0; --i)
          if (SV::elem(q, i) == best) idx = bv * EV + i;  // first element equal to the max
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) idx = min(idx, __shfl_xor_sync(0xffffffffu, idx, o));
    }
    if (lane == 0) {
      s_wm[warp] = Mw;
      s_ws[warp] = sl;
      s_wb[warp] = Bw;
      s_wi[warp] = idx;
    }
    __syncthreads();
    // ---------------- CTA combine (warp order), then cluster combine (rank order)
    float Mc = kNoRef, Bc = -INFINITY;
    for (int w = 0; w < kSampleWarps; ++w) {
      Mc = fmaxf(Mc, s_wm[w]);
      Bc = fmaxf(Bc, s_wb[w]);
    }
    float Sc = 0.f;
    int Ic = INT_MAX;
    for (int w = 0; w < kSampleWarps; ++w) {
      Sc += s_ws[w] * rescale(s_wm[w], Mc, k2);
      if (greedy && s_wb[w] == Bc) Ic = min(Ic, s_wi[w]);
    }
    float M = Mc, S = Sc, B = Bc;
    int I = Ic;
    uint32_t cbase = 0;  // DSMEM address of s_cta[parity] (partials are re-read, not kept in registers)
    auto part = [&](int r, float& Mr, float& Sr) {
      if (kCl) {
        const uint32_t ra = mapa(cbase, uint32_t(r));
        Mr = ld_cluster_f32(ra);
        Sr = ld_cluster_f32(ra + 4);
      } else {
        Mr = Mc;
        Sr = Sc;
      }
    };
    if (kCl) {
      if (tid == 0) {
        s_cta[parity][0] = Mc;
        s_cta[parity][1] = Sc;
        s_cta[parity][2] = __int_as_float(Ic);
        s_cta[parity][3] = Bc;
      }
      cluster_sync_all();
      cbase = smem_u32(&s_cta[parity][0]);
      M = kNoRef;
      B = -INFINITY;
      I = INT_MAX;
      for (int r = 0; r < C; ++r) {
        const uint32_t ra = mapa(cbase, uint32_t(r));
        M = fmaxf(M, ld_cluster_f32(ra));
        if (greedy) {
          const float br = ld_cluster_f32(ra + 12);
          const int ir = __float_as_int(ld_cluster_f32(ra + 8));
          if (br > B) {
            B = br;
            I = ir;
          } else if (br == B) {
            I = min(I, ir);
          }
        }
      }
      S = 0.f;
      for (int r = 0; r < C; ++r) {
        float mr, sr;
        part(r, mr, sr);
        S += sr * rescale(mr, M, k2);
      }
    }
    const bool degenerate = !(M > kNoRef) || (need_sum && !(S > 0.f));  // no finite logit above -1e30
#ifndef OTK_SAMPLE_NO_PREFETCH
    // warm L2 with the start of this thread's slice of the next row while the search below (latency-bound)
    // runs, so the next row's main pass starts from L2 rather than HBM
    if (!greedy && row + ngroups < p.num_rows) {
      const uint4* np = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(p.logits) + (row + ngroups) * p.ld);
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int v = w_v0 + lane + 32 * k;
        if (v < w_v1) asm volatile("prefetch.global.L2 [%0];" ::"l"(np + v));
      }
    }
#endif

    if (greedy || degenerate) {
      if (rank == 0 && tid == 0) {
        p.tokens[row] = degenerate ? 0 : I;
        if (p.logp) p.logp[row] = degenerate ? -INFINITY : ((B - M) * k2 - log2f(S)) * 0.6931471805599453f;
      }
    } else {
      float u = p.u[row];
      if (!(u >= 0.f && u < 1.f)) {
        if (tid == 0 && rank == 0) set_error(p.err, OTK_ERR_INVALID_ARG);
        u = fminf(fmaxf(u, 0.f), 0.99999994f);
      }
      float Tt = u * S;
      if (!(Tt < S)) Tt = S * 0.99999976f;  // u*S rounded up to S: keep the target inside the mass
      // crossing CTA (rank order)
      int rs = -1;
      float P = 0.f, Pc = 0.f, Plast = 0.f;
      int rlast = 0;
      for (int r = 0; r < C; ++r) {
        float mr, sr;
        part(r, mr, sr);
        const float c = sr * rescale(mr, M, k2);
        if (c > 0.f) {
          rlast = r;
          Plast = P;
        }
        const float Pn = P + c;
        if (Pn > Tt) {
          rs = r;
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
        // crossing warp (warp order)
        int ws = -1, wlast = 0;
        float Pw = Pc, Pwl = Pc;
        P = Pc;
        for (int w = 0; w < kSampleWarps; ++w) {
          const float c = s_ws[w] * rescale(s_wm[w], M, k2);
          if (c > 0.f) {
            wlast = w;
            Pwl = P;
          }
          const float Pn = P + c;
          if (Pn > Tt) {
            ws = w;
            Pw = P;
            break;
          }
          P = Pn;
        }
        if (ws < 0) {
          ws = wlast;
          Pw = Pwl;
        }
        // ---------------- pass 3: the whole CTA over warp ws's range, a contiguous slice per thread
        const int a0 = min(c_v0 + ws * nvw, c_v1), a1 = min(a0 + nvw, c_v1);
        const int per = (a1 - a0 + kSampleThreads - 1) / kSampleThreads;
        const int t0 = min(a0 + tid * per, a1), t1 = min(t0 + per, a1);
        const float MK = -M * k2;
        const uint64_t MK2 = f2(MK, MK);
        uint64_t c2 = f2(0.f, 0.f);
        for (int v = t0; v < t1; v += U) {
          uint4 q[U];
#pragma unroll
          for (int k = 0; k < U; ++k)
            if (v + k < t1) q[k] = __ldg(rp + v + k);
#pragma unroll
          for (int k = 0; k < U; ++k) {
            if (v + k >= t1) break;
            if (v + k == nvec - 1) SV::mask_tail(q[k], tail_valid);
            c2 = SV::acc(q[k], k2x2, MK2, c2);
          }
        }
        const float ct = f2_sum(c2);
        // CTA inclusive scan of ct in thread (= column) order
        float incl = ct;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) s_scan[warp] = incl;
        if (tid == 0) {
          s_first = INT_MAX;
          s_lastnz = -1;
        }
        __syncthreads();
        float wbase = 0.f;
        for (int w = 0; w < warp; ++w) wbase += s_scan[w];
        const float base = Pw + wbase + (incl - ct);  // prefix before this thread's slice
        if (Pw + wbase + incl > Tt) atomicMin(&s_first, tid);
        if (ct > 0.f) atomicMax(&s_lastnz, tid);
        __syncthreads();
        const int winner = s_first != INT_MAX ? s_first : max(s_lastnz, 0);
        if (tid == winner) {
          // walk the slice element by element (L1 / L2 hits), first column whose prefix passes T
          float acc = base;
          int t = -1, tnz = -1;
          float xt = 0.f, xnz = 0.f;
          for (int v = t0; v < t1 && t < 0; ++v) {
            uint4 q = __ldg(rp + v);
            if (v == nvec - 1) SV::mask_tail(q, tail_valid);
#pragma unroll
            for (int i = 0; i < EV; ++i) {
              const float x = SV::elem(q, i);
              const float e = ex2(fmaf(x, k2, MK));
              acc += e;
              if (e > 0.f) {
                tnz = v * EV + i;
                xnz = x;
              }
              if (t < 0 && acc > Tt) {
                t = v * EV + i;
                xt = x;
              }
            }
          }
          if (t < 0) {
            t = tnz >= 0 ? tnz : a0 * EV;
            xt = tnz >= 0 ? xnz : SV::load1(rbase, t);
          }
          p.tokens[row] = t;
          if (p.logp) p.logp[row] = ((xt - M) * k2 - log2f(S)) * 0.6931471805599453f;
        }
      }
    }
    __syncthreads();  // s_wm / s_ws / s_scan reused by the next row (s_cta is double-buffered)
  }
  if (kCl) cluster_sync_all();  // no CTA exits while a peer may still read its s_cta
}

// resident CTAs per SM of the clustered variant (the launch shape depends on it); cached in the ctx per (dtype,
// register budget)
template <typename T, int kMinB>
int sample_occupancy(otk_ctx* ctx, int slot) {
  int& o = ctx->sample_occ[slot];
  if (o == 0) {
    int a = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_sample<T, true, kMinB>, kSampleThreads, 0);
    o = std::max(a, 1);
  }
  return o;
}

// resident clusters of c CTAs of k_sample<T, true, kMinB> (cached per process; the same on every B200)
template <typename T, int kMinB>
int sample_max_clusters(int c) {
  static int cache[kSampleMaxCluster + 1] = {};
  int& slot = cache[c];
  if (slot == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(c), 1, 1);
    cfg.blockDim = dim3(kSampleThreads, 1, 1);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(c);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_sample<T, true, kMinB>, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    slot = n > 0 ? n : -1;
  }
  return slot;
}

template <typename T, int kMinB>
static cudaError_t launch_lane_strided(otk_ctx* ctx, SampleParams p, cudaStream_t s, int occ_slot) {
  const int64_t slots = int64_t(ctx->num_sms) * sample_occupancy<T, kMinB>(ctx, occ_slot);
  // cluster size: when rows are few, as many CTAs per row as fit in ONE wave of resident CTAs; one CTA
  // per row otherwise (a cluster barrier per row costs more than the last wave's imbalance)
  // per-row time ~ (rows per cluster) / (CTAs per row); clusters of c are placed by GPC, so fewer than slots / c of
  // them may be resident at once (cudaOccupancyMaxActiveClusters): a cluster size whose clusters do not all fit
  // would run a second wave (48 rows in 6-CTA clusters: 18.4 us)
  int best_c = 1;
  int64_t groups = std::min<int64_t>(p.num_rows, slots);
  {
    double best_t = 1e30;
    for (int c = int(std::min<int64_t>(kSampleMaxCluster, std::max<int64_t>(1, slots / p.num_rows))); c >= 1; --c) {
      const int64_t fit = c == 1 ? slots : std::min<int64_t>(slots / c, sample_max_clusters<T, kMinB>(c));
      if (fit < 1) continue;
      const int64_t g = std::min<int64_t>(p.num_rows, fit);
      const double t = double((p.num_rows + g - 1) / g) / c;
      if (t < best_t) {
        best_t = t;
        best_c = c;
        groups = g;
      }
    }
  }
  p.csize = best_c;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(groups * best_c), 1, 1);
  cfg.blockDim = dim3(kSampleThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(best_c);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (best_c == 1) {
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, k_sample<T, false, kMinB>, p);
  }
  return cudaLaunchKernelEx(&cfg, k_sample<T, true, kMinB>, p);
}

cudaError_t launch_sample(otk_ctx* ctx, const SampleParams& p0, int dtype, cudaStream_t s) {
#ifndef OTK_SAMPLE_NO_DEC
  // decode batches (<= num_sms / 3 rows where the clusters fit; each CTA's range held in registers): k_sample_dec
  {
    int csize = 0, nseg_c = 0;
    if (sample_dec_shape(p0.num_rows, p0.vocab, dtype, ctx->num_sms, &csize, &nseg_c))
      return launch_sample_dec(ctx, p0, dtype, csize, nseg_c, s);
  }
#endif
#ifndef OTK_SAMPLE_V1
  // sampled draws above the decode kernel's range: the ring-streamed kernel with an off-path search warp
  // (k_sample_tm.cu; up to two rows per SM each row split over a cluster of 2-8 CTAs, one CTA per row beyond):
  // 48 rows 8.9 vs 10.7 us, 64 rows 10.4 vs 12.0 lane-strided, 128 rows 14.1 us, 4096 rows 208 vs 262 us;
  // greedy stays here at every size (its lane-strided pass measured faster: 225 vs 272 us at 4096 rows).
#ifndef OTK_SAMPLE_TM_MIN_ROWS
#define OTK_SAMPLE_TM_MIN_ROWS 38
#endif
  if (!p0.greedy && p0.num_rows >= std::min<int64_t>(ctx->num_sms, OTK_SAMPLE_TM_MIN_ROWS) &&
      sample_tm_fits(p0.vocab, dtype))
    return launch_sample_tm(ctx, p0, dtype, s);
#endif
  // lane-strided kernel; at <= 64 rows with twice the registers per thread (2 resident CTAs per SM: 16 rows
  // 8.4 vs 9.5 us, 64 rows 12.2 vs 13.9 us; slower from 128 rows, profiles/r01_sample_tuning_sweep_graph.txt)
  const bool bf = dtype == OTK_BF16;
  if (p0.num_rows <= 64)
    return bf ? launch_lane_strided<__nv_bfloat16, 2>(ctx, p0, s, 2) : launch_lane_strided<float, 2>(ctx, p0, s, 3);
  return bf ? launch_lane_strided<__nv_bfloat16, OTK_SAMPLE_MINB>(ctx, p0, s, 0)
            : launch_lane_strided<float, OTK_SAMPLE_MINB>(ctx, p0, s, 1);
}

}  // namespace otk
