// k_rows.cu — the fused vocab-row kernel behind otk_logprob_entropy_fwd (north_star (3)),
// otk_policy_loss_fwd_bwd (north_star (4)) and the vocab-sharded variants.
//
// One persistent CTA per SM (216 KB ring of 8 KB slots). A row is split across a thread-block
// cluster of `csize` CTAs (csize = 2 for bf16 V = 151936) so each CTA's column segment (148 KB)
// stays resident in shared memory between pass 1 (max / sum-exp / entropy) and pass 2
// (softmax - onehot, scaled): every logit is read from HBM once and every dlogit written once.
//   warp 0, lane 0  : producer — 1-D bulk TMA (cp.async.bulk) of 8 KB chunks into the ring,
//                     L2 evict_first (logits are read once), paced by per-slot empty mbarriers.
//   warps 1..8      : consumers — LDS.128, online max / sum 2^x / sum 2^x*x in fp32 (MUFU ex2),
//                     warp shuffle + CTA combine, cluster exchange of 16-byte row partials via DSMEM
//                     (st.async + mbarrier), loss terms in fp64 by one thread, pass 2 from SMEM with
//                     streaming 16-byte stores.
// Rows with loss mask 0 are never read: their dlogits are zero-filled (write-only).
// Reductions are in a fixed order, so results are deterministic and identical across the CTAs
// of a cluster (and across ranks under vocab sharding).
#include <cuda_bf16.h>

#include <cfloat>

#include "otk_internal.h"
#include "otk_ptx.cuh"

namespace otk {
using namespace ptx;

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Running (max, sum 2^(y-m), sum 2^(y-m)(y-m)) in log2 units: y = log2(e) * s * x.
struct Stat {
  float m, s, t;
};

// combine / finalize use explicitly rounded ops (__fmul_rn / __fadd_rn are never contracted into
// FMAs), so every template instantiation and every CTA produces bitwise-identical row statistics:
// the fwd pool's logp (3) equals the logp recomputed inside the loss (4), making the on-policy ratio
// exactly 1, and all ranks of a vocab shard agree.
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
  float L2;    // log2(e) * lse
  float logp;  // z_y - lse
  float H;     // entropy
  float lse;
};

__device__ __forceinline__ RowStats finalize(const Stat t, const float zy) {
  RowStats r;
  const float lg2S = lg2(t.s);
  r.L2 = __fadd_rn(t.m, lg2S);
  r.lse = __fmul_rn(r.L2, kLn2);
  r.logp = __fsub_rn(zy, r.lse);
  r.H = __fmul_rn(kLn2, __fsub_rn(lg2S, __fdiv_rn(t.t, t.s)));
  return r;
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
  __device__ static __forceinline__ float vmax(const uint4 v) {
    return fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)), fmaxf(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
  __device__ static __forceinline__ uint4 pack(const float (&g)[4]) {
    return make_uint4(__float_as_uint(g[0]), __float_as_uint(g[1]), __float_as_uint(g[2]), __float_as_uint(g[3]));
  }
  __device__ static __forceinline__ float load1(const void* base, int64_t i) {
    return reinterpret_cast<const float*>(base)[i];
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
  __device__ static __forceinline__ float vmax(const uint4 v) {
    const uint32_t m = bmax2(bmax2(v.x, v.y), bmax2(v.z, v.w));
    return fmaxf(bf_lo(m), bf_hi(m));
  }
  __device__ static __forceinline__ uint4 pack(const float (&g)[8]) {
    return make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]), pack_bf16x2(g[4], g[5]),
                      pack_bf16x2(g[6], g[7]));
  }
  __device__ static __forceinline__ float load1(const void* base, int64_t i) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  }
  __device__ static __forceinline__ void store1(void* base, int64_t i, float v) {
    reinterpret_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
  }
};

struct Smem {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t xbar[2];
  float4 xrecv[2][8];
  float4 wred[kConsumerWarps];
  float4 rowbc[2];
  float zy;
};
constexpr size_t kRingBytes = size_t(kSlots) * kChunkBytes;
constexpr size_t kSmemBytes = kRingBytes + sizeof(Smem);

template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_rows(const RowParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  Smem& S = *reinterpret_cast<Smem*>(smem + kRingBytes);

  using VT = Vec<T>;
  constexpr int EV = VT::EV;
  constexpr int CE = kChunkBytes / int(sizeof(T));                    // elements per chunk
  constexpr int NCT = 32 * kConsumerWarps;                             // consumer threads
  constexpr int VPT = kChunkBytes / 16 / NCT;                          // 16-B vectors per thread per chunk
  static_assert(VPT * NCT * 16 == kChunkBytes, "chunk must split evenly over consumers");
  constexpr bool kBwd = (MODE == kModeBwd || MODE == kModeBwdPartials);
  constexpr bool kPass1 = (MODE != kModeBwdPartials);
  constexpr bool kResident = (MODE == kModeBwd);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int csize = p.csize;
  const uint32_t crank = csize > 1 ? cluster_ctarank() : 0u;
  const int64_t group = blockIdx.x / csize;
  const int64_t ngroups = gridDim.x / csize;
  const int64_t c0 = int64_t(crank) * p.seg_elems;
  const int64_t c1 = min(p.vocab, c0 + int64_t(p.seg_elems));
  const int64_t segn = c1 > c0 ? c1 - c0 : 0;
  const uint32_t seg_bytes = uint32_t((segn * int64_t(sizeof(T)) + 15) & ~int64_t(15));
  const int nch = int((seg_bytes + kChunkBytes - 1) / kChunkBytes);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kConsumerWarps);
    }
    mbar_init(&S.xbar[0], 1);
    mbar_init(&S.xbar[1], 1);
    S.zy = 0.f;
    fence_mbar_init();
  }
  if (csize > 1)
    cluster_sync_all();
  else
    __syncthreads();

  if (warp == 0) {
    // ============================== producer ==============================
    if (lane == 0 && nch > 0) {
      const uint64_t pol = policy_evict_first();
      const char* base = reinterpret_cast<const char*>(p.logits) + c0 * int64_t(sizeof(T));
      const int64_t row_bytes = p.ld * int64_t(sizeof(T));
      uint32_t seq = 0;
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
        if (!(m && y >= 0 && int64_t(y) < p.vocab_total)) continue;
        const char* src = base + row * row_bytes;
        for (int c = 0; c < nch; ++c, ++seq) {
          const uint32_t slot = seq % kSlots, ph = (seq / kSlots) & 1u;
          mbar_wait(&S.empty[slot], ph ^ 1u);
          const uint32_t bytes = min(uint32_t(kChunkBytes), seg_bytes - uint32_t(c) * kChunkBytes);
          mbar_arrive_expect_tx(&S.full[slot], bytes);
          bulk_g2s(ring + size_t(slot) * kChunkBytes, src + size_t(c) * kChunkBytes, bytes, &S.full[slot], pol);
        }
      }
    }
    __syncwarp();
  } else {
    // ============================== consumers =============================
    const int ct = threadIdx.x - 32;
    const int cw = warp - 1;
    const float s2 = p.scale * kLog2e;
    double acc_L = 0.0, acc_clip = 0.0, acc_kl = 0.0, acc_H = 0.0, acc_n = 0.0;
    int64_t nl = 0;
    if (kBwd && ct == 0) nl = *p.n_loss;
    uint32_t seq = 0, q = 0;

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
      const bool in_range = y >= 0 && int64_t(y) < p.vocab_total;
      if (!(m && in_range)) {
        // ---------------- inactive row: never read ----------------
        if (m && ct == 0 && crank == 0) set_error(p.err, OTK_ERR_TARGET_RANGE);
        if (kBwd) {
          if (p.zero_masked) {
            char* drow = reinterpret_cast<char*>(p.dlogits) + row * p.ld * int64_t(sizeof(T));
            for (int64_t col = c0 + int64_t(ct) * EV; col < c1; col += int64_t(NCT) * EV) {
              if (col + EV <= c1) {
                stg_cs_v4(drow + col * int64_t(sizeof(T)), make_uint4(0, 0, 0, 0));
              } else {
                for (int64_t k = col; k < c1; ++k) VT::store1(drow, k, 0.f);
              }
            }
          }
          if (ct == 0 && crank == 0) {
            if (p.logp) p.logp[row] = 0.f;
            if (p.entropy) p.entropy[row] = 0.f;
          }
        } else if (ct == 0 && crank == 0) {
          if (MODE == kModeFwd) {
            p.logp[row] = 0.f;
            if (p.entropy) p.entropy[row] = 0.f;
            if (p.lse) p.lse[row] = 0.f;
          } else {
            p.partials_out[row] = make_float4(-INFINITY, 0.f, 0.f, 0.f);
          }
        }
        continue;
      }
      const int64_t yl = int64_t(y) - p.vocab_start;  // local target column (may lie outside this shard)

      // thread 0: side data for the loss, issued early (consumed after pass 1)
      int32_t rt = 0;
      float old_lp = 0.f, ref_lp = 0.f;
      if (kBwd && ct == 0) {
        rt = p.row_traj[row];
        old_lp = p.old_logp[row];
        if (p.ref_logp) ref_lp = p.ref_logp[row];
      }

      // ---------------- pass 1: online max / sum-exp / entropy numerator ----------------
      Stat st{-INFINITY, 0.f, 0.f};
      if (kPass1) {
        for (int c = 0; c < nch; ++c) {
          const uint32_t sq = seq + uint32_t(c);
          const uint32_t slot = sq % kSlots;
          mbar_wait(&S.full[slot], (sq / kSlots) & 1u);
          const uint8_t* buf = ring + size_t(slot) * kChunkBytes;
          const int64_t cbase = c0 + int64_t(c) * CE;
          uint4 v[VPT];
          float mx = -INFINITY;
#pragma unroll
          for (int k = 0; k < VPT; ++k) {
            const int vi = ct + k * NCT;
            const int64_t vcol = cbase + int64_t(vi) * EV;
            v[k] = *reinterpret_cast<const uint4*>(buf + size_t(vi) * 16);
            if (vcol + EV <= c1) {
              mx = fmaxf(mx, VT::vmax(v[k]));
            } else if (vcol < c1) {
              float x[EV];
              VT::unpack(v[k], x);
#pragma unroll
              for (int i = 0; i < EV; ++i)
                if (vcol + i < c1) mx = fmaxf(mx, x[i]);
            }
            if (uint64_t(yl - vcol) < uint64_t(EV) && yl < c1) S.zy = __fmul_rn(p.scale, VT::load1(buf, yl - cbase));
          }
          if (mx > -INFINITY) {
            const float mn = fmaxf(st.m, mx * s2);
            if (mn > st.m) {
              if (st.m != -INFINITY) {
                const float d = st.m - mn, f = ex2(d);
                st.t = f * fmaf(d, st.s, st.t);
                st.s *= f;
              }
              st.m = mn;
            }
            // chunk-local partial sums (short fp32 accumulation chains), then one add per chunk
            float cs = 0.f, ctt = 0.f;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
              const int64_t vcol = cbase + int64_t(ct + k * NCT) * EV;
              float x[EV];
              VT::unpack(v[k], x);
              if (vcol + EV <= c1) {
#pragma unroll
                for (int i = 0; i < EV; ++i) {
                  const float d = fmaxf(fmaf(x[i], s2, -st.m), -FLT_MAX);
                  const float e = ex2(d);
                  cs += e;
                  ctt = fmaf(e, d, ctt);
                }
              } else if (vcol < c1) {
#pragma unroll
                for (int i = 0; i < EV; ++i) {
                  if (vcol + i < c1) {
                    const float d = fmaxf(fmaf(x[i], s2, -st.m), -FLT_MAX);
                    const float e = ex2(d);
                    cs += e;
                    ctt = fmaf(e, d, ctt);
                  }
                }
              }
            }
            st.s += cs;
            st.t += ctt;
          }
          if (!kResident) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[slot]);
          }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          Stat o;
          o.m = __shfl_xor_sync(0xffffffffu, st.m, off);
          o.s = __shfl_xor_sync(0xffffffffu, st.s, off);
          o.t = __shfl_xor_sync(0xffffffffu, st.t, off);
          st = (lane & off) ? combine(o, st) : combine(st, o);
        }
        if (lane == 0) S.wred[cw] = make_float4(st.m, st.s, st.t, 0.f);
        named_bar_sync(1, NCT);
      }

      if (ct == 0) {
        Stat tot{-INFINITY, 0.f, 0.f};
        float zyt = 0.f;
        if (kPass1) {
          Stat r{S.wred[0].x, S.wred[0].y, S.wred[0].z};
#pragma unroll
          for (int w = 1; w < kConsumerWarps; ++w) r = combine(r, Stat{S.wred[w].x, S.wred[w].y, S.wred[w].z});
          const float zy = S.zy;
          S.zy = 0.f;
          if (csize > 1) {
            const uint32_t par = q & 1u;
            for (int dst = 0; dst < csize; ++dst) {
              if (dst == int(crank)) continue;
              st_async_f4(mapa(smem_u32(&S.xrecv[par][crank]), dst), r.m, r.s, r.t, zy,
                          mapa(smem_u32(&S.xbar[par]), dst));
            }
            mbar_arrive_expect_tx(&S.xbar[par], 16u * uint32_t(csize - 1));
            mbar_wait_cluster(&S.xbar[par], (q >> 1) & 1u);
            for (int k = 0; k < csize; ++k) {
              const float4 P = (k == int(crank)) ? make_float4(r.m, r.s, r.t, zy) : S.xrecv[par][k];
              tot = combine(tot, Stat{P.x, P.y, P.z});
              zyt += P.w;
            }
          } else {
            tot = r;
            zyt = zy;
          }
        } else {
          for (int k = 0; k < p.nshards; ++k) {
            const float4 P = p.partials_in[int64_t(k) * p.num_rows + row];
            tot = combine(tot, Stat{P.x, P.y, P.z});
            zyt += P.w;
          }
        }

        if (MODE == kModePartial) {
          if (crank == 0) p.partials_out[row] = make_float4(tot.m, tot.s, tot.t, zyt);
        } else {
          const RowStats rs = finalize(tot, zyt);
          if (MODE == kModeFwd) {
            if (crank == 0) {
              p.logp[row] = rs.logp;
              if (p.entropy) p.entropy[row] = rs.H;
              if (p.lse) p.lse[row] = rs.lse;
            }
          } else {
            // ---------------- loss terms (fp64, one thread) ----------------
            const double lp = double(rs.logp);
            const double A = p.adv[rt];
            const double C = double(p.clamp);
            const double draw = lp - double(old_lp);
            const double delta = fmin(fmax(draw, -C), C);
            const double r = exp(delta);
            const double lo = 1.0 - double(p.clip_low), hi = 1.0 + double(p.clip_high);
            const double rbar = fmin(fmax(r, lo), hi);
            const double pg = fmax(-A * r, -A * rbar);
            const bool clipped = (A > 0.0 && r > hi) || (A < 0.0 && r < lo);
            double G = (clipped || fabs(draw) > C) ? 0.0 : -A * r;
            double kl = 0.0;
            const double beta = double(p.kl_beta);
            if (beta != 0.0) {
              const double ref = double(ref_lp);
              double gk;
              if (p.kl_type == OTK_KL_K3) {
                const double dr = ref - lp;
                const double d = fmin(fmax(dr, -C), C);
                const double ed = exp(d);
                kl = ed - d - 1.0;
                gk = fabs(dr) > C ? 0.0 : 1.0 - ed;
              } else if (p.kl_type == OTK_KL_K1) {
                kl = lp - ref;
                gk = 1.0;
              } else {
                kl = 0.5 * (lp - ref) * (lp - ref);
                gk = lp - ref;
              }
              G += beta * gk;
            }
            const double L = pg + beta * kl;
            const double invN = nl > 0 ? 1.0 / double(nl) : 0.0;
            const float coef = float(-double(p.scale) * invN * G);
            if (crank == 0) {
              acc_L += L;
              acc_clip += clipped ? 1.0 : 0.0;
              acc_kl += kl;
              acc_H += double(rs.H);
              acc_n += 1.0;
              if (p.logp) p.logp[row] = rs.logp;
              if (p.entropy) p.entropy[row] = rs.H;
            }
            S.rowbc[q & 1u] = make_float4(rs.L2, coef, 0.f, 0.f);
          }
        }
      }

      if (kBwd) {
        // ---------------- pass 2: dlogits = coef * (p - onehot) ----------------
        named_bar_sync(1, NCT);
        const float4 bc = S.rowbc[q & 1u];
        const float L2 = bc.x, coef = bc.y;
        char* drow = reinterpret_cast<char*>(p.dlogits) + row * p.ld * int64_t(sizeof(T));
        for (int c = 0; c < nch; ++c) {
          const uint32_t sq = seq + uint32_t(c);
          const uint32_t slot = sq % kSlots;
          if (!kResident) mbar_wait(&S.full[slot], (sq / kSlots) & 1u);
          const uint8_t* buf = ring + size_t(slot) * kChunkBytes;
          const int64_t cbase = c0 + int64_t(c) * CE;
#pragma unroll
          for (int k = 0; k < VPT; ++k) {
            const int vi = ct + k * NCT;
            const int64_t vcol = cbase + int64_t(vi) * EV;
            if (vcol >= c1) continue;
            const uint4 v = *reinterpret_cast<const uint4*>(buf + size_t(vi) * 16);
            float x[EV], g[EV];
            VT::unpack(v, x);
#pragma unroll
            for (int i = 0; i < EV; ++i) g[i] = coef * ex2(fmaf(x[i], s2, -L2));
            if (uint64_t(yl - vcol) < uint64_t(EV)) {
#pragma unroll
              for (int i = 0; i < EV; ++i)
                if (vcol + i == yl) g[i] -= coef;
            }
            if (vcol + EV <= c1) {
              stg_cs_v4(drow + vcol * int64_t(sizeof(T)), VT::pack(g));
            } else {
#pragma unroll
              for (int i = 0; i < EV; ++i)
                if (vcol + i < c1) VT::store1(drow, vcol + i, g[i]);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.empty[slot]);
        }
      }
      seq += uint32_t(nch);
      ++q;
      if (!kBwd) named_bar_sync(1, NCT);  // S.wred / S.zy reuse guard for the next row
    }

    // ---------------- deterministic stats reduction (last CTA) ----------------
    if (kBwd && ct == 0) {
      double* part = p.cta_partials + size_t(blockIdx.x) * kStatSlots;
      part[0] = acc_L;
      part[1] = acc_clip;
      part[2] = acc_kl;
      part[3] = acc_H;
      part[4] = acc_n;
      __threadfence();
      const unsigned int t = atomicAdd(p.ticket, 1u);
      if (t == gridDim.x - 1) {
        __threadfence();
        double tot[5] = {0, 0, 0, 0, 0};
        for (unsigned int b = 0; b < gridDim.x; ++b) {
          const volatile double* q2 = p.cta_partials + size_t(b) * kStatSlots;
          for (int k = 0; k < 5; ++k) tot[k] += q2[k];
        }
        const double invN = nl > 0 ? 1.0 / double(nl) : 0.0;
        otk_loss_stats* o = p.stats;
        if (p.accumulate) {
          o->loss += tot[0] * invN;
          o->n_clipped += tot[1];
          o->kl_sum += tot[2];
          o->entropy_sum += tot[3];
          o->n_tokens += tot[4];
        } else {
          o->loss = tot[0] * invN;
          o->n_clipped = tot[1];
          o->kl_sum = tot[2];
          o->entropy_sum = tot[3];
          o->n_tokens = tot[4];
        }
        *p.ticket = 0u;
      }
    }
  }

  if (csize > 1) cluster_sync_all();
}

// ---- vocab-shard combine (otk_logprob_entropy_combine): same combine / finalize as k_rows ----------
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
    Stat tot{-INFINITY, 0.f, 0.f};
    float zyt = 0.f;
    for (int k = 0; k < nshards; ++k) {
      const float4 P = partials[int64_t(k) * num_rows + row];
      tot = combine(tot, Stat{P.x, P.y, P.z});
      zyt += P.w;
    }
    const RowStats rs = finalize(tot, zyt);
    logp[row] = rs.logp;
    if (entropy) entropy[row] = rs.H;
    if (lse) lse[row] = rs.lse;
  }
}

// ---- launchers -------------------------------------------------------------------------------------
template <typename T, int MODE>
static cudaError_t launch_rows_t(const otk_ctx* ctx, const RowParams& p, cudaStream_t s, int* grid_out) {
  auto kern = k_rows<T, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes));
  if (e != cudaSuccess) return e;
  int64_t groups = ctx->num_sms / p.csize;
  if (groups > p.num_rows) groups = p.num_rows;
  if (groups < 1) groups = 1;
  const int grid = int(groups * p.csize);
  if (grid > kMaxCtas) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.csize > 1 ? 1 : 0;
  if (grid_out) *grid_out = grid;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_rows(const otk_ctx* ctx, RowMode mode, otk_dtype dtype, const RowParams& p, cudaStream_t s,
                        int* grid_out) {
  if (dtype == OTK_BF16) {
    switch (mode) {
      case kModeFwd: return launch_rows_t<__nv_bfloat16, kModeFwd>(ctx, p, s, grid_out);
      case kModePartial: return launch_rows_t<__nv_bfloat16, kModePartial>(ctx, p, s, grid_out);
      case kModeBwd: return launch_rows_t<__nv_bfloat16, kModeBwd>(ctx, p, s, grid_out);
      case kModeBwdPartials: return launch_rows_t<__nv_bfloat16, kModeBwdPartials>(ctx, p, s, grid_out);
    }
  } else {
    switch (mode) {
      case kModeFwd: return launch_rows_t<float, kModeFwd>(ctx, p, s, grid_out);
      case kModePartial: return launch_rows_t<float, kModePartial>(ctx, p, s, grid_out);
      case kModeBwd: return launch_rows_t<float, kModeBwd>(ctx, p, s, grid_out);
      case kModeBwdPartials: return launch_rows_t<float, kModeBwdPartials>(ctx, p, s, grid_out);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_combine(const otk_ctx* ctx, int64_t num_rows, int nshards, const float4* partials,
                           const uint8_t* row_mask, float* logp, float* entropy, float* lse, cudaStream_t s) {
  int64_t blocks = (num_rows + 255) / 256;
  if (blocks > int64_t(ctx->num_sms) * 8) blocks = int64_t(ctx->num_sms) * 8;
  if (blocks < 1) blocks = 1;
  k_combine<<<int(blocks), 256, 0, s>>>(num_rows, nshards, partials, row_mask, logp, entropy, lse);
  return cudaGetLastError();
}

}  // namespace otk
