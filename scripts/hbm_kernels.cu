// Write / mixed-traffic HBM probes (reference points for DESIGN.md §6; not part of the product).
#include <cuda_runtime.h>
#include <cstdint>
__global__ void k_write_stg(uint4* p, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %1, %1, %1};" ::"l"(p + i), "r"(0) : "memory");
}
__global__ void k_write_stg_plain(uint4* p, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}
__global__ void k_write_bulk(char* p, size_t nbytes, uint32_t chunk) {
  extern __shared__ __align__(128) uint4 z[];
  for (int i = threadIdx.x; i < int(chunk / 16); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(z));
    for (size_t off = size_t(blockIdx.x) * chunk; off < nbytes; off += size_t(gridDim.x) * chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(s), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void k_mix12(const uint4* x, uint4* y, uint4* z, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    uint4 v = x[i];
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(y + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %1, %1, %1};" ::"l"(z + i), "r"(0) : "memory");
  }
}
// read-only: 8 independent 16-byte loads in flight per thread, XOR-folded, one word written per thread
__global__ void k_read(const uint4* x, size_t n16, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(x + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n16; i += stride) { uint4 v = __ldg(x + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// read-only through 1-D bulk TMA into a shared-memory ring (the row kernels' load path)
__global__ void k_read_bulk(const char* x, size_t nbytes, uint32_t chunk, unsigned* out) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) unsigned long long bar[8];
  const int slots = 8;
  if (threadIdx.x == 0) {
    for (int k = 0; k < slots; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    size_t n = 0;
    for (size_t off = size_t(blockIdx.x) * chunk; off + chunk <= nbytes; off += size_t(gridDim.x) * chunk, ++n) {
      const int s = int(n % slots);
      const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
      if (n >= (size_t)slots) {  // wait for this slot's previous transfer (no consumer: pure read bandwidth)
        unsigned ok = 0;
        while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(b), "r"(ph[s]) : "memory");
        ph[s] ^= 1u;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                   "r"((unsigned)__cvta_generic_to_shared(ring + size_t(s) * chunk)), "l"(x + off), "r"(chunk), "r"(b) : "memory");
    }
    for (int s = 0; s < slots; ++s) {
      if (n > (size_t)s) {
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned ok = 0;
        while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(b), "r"(ph[s]) : "memory");
      }
    }
    out[blockIdx.x] = ring[0];
  }
}
extern "C" {
int probe_read(const void* x, size_t nbytes, int grid, void* out, cudaStream_t s) {
  k_read<<<grid, 512, 0, s>>>((const uint4*)x, nbytes / 16, (unsigned*)out);
  return cudaGetLastError();
}
int probe_read_bulk(const void* x, size_t nbytes, int grid, unsigned chunk, void* out, cudaStream_t s) {
  cudaFuncSetAttribute(k_read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * chunk);
  k_read_bulk<<<grid, 32, 8 * chunk, s>>>((const char*)x, nbytes, chunk, (unsigned*)out);
  return cudaGetLastError();
}
int probe_write_stg(void* p, size_t nbytes, int grid, int plain, cudaStream_t s) {
  if (plain) k_write_stg_plain<<<grid, 512, 0, s>>>((uint4*)p, nbytes / 16);
  else k_write_stg<<<grid, 512, 0, s>>>((uint4*)p, nbytes / 16);
  return cudaGetLastError();
}
int probe_write_bulk(void* p, size_t nbytes, int grid, unsigned chunk, cudaStream_t s) {
  cudaFuncSetAttribute(k_write_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
  k_write_bulk<<<grid, 128, chunk, s>>>((char*)p, nbytes, chunk);
  return cudaGetLastError();
}
int probe_memset(void* p, size_t nbytes, cudaStream_t s) { return cudaMemsetAsync(p, 0, nbytes, s); }
int probe_mix12(const void* x, void* y, void* z, size_t nbytes, int grid, cudaStream_t s) {
  k_mix12<<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, (uint4*)z, nbytes / 16);
  return cudaGetLastError();
}
}

// ---- round-1 follow-up probes: the K4 traffic mix with more loads in flight --------------------------------
// 1 read : 2 writes, 4 independent 16-byte loads in flight per thread before the 8 stores
__global__ void k_mix12_u4(const uint4* x, uint4* y, uint4* z, size_t n16) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(x + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(y + i + k * stride), "r"(v[k].x), "r"(v[k].y),
                   "r"(v[k].z), "r"(v[k].w) : "memory");
      asm volatile("st.global.cs.v4.b32 [%0], {%1, %1, %1, %1};" ::"l"(z + i + k * stride), "r"(0) : "memory");
    }
  }
  for (; i < n16; i += stride) {
    uint4 v = __ldg(x + i);
    y[i] = v;
    z[i] = make_uint4(0, 0, 0, 0);
  }
}
// row-structured like the loss kernel: rows of `row16` vectors; even rows copied x -> y (read + write), odd rows
// zero-filled in y (write only); one CTA per row at a time, 4 loads in flight per thread
__global__ void k_mix_rows(const uint4* x, uint4* y, size_t nrows, size_t row16, int mode) {
  for (size_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const uint4* xs = x + r * row16;
    uint4* ys = y + r * row16;
    const bool zero_row = mode == 0 ? (r & 1) : mode == 2;   // 0: alternate, 1: all copy, 2: all zero
    if (zero_row) {
      for (size_t i = threadIdx.x; i < row16; i += blockDim.x)
        asm volatile("st.global.cs.v4.b32 [%0], {%1, %1, %1, %1};" ::"l"(ys + i), "r"(0) : "memory");
    } else {
      size_t i = threadIdx.x;
      for (; i + 3 * blockDim.x < row16; i += 4 * blockDim.x) {
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldg(xs + i + k * blockDim.x);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(ys + i + k * blockDim.x), "r"(v[k].x),
                       "r"(v[k].y), "r"(v[k].z), "r"(v[k].w) : "memory");
      }
      for (; i < row16; i += blockDim.x) ys[i] = __ldg(xs + i);
    }
  }
}
extern "C" {
int probe_mix12_u4(const void* x, void* y, void* z, size_t nbytes, int grid, cudaStream_t s) {
  k_mix12_u4<<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, (uint4*)z, nbytes / 16);
  return cudaGetLastError();
}
int probe_mix_rows(const void* x, void* y, size_t nbytes, size_t row_bytes, int grid, int threads, int mode,
                   cudaStream_t s) {
  k_mix_rows<<<grid, threads, 0, s>>>((const uint4*)x, (uint4*)y, nbytes / row_bytes, row_bytes / 16, mode);
  return cudaGetLastError();
}
}
