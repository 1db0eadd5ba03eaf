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
extern "C" {
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
