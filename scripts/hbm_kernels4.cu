// HBM store-path probes (round 2): how the write half of the loss kernel's traffic should be issued. Every kernel is
// a grid-stride stream over 16-byte vectors with 4 operations in flight per thread.
//   store variant 0: st.global.cs.v4 (evict-first, what the row kernels use), 1: st.global.v4 (plain),
//                 2: st.global.v8 (256-bit, plain), 3: st.global.L1::no_allocate.v4
#include <cuda_runtime.h>
#include <cstdint>
template <int SV>
__device__ __forceinline__ void st4(uint4* p, uint4 v, uint4 w) {  // stores v at p and w at p + 1 (SV 2: one 256-bit)
  if constexpr (SV == 0) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p + 1), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
  } else if constexpr (SV == 1) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p + 1), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
  } else if constexpr (SV == 2) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
  } else {
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p + 1), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
  }
}
// coalesced 128-bit forms: a warp instruction covers 512 contiguous bytes (lane-consecutive vectors); the second
// vector of a thread sits one grid-width further
template <int SV>
__device__ __forceinline__ void st1(uint4* p, uint4 v) {
  if constexpr (SV == 0)
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <int SV>
__global__ void k_write_c(uint4* y, size_t n16) {
  const size_t g = size_t(gridDim.x) * blockDim.x;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += 2 * g) {
    st1<SV>(y + i, z);
    if (i + g < n16) st1<SV>(y + i + g, z);
  }
}
template <int SV>
__global__ void k_rows_c(const uint4* x, uint4* y, size_t nrows, size_t row16, const uint8_t* copy_row) {
  for (size_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const uint4* xs = x + r * row16;
    uint4* ys = y + r * row16;
    const uint4 z = make_uint4(0, 0, 0, 0);
    const size_t st = blockDim.x;
    if (!copy_row[r]) {
      for (size_t i = threadIdx.x; i < row16; i += st) st1<SV>(ys + i, z);
    } else {
      size_t i = threadIdx.x;
      for (; i + 3 * st < row16; i += 4 * st) {
        const uint4 a = __ldg(xs + i), b = __ldg(xs + i + st), c = __ldg(xs + i + 2 * st), d = __ldg(xs + i + 3 * st);
        st1<SV>(ys + i, a);
        st1<SV>(ys + i + st, b);
        st1<SV>(ys + i + 2 * st, c);
        st1<SV>(ys + i + 3 * st, d);
      }
      for (; i < row16; i += st) st1<SV>(ys + i, __ldg(xs + i));
    }
  }
}
// pure write: thread t of the grid writes pairs of vectors 2t, 2t+1 (+ 2 stride k)
template <int SV>
__global__ void k_write(uint4* y, size_t n16) {
  const size_t stride = size_t(gridDim.x) * blockDim.x * 2;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < n16; i += stride) st4<SV>(y + i, z, z);
}
// copy: pairs of vectors, 2 pairs in flight
template <int SV>
__global__ void k_copy(const uint4* x, uint4* y, size_t n16) {
  const size_t stride = size_t(gridDim.x) * blockDim.x * 2;
  size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  for (; i + stride < n16; i += 2 * stride) {
    const uint4 a = __ldg(x + i), b = __ldg(x + i + 1), c = __ldg(x + i + stride), d = __ldg(x + i + stride + 1);
    st4<SV>(y + i, a, b);
    st4<SV>(y + i + stride, c, d);
  }
  for (; i < n16; i += stride) st4<SV>(y + i, __ldg(x + i), __ldg(x + i + 1));
}
// the loss kernel's row mix: rows of row16 vectors, one CTA per row at a time; a row is copied (trainable: read +
// write) when its bit in the pattern is set, else zero-filled (write only)
template <int SV>
__global__ void k_rows(const uint4* x, uint4* y, size_t nrows, size_t row16, const uint8_t* copy_row) {
  for (size_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const uint4* xs = x + r * row16;
    uint4* ys = y + r * row16;
    const uint4 z = make_uint4(0, 0, 0, 0);
    if (!copy_row[r]) {
      for (size_t i = threadIdx.x * 2; i < row16; i += blockDim.x * 2) st4<SV>(ys + i, z, z);
    } else {
      size_t i = threadIdx.x * 2;
      const size_t st = blockDim.x * 2;
      for (; i + st < row16; i += 2 * st) {
        const uint4 a = __ldg(xs + i), b = __ldg(xs + i + 1), c = __ldg(xs + i + st), d = __ldg(xs + i + st + 1);
        st4<SV>(ys + i, a, b);
        st4<SV>(ys + i + st, c, d);
      }
      for (; i < row16; i += st) st4<SV>(ys + i, __ldg(xs + i), __ldg(xs + i + 1));
    }
  }
}
extern "C" {
int probe4_write(void* y, size_t nbytes, int grid, int sv, cudaStream_t s) {
  const size_t n = nbytes / 16;
  if (sv == 0) k_write<0><<<grid, 512, 0, s>>>((uint4*)y, n);
  if (sv == 1) k_write<1><<<grid, 512, 0, s>>>((uint4*)y, n);
  if (sv == 2) k_write<2><<<grid, 512, 0, s>>>((uint4*)y, n);
  if (sv == 3) k_write<3><<<grid, 512, 0, s>>>((uint4*)y, n);
  return cudaGetLastError();
}
int probe4_copy(const void* x, void* y, size_t nbytes, int grid, int sv, cudaStream_t s) {
  const size_t n = nbytes / 16;
  if (sv == 0) k_copy<0><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, n);
  if (sv == 1) k_copy<1><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, n);
  if (sv == 2) k_copy<2><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, n);
  if (sv == 3) k_copy<3><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, n);
  return cudaGetLastError();
}
int probe4_write_c(void* y, size_t nbytes, int grid, int sv, cudaStream_t s) {
  if (sv == 0) k_write_c<0><<<grid, 512, 0, s>>>((uint4*)y, nbytes / 16);
  else k_write_c<1><<<grid, 512, 0, s>>>((uint4*)y, nbytes / 16);
  return cudaGetLastError();
}
int probe4_rows_c(const void* x, void* y, size_t nrows, size_t row_bytes, const void* copy_row, int grid, int sv,
                  cudaStream_t s) {
  if (sv == 0) k_rows_c<0><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, nrows, row_bytes / 16, (const uint8_t*)copy_row);
  else k_rows_c<1><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, nrows, row_bytes / 16, (const uint8_t*)copy_row);
  return cudaGetLastError();
}
int probe4_rows(const void* x, void* y, size_t nrows, size_t row_bytes, const void* copy_row, int grid, int sv,
                cudaStream_t s) {
  const size_t r16 = row_bytes / 16;
  if (sv == 0) k_rows<0><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, nrows, r16, (const uint8_t*)copy_row);
  if (sv == 1) k_rows<1><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, nrows, r16, (const uint8_t*)copy_row);
  if (sv == 2) k_rows<2><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, nrows, r16, (const uint8_t*)copy_row);
  if (sv == 3) k_rows<3><<<grid, 512, 0, s>>>((const uint4*)x, (uint4*)y, nrows, r16, (const uint8_t*)copy_row);
  return cudaGetLastError();
}
}
