// Minimal reproducer for the racecheck report on the loss kernel's TMA ring (DESIGN.md §6 "Sanitizers"):
// the k_rows_tm producer / consumer protocol and nothing else. One producer thread fills a 2-slot shared-memory
// ring with 1-D bulk TMA (cp.async.bulk ... mbarrier::complete_tx); a consumer warp waits on the slot's FULL
// mbarrier phase, reads the slot, and releases it by arriving on its EMPTY mbarrier; the producer refills a slot
// only after that phase completed. The mbarrier phases order every bulk write after the previous reads of the
// slot, so the program is race-free (and its checksum is exact); a racecheck hazard reported here is the tool not
// modelling complete_tx / mbarrier ordering of the async proxy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2601_07376_b200/csrc -o /tmp/rr scripts/repro/racecheck_tma_ring.cu
//   compute-sanitizer --tool racecheck /tmp/rr
#include <cstdio>
#include <cstdint>
#include "otk_ptx.cuh"
using namespace otk::ptx;

constexpr int kSlots = 2, kChunk = 4096, kChunks = 16;

__global__ void ring(const uint4* src, unsigned long long* out) {
  __shared__ __align__(128) uint8_t buf[kSlots][kChunk];
  __shared__ uint64_t full[kSlots], empty[kSlots];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // producer
    uint32_t ph = 0;
    for (int c = 0; c < kChunks; ++c) {
      const int s = c % kSlots;
      mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], kChunk);
      bulk_g2s(buf[s], reinterpret_cast<const uint8_t*>(src) + size_t(c) * kChunk, kChunk, &full[s],
               policy_evict_first());
      if (s == kSlots - 1) ph ^= 1u;
    }
  } else if (threadIdx.x >= 32) {  // consumer warp
    const int lane = threadIdx.x - 32;
    uint32_t ph = 0;
    unsigned long long acc = 0;
    for (int c = 0; c < kChunks; ++c) {
      const int s = c % kSlots;
      mbar_wait(&full[s], ph);
      for (int i = lane; i < kChunk / 16; i += 32) {
        const uint4 v = reinterpret_cast<const uint4*>(buf[s])[i];
        acc += v.x + v.y + v.z + v.w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (s == kSlots - 1) ph ^= 1u;
    }
    atomicAdd(out, acc);
  }
}

int main() {
  const size_t n = size_t(kChunks) * kChunk / 16;
  uint4* src;
  unsigned long long* out;
  cudaMalloc(&src, n * 16);
  cudaMalloc(&out, 8);
  cudaMemset(out, 0, 8);
  uint4* h = new uint4[n];
  unsigned long long want = 0;
  for (size_t i = 0; i < n; ++i) {
    h[i] = make_uint4(unsigned(i), unsigned(3 * i), 7u, unsigned(i >> 3));
    want += h[i].x + h[i].y + h[i].z + h[i].w;
  }
  cudaMemcpy(src, h, n * 16, cudaMemcpyHostToDevice);
  ring<<<1, 64>>>(src, out);
  unsigned long long got = 0;
  cudaMemcpy(&got, out, 8, cudaMemcpyDeviceToHost);
  printf("checksum %s (%llu vs %llu), %s\n", got == want ? "exact" : "WRONG", got, want,
         cudaGetErrorString(cudaGetLastError()));
  return got == want ? 0 : 1;
}
