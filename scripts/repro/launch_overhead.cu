// Experiment: per-launch time of an (almost) empty kernel replayed from a CUDA graph, 128 CTAs of 512 threads with
// 40 KB of dynamic shared memory, without and with 8-CTA clusters (the decode sampler's shape).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/lo scripts/repro/launch_overhead.cu && /tmp/lo
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && sm[1] == 12345) out[blockIdx.x] = 1;
}
int main() {
  int* out;
  cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int cl : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(128);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 40960;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = cl > 1 ? 1 : 0;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k, out);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster %d: %.2f us per launch (%s)\n", cl, ms * 1e3 / 100, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
