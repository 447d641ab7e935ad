// Probe (not product): write-only streaming bandwidth on B200 (the merge's dense-G fill):
// cudaMemsetAsync and a float4 store kernel (plain / .cs) over 1.56e9 floats.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/write_probe tools/write_probe.cu && tools/write_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fill(float4* __restrict__ o, size_t n4) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n4) o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__global__ void fill_cs(float4* __restrict__ o, size_t n4) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n4) __stcs(o + i, make_float4(0.f, 0.f, 0.f, 0.f));
}
int main() {
  const size_t n = 1557611200ull;
  float* o;
  cudaMalloc(&o, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    for (int mode = 0; mode < 3; ++mode) {
      cudaEventRecord(e0);
      if (mode == 0) cudaMemsetAsync(o, 0, n * 4);
      else if (mode == 1) fill<<<(unsigned)((n / 4 + 255) / 256), 256>>>((float4*)o, n / 4);
      else fill_cs<<<(unsigned)((n / 4 + 255) / 256), 256>>>((float4*)o, n / 4);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* nm[3] = {"cudaMemsetAsync", "float4 stores", "float4 .cs stores"};
      if (rep == 2) printf("%-18s %.3f ms  %.0f GB/s\n", nm[mode], ms, 4.0 * n / ms / 1e6);
    }
  }
  return 0;
}
