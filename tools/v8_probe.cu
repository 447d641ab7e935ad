// Probe (not product): r = r + g streaming with 128-bit vs 256-bit (ld/st.global.v8.f32) accesses,
// full grids, 1.56e9 floats (the GPT-2 XL gradient), B200.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/v8_probe tools/v8_probe.cu && tools/v8_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void add4(const float4* __restrict__ g, float4* __restrict__ r, size_t n4) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n4) {
    float4 a = __ldcs(g + i), b = __ldcs(r + i);
    __stcs(r + i, make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w));
  }
}
__device__ __forceinline__ void ld8(const float* p, float* x) {
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
               : "l"(p));
}
__device__ __forceinline__ void st8(float* p, const float* x) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(x[0]), "f"(x[1]), "f"(x[2]),
               "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7]));
}
__global__ void add8(const float* __restrict__ g, float* __restrict__ r, size_t n8) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n8) {
    float a[8], b[8];
    ld8(g + 8 * i, a);
    ld8(r + 8 * i, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += b[k];
    st8(r + 8 * i, a);
  }
}
int main() {
  const size_t n = 1557611200ull / 8 * 8;
  float *g, *r;
  cudaMalloc(&g, n * 4);
  cudaMalloc(&r, n * 4);
  cudaMemset(g, 0, n * 4);
  cudaMemset(r, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    for (int mode = 0; mode < 4; ++mode) {
      const int th = (mode & 1) ? 256 : 128;
      cudaEventRecord(e0);
      if (mode < 2) add4<<<(unsigned)((n / 4 + th - 1) / th), th>>>((const float4*)g, (float4*)r, n / 4);
      else add8<<<(unsigned)((n / 8 + th - 1) / th), th>>>(g, r, n / 8);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("%s %d threads: %.3f ms  %.0f GB/s\n", mode < 2 ? "128-bit" : "256-bit", th, ms, 12.0 * n / ms / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
