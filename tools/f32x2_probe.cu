// Probe (not part of the product): are the sm_100a paired fp32 ops bit-identical to scalar ones?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }
__device__ uint64_t mix(uint64_t z) { z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }
__global__ void k(unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (1ull << 26); i += gridDim.x * (uint64_t)blockDim.x) {
    uint64_t h = mix(i), h2 = mix(h);
    float a0 = __uint_as_float((uint32_t)h & 0x3FFFFFFF), a1 = __uint_as_float((uint32_t)(h >> 32) & 0x3FFFFFFF);
    float b0 = __uint_as_float((uint32_t)h2 & 0x3FFFFFFF), b1 = __uint_as_float((uint32_t)(h2 >> 32) & 0x3FFFFFFF);
    float c0 = -a0 * b0 * 0.999f, c1 = -a1 * b1 * 1.001f;
    u64 A = pk(a0, a1), Bv = pk(b0, b1), Cv = pk(c0, c1), r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(A), "l"(Bv), "l"(Cv));
    if (__float_as_uint(lo(r)) != __float_as_uint(__fmaf_rn(a0, b0, c0))) atomicAdd(&bad[0], 1ull);
    if (__float_as_uint(hi(r)) != __float_as_uint(__fmaf_rn(a1, b1, c1))) atomicAdd(&bad[1], 1ull);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(Bv));
    if (__float_as_uint(lo(r)) != __float_as_uint(__fmul_rn(a0, b0))) atomicAdd(&bad[2], 1ull);
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(A), "l"(Cv));
    if (__float_as_uint(lo(r)) != __float_as_uint(__fadd_rn(a0, c0))) atomicAdd(&bad[3], 1ull);
  }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 32); cudaMemset(d, 0, 32);
  k<<<1184, 256>>>(d); unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("fma lo %llu hi %llu  mul %llu  add %llu  (of %llu)\n", h[0], h[1], h[2], h[3], 1ull << 26);
}
