// Roofline probe (not part of the product): achievable HBM bandwidth on this GPU for the access
// patterns of the LowDiff kernels, timed with CUDA events.
//   copy   : dst = src                 (1 read + 1 write stream)  -- the MEASURED_PEAKS pattern
//   ef_add : r = r + g                 (2 read + 1 write streams) -- the scan's traffic
//   read2  : sum(r) + sum(g)           (2 read streams)
// usage: stream_probe [n_floats]   (default 1.56e9, GPT-2 XL)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void copy_k(const float4* __restrict__ s, float4* __restrict__ d, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) d[i] = s[i];
}
__global__ void ef_add_k(const float4* __restrict__ g, float4* __restrict__ r, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 a = g[i], b = r[i];
    r[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
}
template <int U>
__global__ void ef_add_unroll_k(const float4* __restrict__ g, float4* __restrict__ r, size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * stride < n4) { a[u] = g[i0 + u * stride]; b[u] = r[i0 + u * stride]; }
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * stride < n4) r[i0 + u * stride] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
  }
}
__global__ void read2_k(const float4* __restrict__ g, const float4* __restrict__ r, size_t n4, float* out) {
  float s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 a = g[i], b = r[i];
    s += a.x + b.y + a.z + b.w;
  }
  if (s == 123.f) *out = s;
}

int main(int argc, char** argv) {
  size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 1557611200ull;
  size_t n4 = n / 4;
  float *g, *r, *o;
  cudaMalloc(&g, n4 * 16); cudaMalloc(&r, n4 * 16); cudaMalloc(&o, 4);
  cudaMemset(g, 0, n4 * 16); cudaMemset(r, 0, n4 * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 2; ++i) launch();
    cudaEventRecord(a);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    printf("%-28s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  for (int bs : {256, 512, 1024}) for (int w : {1, 2, 4, 8}) {
    int grid = sms * w * (1024 / bs);
    char nm[64];
    snprintf(nm, 64, "copy b%d g%d", bs, grid); run(nm, 8.0 * n, [&] { copy_k<<<grid, bs>>>((float4*)g, (float4*)r, n4); });
    snprintf(nm, 64, "ef_add b%d g%d", bs, grid); run(nm, 12.0 * n, [&] { ef_add_k<<<grid, bs>>>((float4*)g, (float4*)r, n4); });
    snprintf(nm, 64, "ef_add_u4 b%d g%d", bs, grid); run(nm, 12.0 * n, [&] { ef_add_unroll_k<4><<<grid, bs>>>((float4*)g, (float4*)r, n4); });
    snprintf(nm, 64, "read2 b%d g%d", bs, grid); run(nm, 8.0 * n, [&] { read2_k<<<grid, bs>>>((float4*)g, (float4*)r, n4, o); });
  }
  int big = (int)((n4 + 255) / 256);
  run("ef_add b256 full-grid", 12.0 * n, [&] { ef_add_k<<<big, 256>>>((float4*)g, (float4*)r, n4); });
  run("copy b256 full-grid", 8.0 * n, [&] { copy_k<<<big, 256>>>((float4*)g, (float4*)r, n4); });
  return 0;
}
