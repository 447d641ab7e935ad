// Probe (not product): how much does a concurrent device->host transfer slow an HBM-streaming kernel,
// for the copy engine (cudaMemcpyAsync) versus an SM-driven zero-copy store kernel on few CTAs?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/d2h_probe tools/d2h_probe.cu && tools/d2h_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stream_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
}
// zero-copy D2H: 128-bit loads from HBM, 128-bit stores into mapped pinned host memory
__global__ void zc_kernel(const float4* __restrict__ a, float4* __restrict__ h, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    h[i] = __ldcs(a + i);
}

int main() {
  const size_t n = 1557611200ull / 4 * 4, n4 = n / 4, chunk4 = (n4 / 16);
  float *a, *b, *g, *h, *hd;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&g, n * 4);
  cudaMemset(a, 0, n * 4); cudaMemset(g, 0, n * 4);
  cudaHostAlloc(&h, n * 4, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 16;
  auto hbm = [&](cudaStream_t s) {
    for (int r = 0; r < reps; ++r) stream_kernel<<<sms * 8, 512, 0, s>>>((const float4*)a, (float4*)b, chunk4 * 4);
  };
  for (int mode = 0; mode < 6; ++mode) {
    for (int it = 0; it < 2; ++it) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      if (mode == 1) cudaMemcpyAsync(h, g, n * 4, cudaMemcpyDeviceToHost, s2);
      if (mode >= 2) {
        const int ctas[4] = {4, 16, 64, 148};
        zc_kernel<<<ctas[mode - 2], 512, 0, s2>>>((const float4*)g, (float4*)hd, n4);
      }
      hbm(s1);
      cudaEventRecord(e1, s1);
      cudaEventRecord(e2, s2);
      cudaDeviceSynchronize();
      float t1, t2;
      cudaEventElapsedTime(&t1, e0, e1);
      cudaEventElapsedTime(&t2, e0, e2);
      if (it) {
        const char* names[6] = {"alone", "copy engine", "zero-copy 4 CTAs", "zero-copy 16 CTAs", "zero-copy 64 CTAs",
                                "zero-copy 148 CTAs"};
        printf("%-20s hbm kernels %8.2f ms (%.0f GB/s)   d2h %8.2f ms (%.1f GB/s)\n", names[mode], t1,
               reps * 8.0 * chunk4 * 16 / t1 / 1e6, mode ? t2 : 0.f, mode ? n * 4 / t2 / 1e6 : 0.0);
      }
    }
  }
  // many short kernels (a backward pass's granularity): 8M-float pieces, 20 per piece, on a
  // non-blocking stream and on the legacy default stream, with and without the copy-engine D2H
  const size_t piece4 = (8u << 20) / 4;
  const size_t npieces = n4 / piece4;
  for (int mode = 0; mode < 8; ++mode) {
    cudaStream_t sk = (mode & 2) ? (cudaStream_t)0 : s1;
    const int zc = mode >= 4 ? (mode == 4 ? 2 : mode == 5 ? 4 : mode == 6 ? 8 : 16) : 0;
    if (zc) sk = s1;
    for (int it = 0; it < 2; ++it) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, sk);
      cudaStreamWaitEvent(s2, e0, 0);
      if (zc) zc_kernel<<<zc, 512, 0, s2>>>((const float4*)g, (float4*)hd, n4);
      else if (mode & 1) cudaMemcpyAsync(h, g, n * 4, cudaMemcpyDeviceToHost, s2);
      for (size_t p = 0; p < npieces; ++p)
        for (int r = 0; r < 20; ++r)
          stream_kernel<<<sms * 8, 512, 0, sk>>>((const float4*)g + p * piece4, (float4*)b, piece4);
      cudaEventRecord(e1, sk);
      cudaEventRecord(e2, s2);
      cudaDeviceSynchronize();
      float t1, t2;
      cudaEventElapsedTime(&t1, e0, e1);
      cudaEventElapsedTime(&t2, e0, e2);
      if (it && zc) printf("short kernels (%zu x 20), with zero-copy d2h on %d CTAs: %8.2f ms (d2h %.2f ms)\n",
                           npieces, zc, t1, t2);
      else if (it) printf("short kernels (%zu x 20) on %s stream, %s: %8.2f ms (d2h %.2f ms)\n", npieces,
                     (mode & 2) ? "legacy" : "non-blocking", (mode & 1) ? "with copy-engine d2h" : "alone", t1,
                     (mode & 1) ? t2 : 0.f);
    }
  }
  // the d2h alone
  for (int mode = 1; mode < 4; ++mode) {
    cudaDeviceSynchronize();
    cudaEventRecord(e0, s2);
    if (mode == 1) cudaMemcpyAsync(h, g, n * 4, cudaMemcpyDeviceToHost, s2);
    else zc_kernel<<<mode == 2 ? 16 : 148, 512, 0, s2>>>((const float4*)g, (float4*)hd, n4);
    cudaEventRecord(e2, s2);
    cudaDeviceSynchronize();
    float t2;
    cudaEventElapsedTime(&t2, e0, e2);
    printf("d2h alone mode %d: %.2f ms (%.1f GB/s)\n", mode, t2, n * 4 / t2 / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
