// Roofline probe 2 (not part of the product): which parts of the scan cost bandwidth.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>

template <int MODE>   // 0 plain, 1 cs hints
__global__ void add1(const float4* __restrict__ g, float4* __restrict__ r, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 a = MODE ? __ldcs(g + i) : g[i], b = MODE ? __ldcs(r + i) : r[i];
  float4 c = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  if (MODE) __stcs(r + i, c); else r[i] = c;
}
// warp per 256*R elements, R rounds of 2 float4 per lane (scan layout), optional flag+ballot, optional candidate writes
template <int R, int FLAGS, int CANDS>
__global__ void seg(const float* __restrict__ g, float* __restrict__ r, uint64_t* cand, uint32_t* cnt, size_t n, uint32_t thr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t segi = (size_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const size_t base = segi * 256 * R;
  if (base >= n) return;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t run = 0;
#pragma unroll 1
  for (int rd = 0; rd < R; ++rd) {
    float4 a[2], b[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const size_t e0 = base + 4 * ((rd * 2 + j) * 32 + lane);
      a[j] = *reinterpret_cast<const float4*>(g + e0);
      b[j] = *reinterpret_cast<const float4*>(r + e0);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const size_t e0 = base + 4 * ((rd * 2 + j) * 32 + lane);
      float4 c = make_float4(a[j].x + b[j].x, a[j].y + b[j].y, a[j].z + b[j].z, a[j].w + b[j].w);
      *reinterpret_cast<float4*>(r + e0) = c;
      if (FLAGS) {
        float cv[4] = {c.x, c.y, c.z, c.w};
        uint32_t fl = 0;
        for (int k = 0; k < 4; ++k) fl |= ((__float_as_uint(cv[k]) & 0x7fffffffu) >= thr) ? 1u << k : 0u;
        unsigned bm[4];
        for (int k = 0; k < 4; ++k) bm[k] = __ballot_sync(0xffffffffu, (fl >> k) & 1u);
        uint32_t pos = run;
        for (int k = 0; k < 4; ++k) pos += __popc(bm[k] & lt);
        if (CANDS && fl) {
          for (int k = 0; k < 4; ++k)
            if ((fl >> k) & 1u) cand[segi * 256 * R + pos++] = ((uint64_t)__float_as_uint(cv[k]) << 32) | (uint32_t)(e0 + k);
        }
        for (int k = 0; k < 4; ++k) run += __popc(bm[k]);
      }
    }
  }
  if (FLAGS && lane == 0) cnt[segi] = run;
}

// scan-like: per-CTA chunk table lookups before the streaming loads
template <int R, int PREFETCH_THR>
__global__ void segtbl(const float* __restrict__ g, float* __restrict__ r, uint64_t* cand, uint32_t* cnt,
                       const uint64_t* cbase, const uint64_t* clo, const uint64_t* chi, const int* cslot,
                       const uint32_t* thrs, size_t n) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ch = blockIdx.x / (16 / (blockDim.x >> 5) / R * 1);   // 16*1024/(R*256*warps) CTAs per chunk
  const int per = 16384 / (256 * R * (blockDim.x >> 5));
  const int chk = blockIdx.x / per;
  const int seg = (blockIdx.x % per) * (blockDim.x >> 5) + warp;
  const uint64_t sbase = cbase[chk] + (uint64_t)seg * 256 * R;
  const uint64_t lo = clo[chk], hi = chi[chk];
  const uint32_t thr = thrs[cslot[chk]];
  const unsigned lt = (1u << lane) - 1u;
  uint32_t run = 0;
#pragma unroll 1
  for (int rd = 0; rd < R; ++rd) {
    float4 a[2], b[2]; uint32_t vm[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint64_t e0 = sbase + 4 * ((rd * 2 + j) * 32 + lane);
      vm[j] = (e0 >= lo && e0 + 4 <= hi) ? 0xF : 0;
      if (vm[j]) { a[j] = *reinterpret_cast<const float4*>(g + e0); b[j] = *reinterpret_cast<const float4*>(r + e0); }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint64_t e0 = sbase + 4 * ((rd * 2 + j) * 32 + lane);
      float4 c = make_float4(a[j].x + b[j].x, a[j].y + b[j].y, a[j].z + b[j].z, a[j].w + b[j].w);
      if (vm[j]) *reinterpret_cast<float4*>(r + e0) = c;
      float cv[4] = {c.x, c.y, c.z, c.w};
      uint32_t fl = 0;
      for (int k = 0; k < 4; ++k) fl |= (vm[j] && (__float_as_uint(cv[k]) & 0x7fffffffu) >= thr) ? 1u << k : 0u;
      unsigned bm[4];
      for (int k = 0; k < 4; ++k) bm[k] = __ballot_sync(0xffffffffu, (fl >> k) & 1u);
      uint32_t pos = run;
      for (int k = 0; k < 4; ++k) pos += __popc(bm[k] & lt);
      if (fl) for (int k = 0; k < 4; ++k) if ((fl >> k) & 1u) cand[(size_t)chk * 16384 + seg * 256 * R + pos++] = ((uint64_t)__float_as_uint(cv[k]) << 32) | (uint32_t)(e0 + k);
      for (int k = 0; k < 4; ++k) run += __popc(bm[k]);
    }
  }
  if (lane == 0) cnt[(size_t)chk * 64 + seg] = run;
}

__global__ void fill(float* x, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)(i * 2654435761u) ^ seed; h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    float u = (h & 0xFFFFFF) / 16777216.0f;           // uniform -> ~2% above 0.98 in |2u-1|
    x[i] = (2.f * u - 1.f) * 1e-3f;
  }
}

int main(int argc, char** argv) {
  size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 1557611200ull;
  n &= ~(size_t)4095;
  size_t n4 = n / 4;
  float *g, *r; uint64_t* cand; uint32_t* cnt;
  cudaMalloc(&g, n * 4); cudaMalloc(&r, n * 4); cudaMalloc(&cand, n * 8); cudaMalloc(&cnt, n / 256 * 4 + 64);
  // gaussian-ish data: use a hash so that ~2% exceed thr
  cudaMemset(g, 0, n * 4); cudaMemset(r, 0, n * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 2; ++i) launch();
    cudaEventRecord(a);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    printf("%-36s %8.3f ms  %8.1f GB/s  err=%s\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  const double B = 12.0 * n;
  run("add1 plain b256", B, [&] { add1<0><<<(n4 + 255) / 256, 256>>>((float4*)g, (float4*)r, n4); });
  run("add1 cs b256", B, [&] { add1<1><<<(n4 + 255) / 256, 256>>>((float4*)g, (float4*)r, n4); });
  run("add1 plain b128", B, [&] { add1<0><<<(n4 + 127) / 128, 128>>>((float4*)g, (float4*)r, n4); });
  run("seg R1 noflag b128", B, [&] { seg<1, 0, 0><<<n / 1024, 128>>>(g, r, cand, cnt, n, 0x3f000000u); });
  run("seg R4 noflag b128", B, [&] { seg<4, 0, 0><<<n / 4096, 128>>>(g, r, cand, cnt, n, 0x3f000000u); });
  run("seg R4 flags b128", B, [&] { seg<4, 1, 0><<<n / 4096, 128>>>(g, r, cand, cnt, n, 0x3f000000u); });
  run("seg R4 flags+cands(none) b128", B, [&] { seg<4, 1, 1><<<n / 4096, 128>>>(g, r, cand, cnt, n, 0x7f000000u); });
  run("seg R1 flags b256", B, [&] { seg<1, 1, 0><<<n / 2048, 256>>>(g, r, cand, cnt, n, 0x3f000000u); });
  run("seg R4 noflag b256", B, [&] { seg<4, 0, 0><<<n / 8192, 256>>>(g, r, cand, cnt, n, 0x3f000000u); });
  run("seg R2 noflag b256", B, [&] { seg<2, 0, 0><<<n / 4096, 256>>>(g, r, cand, cnt, n, 0x3f000000u); });
  // chunk tables: contiguous chunks of 16384
  const size_t nch = n / 16384;
  uint64_t *cb, *cl, *chh; int* cs; uint32_t* th;
  cudaMalloc(&cb, nch * 8); cudaMalloc(&cl, nch * 8); cudaMalloc(&chh, nch * 8); cudaMalloc(&cs, nch * 4); cudaMalloc(&th, 4096);
  {
    uint64_t* h = (uint64_t*)malloc(nch * 8); int* hs = (int*)malloc(nch * 4);
    for (size_t i = 0; i < nch; ++i) { h[i] = i * 16384; hs[i] = (int)(i * 194 / nch); }
    cudaMemcpy(cb, h, nch * 8, cudaMemcpyHostToDevice); cudaMemcpy(cl, h, nch * 8, cudaMemcpyHostToDevice);
    for (size_t i = 0; i < nch; ++i) h[i] += 16384;
    cudaMemcpy(chh, h, nch * 8, cudaMemcpyHostToDevice); cudaMemcpy(cs, hs, nch * 4, cudaMemcpyHostToDevice);
    cudaMemset(th, 0x7f, 4096);
  }
  fill<<<4096, 256>>>(g, n, 1u); fill<<<4096, 256>>>(r, n, 2u); cudaDeviceSynchronize();
  uint32_t thr_h[1024]; { float t = 1.96e-3f; uint32_t b; memcpy(&b, &t, 4); for (int i = 0; i < 1024; ++i) thr_h[i] = b; }
  cudaMemcpy(th, thr_h, 4096, cudaMemcpyHostToDevice);
  run("segtbl R4 w4 real data ~2% cands", B, [&] { fill<<<4096,256>>>(r, 0, 3u); segtbl<4, 0><<<nch * 4, 128>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  run("segtbl R2 w8 real data", B, [&] { segtbl<2, 0><<<nch * 4, 256>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  memset(thr_h, 0x7f, 4096); cudaMemcpy(th, thr_h, 4096, cudaMemcpyHostToDevice);
  run("segtbl R4 w4 real data no cands", B, [&] { segtbl<4, 0><<<nch * 4, 128>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  run("segtbl R4 w4 (scan-like)", B, [&] { segtbl<4, 0><<<nch * 4, 128>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  run("segtbl R1 w4", B, [&] { segtbl<1, 0><<<nch * 16, 128>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  run("segtbl R2 w8", B, [&] { segtbl<2, 0><<<nch * 4, 256>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  run("segtbl R8 w2", B, [&] { segtbl<8, 0><<<nch * 4, 64>>>(g, r, cand, cnt, cb, cl, chh, cs, th, n); });
  return 0;
}
