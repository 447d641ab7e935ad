// lowdiff_selftest: device-side proofs for the branch-free IEEE helpers of ieee_fast.cuh
// (modes 0-3 below; 4 and 5: every exponent pair of the division / Adam-direction windows).
//   which = 0: sqrt_rn_nb vs __fsqrt_rn over every non-negative float and -0 (2^31 + 1 inputs)
//   which = 1: div_rn_nb vs __fdiv_rn on n pseudo-random operand pairs: raw 32-bit patterns
//              (NaN, Inf, denormals, zeros included) and pairs drawn from the replay's domain
//              (m*r1 over sqrt(v*r2)+eps), plus exhaustive sweeps of the window edges
#include <cuda_runtime.h>

#include "ieee_fast.cuh"
#include "internal.h"

namespace ld {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void sqrt_check_kernel(unsigned long long* bad, unsigned long long* first) {
  const uint64_t total = (1ull << 31) + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = i == (1ull << 31) ? 0x80000000u : (uint32_t)i;
    const float x = __uint_as_float(u);
    const uint32_t a = __float_as_uint(sqrt_rn_nb(x)), b = __float_as_uint(__fsqrt_rn(x));
    if (a != b) {
      atomicAdd(bad, 1ull);
      atomicMin(first, (unsigned long long)u);
    }
  }
}

__global__ void div_check_kernel(uint64_t n, uint64_t seed, unsigned long long* bad, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed ^ mix64(i));
    const uint64_t h2 = mix64(h);
    uint32_t ua, ub;
    switch (i & 3) {
      case 0:   // raw bit patterns
        ua = (uint32_t)h;
        ub = (uint32_t)(h >> 32);
        break;
      case 1: {  // the replay's domain: mh ~ 1e-30..1e3 (either sign), d = sqrt(vh) + eps >= 1e-8
        const float mag = exp2f(-100.f + 110.f * (float)(h & 0xFFFFFF) / 16777216.f);
        const float mh = ((h >> 24) & 1) ? -mag : mag;
        const float vh = exp2f(-80.f + 90.f * (float)((h >> 32) & 0xFFFFFF) / 16777216.f);
        ua = __float_as_uint(mh);
        ub = __float_as_uint(__fadd_rn(__fsqrt_rn(vh), 1e-8f));
        break;
      }
      case 2: {  // exponents swept across the fast-window edges, random mantissas
        const uint32_t ea = 40 + (uint32_t)(h % 180), eb = 40 + (uint32_t)((h >> 16) % 180);
        ua = ((uint32_t)(h2 >> 63) << 31) | (ea << 23) | ((uint32_t)h2 & 0x7FFFFF);
        ub = ((uint32_t)(h2 >> 62 & 1) << 31) | (eb << 23) | ((uint32_t)(h2 >> 23) & 0x7FFFFF);
        break;
      }
      default: {  // near-ties: mantissas with few bits set, zeros, denormals
        ua = (uint32_t)h & 0xFF8000FFu;
        ub = ((uint32_t)(h >> 32) & 0xFFF00001u) | 0x00800000u;
        if ((h2 & 15) == 0) ua &= 0x80000000u;
        if ((h2 & 240) == 0) ub &= 0x807FFFFFu;
        break;
      }
    }
    const float a = __uint_as_float(ua), b = __uint_as_float(ub);
    const uint32_t x = __float_as_uint(div_rn_nb(a, b)), y = __float_as_uint(__fdiv_rn(a, b));
    if (x != y && !((x & 0x7FFFFFFFu) > 0x7F800000u && (y & 0x7FFFFFFFu) > 0x7F800000u)) {
      atomicAdd(bad, 1ull);
      atomicMin(first, (unsigned long long)i);
    }
  }
}

// which = 2: adam_u_fast(mh, vh, eps) + the exact fallback vs __fdiv_rn(mh, __fsqrt_rn(vh) + eps)
__global__ void adam_check_kernel(uint64_t n, uint64_t seed, unsigned long long* bad, unsigned long long* first) {
  const float eps_set[4] = {1e-8f, 1e-6f, 0x1p-60f, 1.0f};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed ^ mix64(i)), h2 = mix64(h);
    const float eps = eps_set[h2 & 3];
    uint32_t ua, uv;
    if ((i & 1) == 0) {   // raw bit patterns (vh forced non-negative, as Adam's v*r2 is)
      ua = (uint32_t)h;
      uv = (uint32_t)(h >> 32) & 0x7FFFFFFFu;
    } else {              // Adam's domain, zeros and window edges
      const float mag = exp2f(-140.f + 270.f * (float)(h & 0xFFFFFF) / 16777216.f);
      ua = __float_as_uint(((h >> 24) & 1) ? -mag : mag);
      uv = __float_as_uint(exp2f(-140.f + 270.f * (float)((h >> 32) & 0xFFFFFF) / 16777216.f));
      if ((h2 & 0x30) == 0) ua &= 0x80000000u;
      if ((h2 & 0xC0) == 0) uv = 0;
    }
    const float mh = __uint_as_float(ua), vh = __uint_as_float(uv);
    bool sl;
    float u = adam_u_fast(mh, vh, eps, &sl);
    if (sl) u = __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), eps));
    const uint32_t x = __float_as_uint(u), y = __float_as_uint(__fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), eps)));
    if (x != y && !((x & 0x7FFFFFFFu) > 0x7F800000u && (y & 0x7FFFFFFFu) > 0x7F800000u)) {
      atomicAdd(bad, 1ull);
      atomicMin(first, (unsigned long long)i);
    }
  }
}

// which = 3: the paired Adam step (adam2_u_agg, the exact form when its window test fails, then p - lr*u) on random states vs
// the scalar R-11 sequence written with the CUDA intrinsics
__global__ void adam2_check_kernel(uint64_t n, uint64_t seed, float neg0, unsigned long long* bad,
                                   unsigned long long* first) {
  const float eps_set[4] = {1e-8f, 1e-6f, 0x1p-60f, 1.0f};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float p[2], m[2], v[2], g[2];
    uint64_t h = mix64(seed ^ mix64(i));
    const float eps = eps_set[h & 3];
    const float b1 = 0.9f, c1 = 0.1f, b2 = 0.999f, c2 = 0.001f;
    const float lr = exp2f(-20.f + 19.f * (float)((h >> 8) & 0xFFFF) / 65536.f);
    const float r1 = 1.f + 9.f * (float)((h >> 24) & 0xFFFF) / 65536.f;
    const float r2 = 1.f + 999.f * (float)((h >> 40) & 0xFFFF) / 65536.f;
    for (int e = 0; e < 2; ++e) {
      h = mix64(h);
      const float mag = exp2f(-150.f + 200.f * (float)(h & 0xFFFFFF) / 16777216.f);
      g[e] = ((h >> 24) & 1) ? -mag : mag;
      if (((h >> 25) & 7) == 0) g[e] = ((h >> 28) & 1) ? -0.0f : 0.0f;
      h = mix64(h);
      p[e] = __uint_as_float((uint32_t)h & 0xBFFFFFFFu);   // finite, any sign
      const float mm = exp2f(-150.f + 160.f * (float)((h >> 32) & 0xFFFFFF) / 16777216.f);
      m[e] = ((h >> 56) & 1) ? -mm : mm;
      if (((h >> 57) & 7) == 0) m[e] = 0.0f;
      h = mix64(h);
      v[e] = exp2f(-150.f + 160.f * (float)(h & 0xFFFFFF) / 16777216.f);
      if (((h >> 24) & 7) == 0) v[e] = 0.0f;
    }
    const AdamK2 k2 = make_adamk2(b1, c1, b2, c2, eps, neg0);
    f32x2 P = pk2(p[0], p[1]), M = pk2(m[0], m[1]), V = pk2(v[0], v[1]);
    WinAcc w = win_init();
    f32x2 u = adam2_u_agg(M, V, pk2(g[0], g[1]), k2, pk2(r1, r1), pk2(-r2, -r2), w);
    const f32x2 mh = mul2(M, pk2(r1, r1)), vh = mul2(V, pk2(r2, r2));
    if (win_bad(w))
      u = pk2(__fdiv_rn(lo2(mh), __fadd_rn(__fsqrt_rn(lo2(vh)), eps)),
              __fdiv_rn(hi2(mh), __fadd_rn(__fsqrt_rn(hi2(vh)), eps)));
    P = sub_prod2(P, pk2(lr, lr), u, k2.nz);
    const float got[6] = {lo2(P), hi2(P), lo2(M), hi2(M), lo2(V), hi2(V)};
    for (int e = 0; e < 2; ++e) {
      const float me = __fadd_rn(__fmul_rn(b1, m[e]), __fmul_rn(c1, g[e]));
      const float ve = __fadd_rn(__fmul_rn(b2, v[e]), __fmul_rn(c2, __fmul_rn(g[e], g[e])));
      const float ue = __fdiv_rn(__fmul_rn(me, r1), __fadd_rn(__fsqrt_rn(__fmul_rn(ve, r2)), eps));
      const float pe = __fsub_rn(p[e], __fmul_rn(lr, ue));
      const float want[3] = {pe, me, ve};
      const float have[3] = {got[e], got[2 + e], got[4 + e]};
      for (int q = 0; q < 3; ++q) {
        const uint32_t x = __float_as_uint(have[q]), y = __float_as_uint(want[q]);
        if (x != y && !((x & 0x7FFFFFFFu) > 0x7F800000u && (y & 0x7FFFFFFFu) > 0x7F800000u)) {
          atomicAdd(bad, 1ull);
          atomicMin(first, (unsigned long long)i);
        }
      }
    }
  }
}

// which = 4: division, every exponent pair: for each pair (ea, eb) of biased exponents in
// [57, 194] (|a|, |b| from 2^-70 to 2^67: the window [2^-60, 2^61) of div_rn_fast and ten binades
// around each edge) the four extreme mantissa combinations and n / 138^2 - 4 random mantissa pairs,
// all four sign combinations -- div_rn_nb vs __fdiv_rn.  Item i: pair = i % 138^2, k = i / 138^2.
// which = 5: the paired Adam direction adam2_u_agg (+ the exact form when win_bad) vs the scalar
// R-11 sequence, every exponent pair of (mh, vh) in [37, 214] x [0, 254] (vh down to denormals),
// extreme and random mantissas, eps in {1e-8, 1e-6, 2^-60, 1}, zeros mixed in.
__global__ void pair_sweep_kernel(int which, uint64_t n, uint64_t seed, float neg0, unsigned long long* bad,
                                  unsigned long long* first) {
  const uint32_t A0 = which == 4 ? 57u : 37u, NA = which == 4 ? 138u : 178u;
  const uint32_t B0 = which == 4 ? 57u : 0u, NB = which == 4 ? 138u : 255u;
  const uint64_t npairs = (uint64_t)NA * NB;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pr = i % npairs, k = i / npairs;
    const uint32_t ea = A0 + (uint32_t)(pr % NA), eb = B0 + (uint32_t)(pr / NA);
    const uint64_t h = mix64(seed ^ mix64(i));
    uint32_t ma, mb;
    if (k < 4) {   // extreme mantissas
      ma = (k & 1) ? 0x7FFFFFu : 0u;
      mb = (k & 2) ? 0x7FFFFFu : 0u;
    } else {
      ma = (uint32_t)h & 0x7FFFFFu;
      mb = (uint32_t)(h >> 23) & 0x7FFFFFu;
    }
    const uint32_t sa = (uint32_t)(h >> 62) & 1u, sb = which == 4 ? (uint32_t)(h >> 63) : 0u;
    const float a = __uint_as_float((sa << 31) | (ea << 23) | ma);
    const float b = __uint_as_float((sb << 31) | (eb << 23) | mb);
    uint32_t x, y;
    if (which == 4) {
      x = __float_as_uint(div_rn_nb(a, b));
      y = __float_as_uint(__fdiv_rn(a, b));
    } else {
      const float eps_set[4] = {1e-8f, 1e-6f, 0x1p-60f, 1.0f};
      const float eps = eps_set[(h >> 48) & 3];
      const float mh = ((h >> 50) & 15) == 0 ? 0.0f : a, vh = ((h >> 54) & 15) == 0 ? 0.0f : b;
      // one Adam step from m = (mh, -mh), v = vh with g = 0, b1 = b2 = 1, c1 = c2 = 0, r1 = r2 = 1:
      // the moments pass through (up to the sign of a zero: -0 + +0 = +0, as in the scalar R-11
      // sequence written out below), so the direction is mh / (sqrt(vh) + eps) for each half
      const AdamK2 k2 = make_adamk2(1.f, 0.f, 1.f, 0.f, eps, neg0);
      f32x2 M = pk2(mh, -mh), V = pk2(vh, vh);
      WinAcc w = win_init();
      f32x2 u = adam2_u_agg(M, V, pk2(0.f, 0.f), k2, pk2(1.f, 1.f), pk2(-1.f, -1.f), w);
      float want[2];
      for (int e = 0; e < 2; ++e) {
        const float m0 = e ? -mh : mh;
        const float me = __fadd_rn(__fmul_rn(1.f, m0), __fmul_rn(0.f, 0.f));
        const float ve = __fadd_rn(__fmul_rn(1.f, vh), __fmul_rn(0.f, __fmul_rn(0.f, 0.f)));
        want[e] = __fdiv_rn(__fmul_rn(me, 1.f), __fadd_rn(__fsqrt_rn(__fmul_rn(ve, 1.f)), eps));
      }
      if (win_bad(w)) u = pk2(want[0], want[1]);   // the caller's exact re-run
      const uint32_t x1 = __float_as_uint(hi2(u)), y1 = __float_as_uint(want[1]);
      const bool hi_ok = x1 == y1 || ((x1 & 0x7FFFFFFFu) > 0x7F800000u && (y1 & 0x7FFFFFFFu) > 0x7F800000u);
      x = hi_ok ? __float_as_uint(lo2(u)) : ~__float_as_uint(want[0]);   // a wrong high half fails too
      y = __float_as_uint(want[0]);
    }
    if (x != y && !((x & 0x7FFFFFFFu) > 0x7F800000u && (y & 0x7FFFFFFFu) > 0x7F800000u)) {
      atomicAdd(bad, 1ull);
      atomicMin(first, (unsigned long long)i);
    }
  }
}

}  // namespace

cudaError_t run_selftest(int which, uint64_t n, uint64_t seed, uint64_t* mismatches, uint64_t* first) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 16);
  if (e != cudaSuccess) return e;
  unsigned long long init[2] = {0ull, ~0ull};
  cudaMemcpy(d, init, 16, cudaMemcpyHostToDevice);
  if (which == 0) sqrt_check_kernel<<<148 * 16, 256>>>(d, d + 1);
  else if (which == 1) div_check_kernel<<<148 * 16, 256>>>(n, seed, d, d + 1);
  else if (which == 2) adam_check_kernel<<<148 * 16, 256>>>(n, seed, d, d + 1);
  else if (which == 3) adam2_check_kernel<<<148 * 16, 256>>>(n, seed, -0.0f, d, d + 1);
  else pair_sweep_kernel<<<148 * 16, 256>>>(which, n, seed, -0.0f, d, d + 1);
  e = cudaDeviceSynchronize();
  unsigned long long h[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  *mismatches = h[0];
  *first = h[1];
  return e;
}

}  // namespace ld
