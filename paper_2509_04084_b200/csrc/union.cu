// Union-compacted differentials on sm_100a (lowdiff_union_compact / lowdiff_union_persist).
//
// What it computes (R-29): the synchronised compressed gradient G~_t of
// Alg. 1 line 5, put in the reusing queue after Sync (line 6) and kept
// as an index -> value dictionary: for the element range [lo, hi) of this rank's
// shard, every index j that appears in some rank's block, ascending, with the merged value
// G_t[j] = (((+0 + v_0[j]) + v_1[j]) + ... ) / N -- exactly the value lowdiff_exchange writes into
// the dense gradient (same rank order, same division).  When the ranks' supports overlap the union
// is smaller than the N fixed-K blocks (0.47 N K at rank correlation 0.9).
//
// How: the merge's 8192-element tile grid.  Pass 1 (one CTA per tile in the window): a 8192-bit
// membership bitmap in shared memory from every rank's entries of the tile (binary-searched start
// table, as in the merge), popcount inside [lo, hi) -> tile count.  Pass 2 (one CTA): exclusive scan
// of the tile counts -> output offsets and the total.  Pass 3 (one CTA per tile): the bitmap again
// plus the rank-order sum in a shared-memory accumulator, a block scan of the per-word popcounts,
// and every thread writes the members of its 32-element word in index order.
// HBM: the gathered entries of the window twice (2 x 8 B per entry) + 8 B per union entry.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace ld {
namespace {

constexpr int kUT = kMergeTile;               // elements per tile
constexpr int kUWords = kUT / 32;             // bitmap words per tile (= threads per CTA)
static_assert(kUWords == 256, "one bitmap word per thread");

// G = S / N, as the merge (merge_replay.cu): DIV 0 none, 1 power of two (exact scaling), 2 IEEE
template <int DIV>
__device__ __forceinline__ float umean(float s, float n, float inv) {
  if (DIV == 0) return s;
  if (DIV == 1) return __fmul_rn(s, inv);
  return __fdiv_rn(s, n);
}

// bits of word w (elements j0 + 32 w + b) that lie in [lo, hi)
__device__ __forceinline__ uint32_t word_mask(uint64_t jw, uint64_t lo, uint64_t hi) {
  if (jw >= hi || jw + 32 <= lo) return 0u;
  uint32_t m = 0xFFFFFFFFu;
  if (jw < lo) m &= 0xFFFFFFFFu << (uint32_t)(lo - jw);
  if (jw + 32 > hi) m &= 0xFFFFFFFFu >> (uint32_t)(jw + 32 - hi);
  return m;
}

__device__ __forceinline__ uint32_t block_scan256(uint32_t x, uint32_t* sh, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < 8 ? sh[lane] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, vi, o);
      if (lane >= o) vi += y;
    }
    if (lane < 8) sh[lane] = vi - v;
    if (lane == 7) sh[8] = vi;
  }
  __syncthreads();
  const uint32_t r = sh[wid] + inc - x;
  *total = sh[8];
  return r;
}

// membership bitmap of tile t (relative window tile tl) from every rank's entries
__device__ __forceinline__ void build_bitmap(const uint32_t* __restrict__ gathered, int world, uint64_t K,
                                             const uint32_t* __restrict__ start, int64_t nt, int64_t tl,
                                             uint32_t j0, uint32_t* bm) {
  for (int r = 0; r < world; ++r) {
    const uint32_t* idx = gathered + (uint64_t)r * 2 * K;
    const uint32_t* st = start + (uint64_t)r * (nt + 1) + tl;
    const uint32_t a = __ldg(st), b = __ldg(st + 1);
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const uint32_t j = __ldg(idx + e) - j0;
      atomicOr(&bm[j >> 5], 1u << (j & 31));
    }
  }
}

__global__ void __launch_bounds__(256)
union_count_kernel(const uint32_t* __restrict__ gathered, int world, uint64_t K, const uint32_t* __restrict__ start,
                   int64_t nt, int64_t t0, uint64_t lo, uint64_t hi, uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t bm[kUWords];
  __shared__ uint32_t sh[9];
  const int64_t tl = blockIdx.x;
  const uint64_t j0 = (uint64_t)(t0 + tl) * kUT;
  bm[threadIdx.x] = 0u;
  __syncthreads();
  build_bitmap(gathered, world, K, start, nt, tl, (uint32_t)j0, bm);
  __syncthreads();
  const uint32_t c = __popc(bm[threadIdx.x] & word_mask(j0 + 32u * threadIdx.x, lo, hi));
  uint32_t tot;
  block_scan256(c, sh, &tot);
  if (threadIdx.x == 0) tile_cnt[tl] = tot;
}

// exclusive scan of nt tile counts by one 1024-thread CTA (thread q owns a contiguous run)
__global__ void __launch_bounds__(1024)
union_scan_kernel(const uint32_t* __restrict__ cnt, int64_t nt, uint32_t* __restrict__ off,
                  unsigned long long* __restrict__ total) {
  __shared__ uint32_t sh[33];
  const int64_t per = (nt + 1023) / 1024;
  const int64_t a0 = (int64_t)threadIdx.x * per, a = a0 < nt ? a0 : nt, b = a + per < nt ? a + per : nt;
  uint32_t s = 0;
  for (int64_t i = a; i < b; ++i) s += cnt[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = sh[lane];
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, vi, o);
      if (lane >= o) vi += y;
    }
    sh[lane] = vi - v;
    if (lane == 31) sh[32] = vi;
  }
  __syncthreads();
  uint32_t run = sh[wid] + inc - s;
  for (int64_t i = a; i < b; ++i) {
    off[i] = run;
    run += cnt[i];
  }
  if (threadIdx.x == 0) *total = sh[32];
}

template <int DIV>
__global__ void __launch_bounds__(256)
union_emit_kernel(const uint32_t* __restrict__ gathered, int world, uint64_t K, const uint32_t* __restrict__ start,
                  int64_t nt, int64_t t0, uint64_t lo, uint64_t hi, const uint32_t* __restrict__ off, uint64_t cap,
                  uint32_t* __restrict__ out) {
  __shared__ float acc[kUT];
  __shared__ uint32_t bm[kUWords];
  __shared__ uint32_t sh[9];
  const int64_t tl = blockIdx.x;
  const uint64_t j0 = (uint64_t)(t0 + tl) * kUT;
  float4* acc4 = reinterpret_cast<float4*>(acc);
  for (int q = threadIdx.x; q < kUT / 4; q += blockDim.x) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  bm[threadIdx.x] = 0u;
  __syncthreads();
  // rank by rank from +0 (the merge's order; indices are unique within a rank)
  for (int r = 0; r < world; ++r) {
    const uint32_t* idx = gathered + (uint64_t)r * 2 * K;
    const uint32_t* val = idx + K;
    const uint32_t* st = start + (uint64_t)r * (nt + 1) + tl;
    const uint32_t a = __ldg(st), b = __ldg(st + 1);
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const uint32_t j = __ldg(idx + e) - (uint32_t)j0;
      acc[j] = __fadd_rn(acc[j], __uint_as_float(__ldg(val + e)));
      atomicOr(&bm[j >> 5], 1u << (j & 31));
    }
    __syncthreads();
  }
  uint32_t word = bm[threadIdx.x] & word_mask(j0 + 32u * threadIdx.x, lo, hi);
  uint32_t tot;
  uint64_t pos = (uint64_t)off[tl] + block_scan256(__popc(word), sh, &tot);
  const float n = (float)world, inv = 1.0f / (float)world;
  while (word) {
    const int bit = __ffs(word) - 1;
    word &= word - 1;
    const uint32_t jl = 32u * threadIdx.x + (uint32_t)bit;
    if (pos < cap) {
      out[pos] = (uint32_t)j0 + jl;
      out[cap + pos] = __float_as_uint(umean<DIV>(acc[jl], n, inv));
    }
    ++pos;
  }
}

}  // namespace

size_t union_scratch_bytes(int world, uint64_t lo, uint64_t hi) {
  if (hi <= lo) return 0;
  const int64_t t0 = (int64_t)(lo / kUT), nt = (int64_t)((hi - 1) / kUT) - t0 + 1;
  return ((size_t)world * (nt + 1) + 2 * (size_t)nt) * sizeof(uint32_t);
}

cudaError_t launch_union(lowdiff_ctx* c, int world, bool mean, const uint32_t* gathered, uint64_t lo, uint64_t hi,
                         uint32_t* out, uint64_t cap, unsigned long long* count_dev, cudaStream_t s) {
  if (hi <= lo) return cudaMemsetAsync(count_dev, 0, sizeof(unsigned long long), s);
  const uint64_t K = (uint64_t)c->K;
  const int64_t t0 = (int64_t)(lo / kUT), nt = (int64_t)((hi - 1) / kUT) - t0 + 1;
  const size_t need = union_scratch_bytes(world, lo, hi);
  if (c->union_scratch_bytes < need) {
    if (c->union_scratch) cudaFree(c->union_scratch);
    c->union_scratch = nullptr;
    c->union_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&c->union_scratch, need);
    if (e != cudaSuccess) return e;
    c->union_scratch_bytes = need;
  }
  uint32_t* start = static_cast<uint32_t*>(c->union_scratch);
  uint32_t* cnt = start + (size_t)world * (nt + 1);
  uint32_t* off = cnt + nt;
  int h;
  prof_begin(c, "union", s, &h);
  cudaError_t e = launch_tile_window(gathered, world, K, kMergeTileShift, (uint32_t)t0, (uint32_t)(t0 + nt), start, s);
  if (e != cudaSuccess) return e;
  union_count_kernel<<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, cnt);
  union_scan_kernel<<<1, 1024, 0, s>>>(cnt, nt, off, count_dev);
  const int dm = !mean || world == 1 ? 0 : ((world & (world - 1)) == 0 ? 1 : 2);
  if (dm == 0) union_emit_kernel<0><<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, off, cap, out);
  else if (dm == 1) union_emit_kernel<1><<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, off, cap, out);
  else union_emit_kernel<2><<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, off, cap, out);
  prof_end(c, h, s);
  c->launches += 4;
  return cudaGetLastError();
}

}  // namespace ld
