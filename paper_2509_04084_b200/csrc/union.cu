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
// How: the merge's 8192-element tile grid, one CTA per tile of the window, one pass: a 8192-bit
// membership bitmap and the rank-order sums in shared memory (binary-searched tile-start table, as
// in the merge), the tile's count inside [lo, hi), its output offset by a decoupled look-back over
// the preceding tiles, and every thread writes the members of its 32-element word in index order.
// (A three-kernel version -- count, scan, emit -- read the entries twice: 0.61 ms per GPT-2 XL shard
// at 8 ranks.)  HBM: 8 B per gathered entry in the window + 8 B per union entry.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace ld {
namespace {

constexpr int kUT = kMergeTile;               // elements per tile
constexpr int kUWords = kUT / 32;             // bitmap words per tile (= threads per CTA)
constexpr int kUGroup = 8;                    // ranks whose first entries are loaded together
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

// Single pass (one CTA per tile): membership bitmap and rank-order sums built together -- an
// element's first rank writes +0 + v, later ranks add (the bitmap says whether the element was
// already touched; indices are unique within a rank, ranks are separated by barriers), so the
// 32 KB accumulator needs no zeroing -- then the tile's count, its output offset by a decoupled
// look-back over the preceding tiles' published counts (warp 0 reads 32 predecessors at a time),
// and the ordered emit.  One read of the entries, one launch.

template <int DIV>
__global__ void __launch_bounds__(256)
union_tile_kernel(const uint32_t* __restrict__ gathered, int world, uint64_t K, const uint32_t* __restrict__ start,
                  int64_t nt, int64_t t0, uint64_t lo, uint64_t hi, unsigned long long* __restrict__ tile_state,
                  uint64_t cap, uint32_t* __restrict__ out, unsigned long long* __restrict__ count) {
  __shared__ float acc[kUT];
  __shared__ uint32_t bm[kUWords];
  __shared__ uint32_t sh[9];
  __shared__ unsigned long long s_excl;
  const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kValMask = (1ull << 62) - 1;
  const int64_t tl = blockIdx.x;
  const uint64_t j0 = (uint64_t)(t0 + tl) * kUT;
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t s_a[kUGroup], s_b[kUGroup];
  bm[threadIdx.x] = 0u;
  auto add = [&](uint32_t j, float v) {
    const uint32_t bit = 1u << (j & 31);
    const bool seen = (bm[j >> 5] & bit) != 0u;   // set by an earlier rank (barrier-ordered)
    acc[j] = __fadd_rn(seen ? acc[j] : 0.0f, v);
    if (!seen) atomicOr(&bm[j >> 5], bit);
  };
  // ranks in groups of kUGroup: their tile ranges in one round trip, the first round of every rank's
  // entries in registers in a second, then the rank-ordered adds out of registers
  for (int r0 = 0; r0 < world; r0 += kUGroup) {
    const int ng = world - r0 < kUGroup ? world - r0 : kUGroup;
    if ((int)threadIdx.x < ng) {
      const uint32_t* st = start + (uint64_t)(r0 + threadIdx.x) * (nt + 1) + tl;
      s_a[threadIdx.x] = __ldg(st);
      s_b[threadIdx.x] = __ldg(st + 1);
    }
    __syncthreads();
    uint32_t pj[kUGroup], pv[kUGroup];
#pragma unroll
    for (int g = 0; g < kUGroup; ++g) {
      pj[g] = 0xFFFFFFFFu;
      pv[g] = 0u;
      if (g < ng) {
        const uint32_t e = s_a[g] + threadIdx.x;
        if (e < s_b[g]) {
          const uint32_t* idx = gathered + (uint64_t)(r0 + g) * 2 * K;
          pj[g] = __ldg(idx + e) - (uint32_t)j0;
          pv[g] = __ldg(idx + K + e);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kUGroup; ++g) {
      if (g < ng) {
        if (pj[g] != 0xFFFFFFFFu) add(pj[g], __uint_as_float(pv[g]));
        const uint32_t* idx = gathered + (uint64_t)(r0 + g) * 2 * K;
        for (uint32_t e = s_a[g] + blockDim.x + threadIdx.x; e < s_b[g]; e += blockDim.x)
          add(__ldg(idx + e) - (uint32_t)j0, __uint_as_float(__ldg(idx + K + e)));
        __syncthreads();
      }
    }
  }
  uint32_t word = bm[threadIdx.x] & word_mask(j0 + 32u * threadIdx.x, lo, hi);
  uint32_t tot;
  const uint32_t pre = block_scan256(__popc(word), sh, &tot);
  if (threadIdx.x < 32) {
    unsigned long long excl = 0;
    if (tl == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(tile_state, kInc | tot);
      }
    } else {
      if (lane == 0) atomicExch(tile_state + tl, kAgg | tot);
      int64_t p = tl - 1;
      for (;;) {
        const int64_t q = p - lane;   // lane 0: the nearest predecessor
        unsigned long long w = q >= 0 ? *reinterpret_cast<volatile unsigned long long*>(tile_state + q) : kInc;
        if (__any_sync(0xFFFFFFFFu, (w >> 62) == 0ull)) continue;   // a predecessor has not published yet
        const unsigned inc = __ballot_sync(0xFFFFFFFFu, (w >> 62) == 2ull);
        const int stop = inc ? __ffs(inc) - 1 : 31;                 // nearest inclusive prefix
        unsigned long long v = lane <= stop ? (w & kValMask) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        excl += v;
        if (inc) break;
        p -= 32;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(tile_state + tl, kInc | (excl + tot));
      }
    }
    if (lane == 0) {
      s_excl = excl;
      if (tl == nt - 1) *count = excl + tot;
    }
  }
  __syncthreads();
  uint64_t pos = s_excl + pre;
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
  const size_t starts = ((size_t)world * (nt + 1) + 2 * (size_t)world + 1) / 2 * 2;   // + ranges; 8-B aligned
  return starts * sizeof(uint32_t) + (size_t)nt * sizeof(unsigned long long);
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
  const size_t starts = ((size_t)world * (nt + 1) + 2 * (size_t)world + 1) / 2 * 2;
  uint32_t* ranges = start + (size_t)world * (nt + 1);
  unsigned long long* tile_state = reinterpret_cast<unsigned long long*>(start + starts);
  int h;
  prof_begin(c, "union", s, &h);
  cudaError_t e = launch_tile_window(gathered, world, K, kMergeTileShift, (uint32_t)t0, (uint32_t)(t0 + nt), start,
                                     ranges, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(tile_state, 0, (size_t)nt * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const int dm = !mean || world == 1 ? 0 : ((world & (world - 1)) == 0 ? 1 : 2);
  if (dm == 0) union_tile_kernel<0><<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, tile_state, cap, out, count_dev);
  else if (dm == 1) union_tile_kernel<1><<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, tile_state, cap, out, count_dev);
  else union_tile_kernel<2><<<(unsigned)nt, kUWords, 0, s>>>(gathered, world, K, start, nt, t0, lo, hi, tile_state, cap, out, count_dev);
  prof_end(c, h, s);
  c->launches += 3;
  return cudaGetLastError();
}

}  // namespace ld
