// Per-layer top-k compression with error feedback on sm_100a (lowdiff_compress).
//
// What it computes (Alg. 1 line 4 "Comp"; rho = 0.01 sparsification,
// PAPER.md:524; error feedback and per-layer scope from the north star; R-1..R-6):
//   acc = residual + grad; select per layer the k_l largest keys bits(acc) & 0x7FFFFFFF,
//   ties to the lower index; emit index-ascending; residual' = acc with the selection zeroed.
//
// How:
//   small layers (n <= 16384): one CTA per layer, acc staged in shared memory, 3-digit MSB
//     radix select (11/11/9 key bits) with shared-memory histograms, ordered emit by block scan.
//   large layers: 16384-element chunks, each cut into four 4096-element sub-tiles and 64
//     "segments" of 256 elements (one per compute warp per sub-tile).
//     scan:    warp-specialised persistent kernel.  A producer warp streams grad and residual
//              sub-tiles into a 3-stage shared-memory ring with 1-D bulk copies
//              (cp.async.bulk + mbarrier expect_tx); 16 compute warps add them (EF), store
//              residual' = acc with 128-bit stores, and compact the candidates key >= tau_l of
//              their segment in index order with warp ballots -- no block-wide barrier on the
//              hot path (segments are independent; their counts go to a table).  tau_l is the
//              speculative band predicted by the previous call; the first radix digit of the
//              candidates is histogrammed in shared memory on the fly.
//     plan:    per layer, if #candidates >= k_l the exact top-k lies inside the candidates
//              (speculation hit); otherwise the layer is "refilled": the same scan kernel
//              re-reads acc with tau = 0, so every element becomes a candidate.  Exactness
//              never depends on the prediction.
//     digits:  two more radix digits over the (small) candidate lists -> exact k-th key T and
//              the number of ties at T to take (lowest indices first).
//     count / layer scan / emit: per-chunk counts of key > T and key == T, per-layer exclusive
//              scans, then a warp per chunk writes its selected entries at their final position
//              (index order = chunk, segment, in-segment order) and zeroes residual' there.
//   HBM traffic in the steady state: 12 B/param (+ ~0.2 B/param of candidates) + 8 B/entry.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace ld {
namespace {

constexpr int kH0 = 2048, kH1 = 2048, kH2 = 512;   // digit sizes: key bits [30:20] [19:9] [8:0]
constexpr int kHistRow = kH0 + kH1 + kH2;

constexpr int kSub = 4096;                          // elements per sub-tile (16 KB per operand)
constexpr int kWsWarps = 16;                        // compute warps of the scan kernel
constexpr int kWsThreads = (kWsWarps + 1) * 32;     // + one producer warp
constexpr int kStages = 3;                          // shared-memory ring depth
static_assert(kSub / kWsWarps == kSeg, "one segment per compute warp per sub-tile");
static_assert(kChunk / kSeg == kSegsPerChunk, "segment table shape");

__device__ __forceinline__ void st_stream(float* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float f4get(const float4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}
__device__ __forceinline__ void f4set(float4& v, int q, float x) {
  if (q == 0) v.x = x; else if (q == 1) v.y = x; else if (q == 2) v.z = x; else v.w = x;
}
__device__ __forceinline__ uint32_t key_of(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LD_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LD_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on an mbarrier; L2 evict_first (streamed once)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(0x12F0000000000000ull)
      : "memory");
}
__device__ __forceinline__ void compute_bar() {   // named barrier over the 16 compute warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kWsWarps * 32) : "memory");
}

// Warp-cooperative search of the radix bin that holds the kleft-th largest key among the
// entries counted in h[0..nb) (bins ordered by key).  Returns the bin and the number of
// entries in strictly higher bins.  All 32 lanes call it; nb is a multiple of 32.
__device__ __forceinline__ void warp_find_bin(const uint32_t* h, int nb, uint32_t kleft,
                                              uint32_t* bin_out, uint32_t* above_out) {
  const int lane = threadIdx.x & 31;
  const int w = nb / 32;
  const int top = nb - lane * w;                 // lane 0 owns the highest bins
  uint32_t s = 0;
  for (int b = top - 1; b >= top - w; --b) s += h[b];
  uint32_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  const uint32_t exc = inc - s;
  const bool mine = exc < kleft && kleft <= inc;
  const unsigned who = __ballot_sync(0xFFFFFFFFu, mine);
  const int src = who ? __ffs(who) - 1 : 31;
  uint32_t bin = 0, above = 0;
  if (lane == src) {
    uint32_t run = exc;
    bin = (uint32_t)(top - w);
    for (int b = top - 1; b >= top - w; --b) {
      if (run + h[b] >= kleft) { bin = (uint32_t)b; break; }
      run += h[b];
    }
    above = run;
  }
  *bin_out = __shfl_sync(0xFFFFFFFFu, bin, src);
  *above_out = __shfl_sync(0xFFFFFFFFu, above, src);
}

// Block-wide exclusive scan of one value per thread (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* sh32, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh32[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t v = lane < nw ? sh32[lane] : 0, vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, vi, o);
      if (lane >= o) vi += y;
    }
    if (lane < nw) sh32[lane] = vi - v;
    if (lane == 31) sh32[32] = vi;
  }
  __syncthreads();
  const uint32_t r = sh32[wid] + inc - x;
  *total = sh32[32];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- segment tables
// The candidates of chunk ch live in 64 segments of 256 slots; segment s holds its cnt[s]
// candidates, index-ascending, at cand[(ch*64 + s)*256 ...].  A warp loads the 64 counts,
// scans them into so[0..64] (so[64] = chunk total) and addresses candidate c of the chunk as
// segment s = max{s : so[s] <= c}, slot c - so[s].
__device__ __forceinline__ uint32_t warp_load_segs(const DevPlan& P, int ch, uint32_t* so) {
  const int lane = threadIdx.x & 31;
  const uint16_t* cnt = P.seg_count + (uint64_t)ch * kSegsPerChunk;
  const uint32_t c0 = cnt[lane], c1 = cnt[32 + lane];
  uint32_t i0 = c0, i1 = c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, i0, o), y1 = __shfl_up_sync(0xFFFFFFFFu, i1, o);
    if (lane >= o) { i0 += y0; i1 += y1; }
  }
  const uint32_t t0 = __shfl_sync(0xFFFFFFFFu, i0, 31);
  so[lane] = i0 - c0;
  so[32 + lane] = t0 + i1 - c1;
  const uint32_t total = t0 + __shfl_sync(0xFFFFFFFFu, i1, 31);
  if (lane == 0) so[64] = total;
  __syncwarp();
  return total;
}
__device__ __forceinline__ uint64_t seg_addr(int ch, const uint32_t* so, uint32_t c) {
  int s = 0;
#pragma unroll
  for (int step = 32; step; step >>= 1)
    if (so[s + step] <= c) s += step;
  return ((uint64_t)ch * kSegsPerChunk + s) * kSeg + (c - so[s]);
}

// ---------------------------------------------------------------- small layers
template <bool EF>
__global__ void __launch_bounds__(kSmallThreads)
small_layer_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r,
                   uint32_t* __restrict__ send, uint64_t K) {
  extern __shared__ uint32_t sm[];
  uint32_t* acc = sm;                 // [kSmallMax] acc bits
  uint32_t* hist = sm + kSmallMax;    // [2048]
  __shared__ uint32_t sh32[33];
  __shared__ uint32_t s_prefix, s_kleft;
  const int li = P.small_layers[blockIdx.x];
  const uint64_t off = P.layer_off[li];
  const int n = (int)(P.layer_off[li + 1] - off);
  const uint32_t k = P.layer_k[li];
  const uint64_t koff = P.layer_koff[li];
  const int tid = threadIdx.x;

  bool bad = false;
  for (int i = tid; i < n; i += kSmallThreads) {
    float a = EF ? __fadd_rn(r[off + i], g[off + i]) : g[off + i];
    uint32_t u = __float_as_uint(a);
    bad |= (u & 0x7F800000u) == 0x7F800000u;
    acc[i] = u;
  }
  if (bad) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)li); }
  if (tid == 0) { s_prefix = 0; s_kleft = k; }

  const int shifts[3] = {20, 9, 0};
  const int bits[3] = {11, 11, 9};
#pragma unroll 1
  for (int d = 0; d < 3; ++d) {
    const int nb = 1 << bits[d];
    for (int b = tid; b < nb; b += kSmallThreads) hist[b] = 0;
    __syncthreads();
    const uint32_t pre = s_prefix;
    const int hs = shifts[d] + bits[d];
    for (int i = tid; i < n; i += kSmallThreads) {
      const uint32_t key = acc[i] & 0x7FFFFFFFu;
      if ((key >> hs) == pre) atomicAdd(&hist[(key >> shifts[d]) & (nb - 1)], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      uint32_t bin, above;
      warp_find_bin(hist, nb, s_kleft, &bin, &above);
      if (tid == 0) { s_prefix = (pre << bits[d]) | bin; s_kleft -= above; }
    }
    __syncthreads();
  }
  const uint32_t T = s_prefix, need = s_kleft;

  // ordered emit: thread t owns the contiguous run [t*E, t*E+E)
  const int E = (n + kSmallThreads - 1) / kSmallThreads;
  const int b0 = min(n, tid * E), b1 = min(n, b0 + E);
  uint32_t eq = 0;
  for (int i = b0; i < b1; ++i) eq += (acc[i] & 0x7FFFFFFFu) == T;
  uint32_t tot;
  uint32_t eq_before = block_excl_scan(eq, sh32, &tot);
  uint32_t cnt = 0, e_run = eq_before;
  for (int i = b0; i < b1; ++i) {
    const uint32_t key = acc[i] & 0x7FFFFFFFu;
    const bool take = key > T || (key == T && e_run < need);
    e_run += key == T;
    cnt += take;
  }
  uint32_t out_before = block_excl_scan(cnt, sh32, &tot);
  e_run = eq_before;
  uint32_t pos = (uint32_t)koff + out_before;
  for (int i = b0; i < b1; ++i) {
    const uint32_t key = acc[i] & 0x7FFFFFFFu;
    const bool take = key > T || (key == T && e_run < need);
    e_run += key == T;
    if (take) {
      send[pos] = (uint32_t)(off + i);
      send[K + pos] = acc[i];
      ++pos;
      acc[i] = 0u;   // +0.0f in residual'
    }
  }
  if (EF) {
    __syncthreads();
    for (int i = tid; i < n; i += kSmallThreads) r[off + i] = __uint_as_float(acc[i]);
  }
}

// ---------------------------------------------------------------- large layers: warp-specialised scan
// REFILL = false: all chunks, acc = r + g, residual' = acc stored, candidates key >= thr[layer].
// REFILL = true : the chunks in refill_list (count in counters[0]); acc re-read (r when EF, else g),
//                 nothing stored but the candidates, thr = 0 (every element is a candidate).
template <bool EF, bool REFILL>
__global__ void __launch_bounds__(kWsThreads, 2)
scan_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r, uint64_t psi) {
  constexpr bool TWO = EF && !REFILL;             // grad and residual both streamed
  extern __shared__ __align__(128) uint8_t dsm[];
  float* sA = reinterpret_cast<float*>(dsm);      // [kStages][kSub]  grad (or acc when REFILL)
  float* sB = sA + kStages * kSub;                // [kStages][kSub]  residual (TWO only)
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t sh_hist[kH0];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t n_work = REFILL ? P.counters[0] : (uint32_t)P.n_chunks;
  if (blockIdx.x >= n_work) return;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], kWsWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int b = tid; b < kH0; b += kWsThreads) sh_hist[b] = 0;
  __syncthreads();
  const float* srcA = REFILL ? (EF ? r : g) : g;

  if (warp == kWsWarps) {   // ------------------------------------------------ producer warp
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int ch = REFILL ? (int)P.refill_list[w] : (int)w;
        const uint64_t hi = P.chunk_hi[ch];
        for (uint64_t sb = P.chunk_base[ch]; sb < hi; sb += kSub, ++it) {
          const int st = (int)(it % kStages);
          mbar_wait(&empty[st], ((it / kStages) & 1u) ^ 1u);
          uint64_t ve = (min(sb + kSub, hi) + 3) & ~3ull;   // whole float4 slots ...
          if (ve > psi) ve = psi & ~3ull;                     // ... inside the caller's buffer
          const uint32_t bytes = ve > sb ? (uint32_t)((ve - sb) * 4) : 0u;
          mbar_arrive_expect_tx(&full[st], bytes * (TWO ? 2u : 1u));
          if (bytes) {
            bulk_g2s(sA + st * kSub, srcA + sb, bytes, &full[st]);
            if (TWO) bulk_g2s(sB + st * kSub, r + sb, bytes, &full[st]);
          }
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------------- compute warps
  const unsigned lt = (1u << lane) - 1u;
  uint32_t it = 0;
  int cur_slot = -1;
  uint32_t thr = 0;
  for (uint32_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int ch = REFILL ? (int)P.refill_list[w] : (int)w;
    const int slot = P.chunk_slot[ch];
    if (slot != cur_slot) {   // flush the digit-0 histogram of the previous layer
      if (cur_slot >= 0) {
        compute_bar();
        uint32_t* hrow = P.hist + (uint64_t)cur_slot * kHistRow;
        for (int b = tid; b < kH0; b += kWsWarps * 32) {
          const uint32_t h = sh_hist[b];
          if (h) { atomicAdd(&hrow[b], h); sh_hist[b] = 0; }
        }
        compute_bar();
      }
      cur_slot = slot;
      thr = REFILL ? 0u : P.thr[slot];
    }
    const uint64_t lo = P.chunk_lo[ch], hi = P.chunk_hi[ch];
    uint16_t* segc = P.seg_count + (uint64_t)ch * kSegsPerChunk;
    int sub = 0;
    for (uint64_t sb = P.chunk_base[ch]; sb < hi; sb += kSub, ++it, ++sub) {
      const int st = (int)(it % kStages);
      mbar_wait(&full[st], (it / kStages) & 1u);
      const float4* tA = reinterpret_cast<const float4*>(sA + st * kSub);
      const float4* tB = reinterpret_cast<const float4*>(sB + st * kSub);
      float4 a[2];
      uint32_t f[2];
      bool bad = false;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = warp * (kSeg / 4) + j * 32 + lane;   // float4 slot inside the sub-tile
        const uint64_t e0 = sb + 4ull * q;
        uint32_t vm = 0;
        if (e0 >= lo && e0 + 4 <= hi) vm = 0xF;
        else if (e0 + 4 > lo && e0 < hi)
          for (int k = 0; k < 4; ++k) vm |= (e0 + k >= lo && e0 + k < hi) ? 1u << k : 0u;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (vm) {
          if (e0 + 4 <= psi) {
            const float4 av = tA[q];
            if (TWO) {
              const float4 rv = tB[q];
              x = make_float4(__fadd_rn(rv.x, av.x), __fadd_rn(rv.y, av.y), __fadd_rn(rv.z, av.z),
                              __fadd_rn(rv.w, av.w));
            } else {
              x = av;
            }
          } else {   // the buffer's last partial float4 was not bulk-copied
            for (int k = 0; k < 4; ++k)
              if ((vm >> k) & 1u) {
                float y;
                if (REFILL) y = EF ? r[e0 + k] : g[e0 + k];
                else y = EF ? __fadd_rn(r[e0 + k], g[e0 + k]) : g[e0 + k];
                f4set(x, k, y);
              }
          }
          if (TWO) {
            if (vm == 0xF) st_stream(r + e0, x);
            else
              for (int k = 0; k < 4; ++k)
                if ((vm >> k) & 1u) r[e0 + k] = f4get(x, k);
          }
        }
        uint32_t fl = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t key = key_of(f4get(x, k));
          const bool v = (vm >> k) & 1u;
          bad |= v && key >= 0x7F800000u;
          if (v && key >= thr) { fl |= 1u << k; atomicAdd(&sh_hist[key >> 20], 1u); }
        }
        f[j] = fl;
        a[j] = x;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);   // this warp is done with the stage
      if (bad) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)P.large_layers[slot]); }
      // ordered compaction of the warp's segment: elements in (j, lane, k) order = index order
      const int seg = sub * kWsWarps + warp;
      uint32_t* cidx = P.cand_idx + ((uint64_t)ch * kSegsPerChunk + seg) * kSeg;
      uint32_t* cval = P.cand_val + ((uint64_t)ch * kSegsPerChunk + seg) * kSeg;
      uint32_t run = 0;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t fl = f[j];
        unsigned bm[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) bm[k] = __ballot_sync(0xFFFFFFFFu, (fl >> k) & 1u);
        uint32_t pos = run;
#pragma unroll
        for (int k = 0; k < 4; ++k) pos += __popc(bm[k] & lt);
        if (fl) {
          const uint64_t e0 = sb + 4ull * (warp * (kSeg / 4) + j * 32 + lane);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if ((fl >> k) & 1u) { cidx[pos] = (uint32_t)(e0 + k); cval[pos] = __float_as_uint(f4get(a[j], k)); ++pos; }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) run += __popc(bm[k]);
      }
      if (lane == 0) segc[seg] = (uint16_t)run;
    }
    if (lane == 0)
      for (int s2 = sub; s2 < kSegsPerChunk / kWsWarps; ++s2) segc[s2 * kWsWarps + warp] = 0;
  }
  if (cur_slot >= 0) {
    compute_bar();
    uint32_t* hrow = P.hist + (uint64_t)cur_slot * kHistRow;
    for (int b = tid; b < kH0; b += kWsWarps * 32)
      if (sh_hist[b]) atomicAdd(&hrow[b], sh_hist[b]);
  }
}

// per chunk: candidate total (sum of its 64 segment counts); warp per chunk
__global__ void chunk_total_kernel(DevPlan P) {
  __shared__ uint32_t so_all[8][kSegsPerChunk + 1];
  const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ch >= P.n_chunks) return;
  const uint32_t tot = warp_load_segs(P, ch, so_all[threadIdx.x >> 5]);
  if ((threadIdx.x & 31) == 0) P.chunk_count[ch] = tot;
}

// ---------------------------------------------------------------- per-layer plan / digit search
// mode 0: after scan -- decide hit/refill, find digit 0 for hits, queue refills
// mode 1: after rescan -- find digit 0 for refilled layers
// mode 2/3: find digit 1/2 for every large layer (mode 2 also predicts the next band)
__global__ void find_kernel(DevPlan P, int mode) {
  const int slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slot >= P.n_large) return;
  const int li = P.large_layers[slot];
  const uint32_t k = P.layer_k[li];
  LayerSel& S = P.sel[slot];
  uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
  if (mode == 0) {
    const int c0 = P.large_chunk0[slot], c1 = P.large_chunk0[slot + 1];
    uint32_t tot = 0;
    for (int c = c0 + lane; c < c1; c += 32) tot += P.chunk_count[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
    if (tot >= k) {
      uint32_t bin, above;
      warp_find_bin(hrow, kH0, k, &bin, &above);
      if (lane == 0) {
        S.prefix = bin; S.kleft = k - above; S.total = tot; S.refill = 0;
        // adapt the band: the previous call chose it to admit `band` x k keys of ITS distribution;
        // under error feedback the accumulated values drift upward between calls, so the band
        // admitted tot / k x k now.  Aim the next band at 1.5 k_l admitted.
        const float b = S.band > 0.f ? S.band : 1.5f;
        S.band = fminf(4.f, fmaxf(1.02f, b * 1.5f * (float)k / (float)tot));
        atomicAdd(&P.counters[1], 1u);
        atomicAdd(&P.counters[3], tot);
      }
    } else {
      for (int b = lane; b < kH0; b += 32) hrow[b] = 0;
      uint32_t base = 0;
      if (lane == 0) {
        base = atomicAdd(&P.counters[0], (uint32_t)(c1 - c0));
        S.refill = 1;
        S.total = (uint32_t)(P.layer_off[li + 1] - P.layer_off[li]);
        S.band = S.band > 0.f ? fminf(4.f, S.band * 2.f) : 1.5f;   // missed: widen
        atomicAdd(&P.counters[2], 1u);
      }
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      for (int c = c0 + lane; c < c1; c += 32) P.refill_list[base + (c - c0)] = (uint32_t)c;
    }
  } else if (mode == 1) {
    if (!S.refill) return;
    uint32_t bin, above;
    warp_find_bin(hrow, kH0, k, &bin, &above);
    if (lane == 0) { S.prefix = bin; S.kleft = k - above; }
  } else {
    const int nb = mode == 2 ? kH1 : kH2;
    const uint32_t* h = hrow + (mode == 2 ? kH0 : kH0 + kH1);
    uint32_t bin, above;
    warp_find_bin(h, nb, S.kleft, &bin, &above);
    if (mode == 2) {
      // Speculative band for the next call: the key with C = band x k_l candidate keys at or above
      // it (digit-0 resolution, refined with the digit-1 histogram when C falls in T's digit-0
      // bin).  Only a prediction -- the next call checks #candidates >= k_l and refills otherwise.
      const float band = S.band > 0.f ? S.band : 1.5f;
      const uint32_t C = max(k + 32u, (uint32_t)fminf((float)k * band, 4.0e9f));
      uint32_t nt = P.thr[slot];
      if (S.total >= C) {
        uint32_t b0, a0;
        warp_find_bin(hrow, kH0, C, &b0, &a0);
        if (b0 == S.prefix) {
          uint32_t b1, a1;
          warp_find_bin(h, nb, C - a0, &b1, &a1);
          nt = (b0 << 20) | (b1 << 9);
        } else {
          nt = b0 << 20;
        }
      }
      if (lane == 0) S.next_thr = nt;
    }
    if (lane == 0) { S.prefix = (S.prefix << (mode == 2 ? 11 : 9)) | bin; S.kleft -= above; }
  }
}

// digit d (1 or 2) histogram over candidates matching the prefix: warp per chunk
__global__ void digit_kernel(DevPlan P, int d) {
  __shared__ uint32_t so_all[8][kSegsPerChunk + 1];
  const int lane = threadIdx.x & 31;
  const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ch >= P.n_chunks) return;
  uint32_t* so = so_all[threadIdx.x >> 5];
  const int shift = d == 1 ? 9 : 0;
  const int hs = d == 1 ? 20 : 9;
  const uint32_t mask = d == 1 ? 0x7FFu : 0x1FFu;
  const int slot = P.chunk_slot[ch];
  const uint32_t pre = P.sel[slot].prefix;
  uint32_t* h = P.hist + (uint64_t)slot * kHistRow + (d == 1 ? kH0 : kH0 + kH1);
  const uint32_t cnt = warp_load_segs(P, ch, so);
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t key = i < cnt ? P.cand_val[seg_addr(ch, so, i)] & 0x7FFFFFFFu : 0u;
    const bool m = i < cnt && (key >> hs) == pre;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, m);
    if (m) {
      const uint32_t bin = (key >> shift) & mask;
      const unsigned peers = __match_any_sync(act, bin);
      if (lane == __ffs(peers) - 1) atomicAdd(&h[bin], (uint32_t)__popc(peers));
    }
  }
}

// per chunk: #(key > T) and #(key == T)
__global__ void count_kernel(DevPlan P) {
  __shared__ uint32_t so_all[8][kSegsPerChunk + 1];
  const int lane = threadIdx.x & 31;
  const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ch >= P.n_chunks) return;
  uint32_t* so = so_all[threadIdx.x >> 5];
  const uint32_t T = P.sel[P.chunk_slot[ch]].prefix;
  const uint32_t cnt = warp_load_segs(P, ch, so);
  uint32_t gt = 0, eq = 0;
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint32_t key = P.cand_val[seg_addr(ch, so, i)] & 0x7FFFFFFFu;
    gt += key > T;
    eq += key == T;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    gt += __shfl_xor_sync(0xFFFFFFFFu, gt, o);
    eq += __shfl_xor_sync(0xFFFFFFFFu, eq, o);
  }
  if (lane == 0) { P.chunk_gt[ch] = gt; P.chunk_eq[ch] = eq; }
}

// per large layer (one CTA): exclusive scans over its chunks; next speculative threshold
__global__ void __launch_bounds__(256) layer_scan_kernel(DevPlan P) {
  __shared__ uint32_t sh32[33];
  const int slot = blockIdx.x;
  const int c0 = P.large_chunk0[slot], c1 = P.large_chunk0[slot + 1];
  const uint32_t T = P.sel[slot].prefix, need = P.sel[slot].kleft;
  uint32_t eq_carry = 0, out_carry = 0;
  for (int cb = c0; cb < c1; cb += 256) {
    const int c = cb + threadIdx.x;
    const uint32_t eq = c < c1 ? P.chunk_eq[c] : 0, gt = c < c1 ? P.chunk_gt[c] : 0;
    uint32_t tot;
    const uint32_t eb = eq_carry + block_excl_scan(eq, sh32, &tot);
    eq_carry += tot;
    const uint32_t take = eb >= need ? 0u : min(eq, need - eb);
    const uint32_t o = gt + take;
    const uint32_t ob = out_carry + block_excl_scan(o, sh32, &tot);
    out_carry += tot;
    if (c < c1) { P.chunk_out[c] = ob; P.chunk_take[c] = take; }
  }
  if (threadIdx.x == 0) {
    // speculative band for the next call, never above this call's T
    const uint32_t nt = P.sel[slot].next_thr;
    P.thr[slot] = nt <= T ? nt : T;
  }
}

// warp per chunk: ordered emit of the selected candidates, residual' zeroing
template <bool EF>
__global__ void emit_kernel(DevPlan P, uint32_t* __restrict__ send, uint64_t K, float* __restrict__ r) {
  __shared__ uint32_t so_all[8][kSegsPerChunk + 1];
  const int lane = threadIdx.x & 31;
  const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ch >= P.n_chunks) return;
  uint32_t* so = so_all[threadIdx.x >> 5];
  const unsigned lt = (1u << lane) - 1u;
  const int slot = P.chunk_slot[ch];
  const uint32_t T = P.sel[slot].prefix;
  const uint32_t take = P.chunk_take[ch];
  const uint64_t dst0 = P.layer_koff[P.large_layers[slot]] + P.chunk_out[ch];
  const uint32_t cnt = warp_load_segs(P, ch, so);
  uint32_t eq_run = 0, out_run = 0;
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool v = i < cnt;
    const uint64_t a = v ? seg_addr(ch, so, i) : 0;
    const uint32_t val = v ? P.cand_val[a] : 0u;
    const uint32_t idx = v ? P.cand_idx[a] : 0u;
    const uint32_t key = val & 0x7FFFFFFFu;
    const bool is_eq = v && key == T;
    const unsigned eqm = __ballot_sync(0xFFFFFFFFu, is_eq);
    const bool sel = v && (key > T || (is_eq && eq_run + __popc(eqm & lt) < take));
    const unsigned sm = __ballot_sync(0xFFFFFFFFu, sel);
    if (sel) {
      const uint64_t o = dst0 + out_run + __popc(sm & lt);
      send[o] = idx;
      send[K + o] = val;
      if (EF) r[idx] = 0.0f;
    }
    eq_run += __popc(eqm);
    out_run += __popc(sm);
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <bool EF, bool REFILL>
cudaError_t launch_scan(const DevPlan& P, int grid, const float* g, float* r, uint64_t psi, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = (size_t)kStages * kSub * sizeof(float) * 2;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(scan_kernel<EF, REFILL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  scan_kernel<EF, REFILL><<<grid, kWsThreads, smem, s>>>(P, g, r, psi);
  return cudaSuccess;
}

}  // namespace

size_t compress_hist_bytes(int n_large) { return (size_t)n_large * kHistRow * sizeof(uint32_t); }

cudaError_t launch_compress(lowdiff_ctx* c, const float* grad, float* residual, uint32_t* send,
                            cudaStream_t s) {
  DevPlan& P = c->plan;
  const bool ef = c->cfg.error_feedback != 0;
  int h;
  cudaError_t e;
  if (P.n_small) {
    static bool attr_set[2] = {false, false};
    const size_t smem = (size_t)(kSmallMax + 2048) * sizeof(uint32_t);
    if (!attr_set[ef]) {
      e = ef ? cudaFuncSetAttribute(small_layer_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
             : cudaFuncSetAttribute(small_layer_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr_set[ef] = true;
    }
    prof_begin(c, "small_layer", s, &h);
    if (ef) small_layer_kernel<true><<<P.n_small, kSmallThreads, smem, s>>>(P, grad, residual, send, (uint64_t)c->K);
    else small_layer_kernel<false><<<P.n_small, kSmallThreads, smem, s>>>(P, grad, residual, send, (uint64_t)c->K);
    prof_end(c, h, s);
    c->launches += 1;
  }
  if (!P.n_large) return cudaGetLastError();
  e = cudaMemsetAsync(P.hist, 0, compress_hist_bytes(P.n_large), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(P.counters, 0, 4 * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int sms = num_sms();
  const int layer_blocks = (P.n_large * 32 + 255) / 256;     // warp per large layer
  const int chunk_blocks = (P.n_chunks + 7) / 8;              // warp per chunk
  const int scan_grid = std::min(P.n_chunks, sms * 2);        // persistent: 2 CTAs per SM

  prof_begin(c, "scan", s, &h);
  e = ef ? launch_scan<true, false>(P, scan_grid, grad, residual, (uint64_t)c->psi, s)
         : launch_scan<false, false>(P, scan_grid, grad, residual, (uint64_t)c->psi, s);
  if (e != cudaSuccess) return e;
  prof_end(c, h, s);
  prof_begin(c, "select", s, &h);
  chunk_total_kernel<<<chunk_blocks, 256, 0, s>>>(P);
  find_kernel<<<layer_blocks, 256, 0, s>>>(P, 0);
  e = ef ? launch_scan<true, true>(P, sms * 2, grad, residual, (uint64_t)c->psi, s)
         : launch_scan<false, true>(P, sms * 2, grad, residual, (uint64_t)c->psi, s);
  if (e != cudaSuccess) return e;
  find_kernel<<<layer_blocks, 256, 0, s>>>(P, 1);
  digit_kernel<<<chunk_blocks, 256, 0, s>>>(P, 1);
  find_kernel<<<layer_blocks, 256, 0, s>>>(P, 2);
  digit_kernel<<<chunk_blocks, 256, 0, s>>>(P, 2);
  find_kernel<<<layer_blocks, 256, 0, s>>>(P, 3);
  count_kernel<<<chunk_blocks, 256, 0, s>>>(P);
  layer_scan_kernel<<<P.n_large, 256, 0, s>>>(P);
  prof_end(c, h, s);
  prof_begin(c, "emit", s, &h);
  if (ef) emit_kernel<true><<<chunk_blocks, 256, 0, s>>>(P, send, (uint64_t)c->K, residual);
  else emit_kernel<false><<<chunk_blocks, 256, 0, s>>>(P, send, (uint64_t)c->K, residual);
  prof_end(c, h, s);
  c->launches += 12;
  return cudaGetLastError();
}

}  // namespace ld
