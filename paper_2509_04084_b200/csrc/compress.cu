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
//   large layers: 16384-element chunks, one 512-thread CTA each.
//     scan:    128-bit streaming loads of grad and residual, EF add, residual' = acc
//              (128-bit stores), and an ORDER-PRESERVING compaction of the candidates
//              key >= tau_l (tau_l = 0.98 x the layer's previous k-th key) into the chunk's
//              slot of a candidate buffer, with the first radix digit histogrammed on the fly.
//     plan:    per layer, if #candidates >= k_l the exact top-k lies inside the candidates
//              (speculation hit); else the layer is "refilled": every element becomes a
//              candidate (rescan).  Exactness never depends on the prediction.
//     digits:  two more radix digits over the (small) candidate lists -> exact k-th key T
//              and the number of ties at T to take.
//     count/scan/emit: per-chunk counts of key > T and key == T, per-layer exclusive scans,
//              then a warp per chunk writes its selected entries at their final position
//              (index order is chunk order, then in-chunk order) and zeroes residual'.
//   HBM traffic in the steady state: 12 B/param (+ ~0.13 B/param of candidates) + 8 B/entry.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace ld {
namespace {

constexpr int kH0 = 2048, kH1 = 2048, kH2 = 512;   // digit sizes: key bits [30:20] [19:9] [8:0]
constexpr int kHistRow = kH0 + kH1 + kH2;

__device__ __forceinline__ float4 ld_stream(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_rw(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
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

// ---------------------------------------------------------------- large layers: scan
template <bool EF, bool REFILL>
__device__ __forceinline__ void scan_chunk(const DevPlan& P, int ch, const float* __restrict__ g,
                                           float* __restrict__ r, uint32_t* sh_hist, uint32_t* sh_tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = P.chunk_slot[ch];
  const uint64_t base = P.chunk_base[ch], lo = P.chunk_lo[ch], hi = P.chunk_hi[ch];
  const uint32_t thr = REFILL ? 0u : P.thr[slot];
  for (int b = tid; b < kH0; b += kScanThreads) sh_hist[b] = 0;

  float4 a[8];
  uint32_t vmask = 0;   // bit 4j+q: element q of slot j belongs to the chunk
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint64_t e0 = base + 4ull * (uint64_t)(j * kScanThreads + tid);
    a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 >= lo && e0 + 4 <= hi) {
      vmask |= 0xFu << (4 * j);
      if (REFILL) {
        a[j] = EF ? ld_rw(r + e0) : ld_stream(g + e0);
      } else {
        const float4 gv = ld_stream(g + e0);
        if (EF) {
          const float4 rv = ld_rw(r + e0);
          a[j] = make_float4(__fadd_rn(rv.x, gv.x), __fadd_rn(rv.y, gv.y), __fadd_rn(rv.z, gv.z),
                             __fadd_rn(rv.w, gv.w));
        } else {
          a[j] = gv;
        }
      }
    } else if (e0 + 4 > lo && e0 < hi) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t e = e0 + q;
        if (e >= lo && e < hi) {
          vmask |= 1u << (4 * j + q);
          float x;
          if (REFILL) x = EF ? r[e] : g[e];
          else x = EF ? __fadd_rn(r[e], g[e]) : g[e];
          f4set(a[j], q, x);
        }
      }
    }
  }
  if (EF && !REFILL) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t e0 = base + 4ull * (uint64_t)(j * kScanThreads + tid);
      const uint32_t vj = (vmask >> (4 * j)) & 0xFu;
      if (vj == 0xF) {
        st_stream(r + e0, a[j]);
      } else if (vj) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (vj & (1u << q)) r[e0 + q] = f4get(a[j], q);
      }
    }
  }
  __syncthreads();   // histogram zeroed

  // candidate flags, digit-0 histogram, per-(j, warp) counts
  uint32_t fmask = 0;   // bit 4j+q: candidate
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t f = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t key = key_of(f4get(a[j], q));
      const bool v = (vmask >> (4 * j + q)) & 1u;
      bad |= v && key >= 0x7F800000u;
      if (v && key >= thr) {
        f |= 1u << q;
        atomicAdd(&sh_hist[key >> 20], 1u);
      }
    }
    fmask |= f << (4 * j);
    uint32_t tot = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) tot += __popc(__ballot_sync(0xFFFFFFFFu, (f >> q) & 1u));
    if (lane == 0) sh_tot[j * (kScanThreads / 32) + warp] = tot;
  }
  if (bad) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)P.large_layers[slot]); }
  __syncthreads();
  // exclusive scan of the 8 x 16 segment counts in (j, warp) order: one warp, 4 per lane
  if (warp == 0) {
    uint32_t v[4], s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) { v[q] = sh_tot[lane * 4 + q]; s += v[q]; }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += y;
    }
    uint32_t run = inc - s;
#pragma unroll
    for (int q = 0; q < 4; ++q) { sh_tot[lane * 4 + q] = run; run += v[q]; }
    if (lane == 31) sh_tot[128] = inc;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  uint32_t* cidx = P.cand_idx + (uint64_t)ch * kChunk;
  uint32_t* cval = P.cand_val + (uint64_t)ch * kChunk;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t f = (fmask >> (4 * j)) & 0xFu;
    uint32_t pos = sh_tot[j * (kScanThreads / 32) + warp];
#pragma unroll
    for (int q = 0; q < 4; ++q) pos += __popc(__ballot_sync(0xFFFFFFFFu, (f >> q) & 1u) & lt);
    if (f) {
      const uint64_t e0 = base + 4ull * (uint64_t)(j * kScanThreads + tid);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((f >> q) & 1u) {
          cidx[pos] = (uint32_t)(e0 + q);
          cval[pos] = __float_as_uint(f4get(a[j], q));
          ++pos;
        }
      }
    }
  }
  if (tid == 0) P.chunk_count[ch] = sh_tot[128];
  uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
  for (int b = tid; b < kH0; b += kScanThreads)
    if (sh_hist[b]) atomicAdd(&hrow[b], sh_hist[b]);
}

// ---------------------------------------------------------------- large layers: TMA-pipelined scan
// Persistent CTAs (2 per SM) stream their chunks through a 3-stage shared-memory ring filled by
// 1-D bulk tensor copies (cp.async.bulk, completion on an mbarrier with expect_tx), so the next
// sub-tiles are already in flight while the current one is added, stored and compacted.
constexpr int kSub = 4096;                  // elements per sub-tile (16 KB per operand)
constexpr int kStages = 3;
constexpr int kSlotsPerThread = kSub / 4 / kScanThreads;   // 2 float4 slots per thread per sub-tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(0x12F0000000000000ull)  // evict_first
      : "memory");
}

struct SubTile {
  int ch;          // chunk id (-1: none)
  int sub;         // sub-tile within the chunk
};

__device__ __forceinline__ bool next_sub(const DevPlan& P, SubTile& s) {
  // advance (ch, sub) over this CTA's chunks: ch = blockIdx.x + i * gridDim.x
  const uint64_t span = P.chunk_hi[s.ch] - P.chunk_base[s.ch];
  if ((uint64_t)(s.sub + 1) * kSub < span) { ++s.sub; return true; }
  s.ch += gridDim.x;
  s.sub = 0;
  return s.ch < P.n_chunks;
}

// issue the bulk copies of one sub-tile into stage st (thread 0 only)
template <bool EF>
__device__ __forceinline__ void issue_sub(const DevPlan& P, const SubTile& s, int st, float* sg, float* sr,
                                          uint64_t* full, const float* g, const float* r, uint64_t psi) {
  const uint64_t sb = P.chunk_base[s.ch] + (uint64_t)s.sub * kSub;
  const uint64_t se = min(sb + kSub, P.chunk_hi[s.ch]);
  uint64_t ve = (se + 3) & ~3ull;           // whole float4 slots ...
  if (ve > psi) ve = psi & ~3ull;           // ... that lie inside the caller's buffer
  const uint32_t bytes = ve > sb ? (uint32_t)((ve - sb) * 4) : 0u;
  mbar_arrive_expect_tx(&full[st], bytes * (EF ? 2u : 1u));
  if (bytes) {
    bulk_g2s(sg + st * kSub, g + sb, bytes, &full[st]);
    if (EF) bulk_g2s(sr + st * kSub, r + sb, bytes, &full[st]);
  }
}

template <bool EF>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_tma_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r, uint64_t psi) {
  extern __shared__ __align__(128) uint8_t dsm[];
  float* sg = reinterpret_cast<float*>(dsm);                 // [kStages][kSub]
  float* sr = sg + kStages * kSub;                           // [kStages][kSub] (EF)
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ uint32_t sh_hist[kH0];
  __shared__ uint32_t sh_tot[2 * (kScanThreads / 32) + 1];
  __shared__ uint32_t s_run;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if ((int)blockIdx.x >= P.n_chunks) return;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int b = tid; b < kH0; b += kScanThreads) sh_hist[b] = 0;
  if (tid == 0) s_run = 0;
  __syncthreads();
  SubTile prod{(int)blockIdx.x, 0};
  bool prod_ok = true;
  if (tid == 0) {
    for (int st = 0; st < kStages && prod_ok; ++st) {
      issue_sub<EF>(P, prod, st, sg, sr, full, g, r, psi);
      prod_ok = next_sub(P, prod);
    }
  }
  SubTile cur{(int)blockIdx.x, 0};
  int stage = 0;
  uint32_t phase = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (;;) {
    bool bad = false;
    const int ch = cur.ch;
    const int slot = P.chunk_slot[ch];
    const uint64_t lo = P.chunk_lo[ch], hi = P.chunk_hi[ch];
    const uint64_t sb = P.chunk_base[ch] + (uint64_t)cur.sub * kSub;
    const uint32_t thr = P.thr[slot];
    mbar_wait(&full[stage], phase);
    const float* tg = sg + stage * kSub;
    const float* tr = sr + stage * kSub;
    float4 a[kSlotsPerThread];
    uint32_t f[kSlotsPerThread];
#pragma unroll
    for (int j = 0; j < kSlotsPerThread; ++j) {
      const int q = j * kScanThreads + tid;
      const uint64_t e0 = sb + 4ull * q;
      uint32_t vm = 0;
      if (e0 >= lo && e0 + 4 <= hi) vm = 0xF;
      else if (e0 + 4 > lo && e0 < hi)
        for (int k = 0; k < 4; ++k) vm |= (e0 + k >= lo && e0 + k < hi) ? 1u << k : 0u;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vm) {
        if (e0 + 4 <= psi) {
          const float4 gv = reinterpret_cast<const float4*>(tg)[q];
          if (EF) {
            const float4 rv = reinterpret_cast<const float4*>(tr)[q];
            x = make_float4(__fadd_rn(rv.x, gv.x), __fadd_rn(rv.y, gv.y), __fadd_rn(rv.z, gv.z), __fadd_rn(rv.w, gv.w));
          } else {
            x = gv;
          }
        } else {   // the last partial float4 of the buffer was not bulk-copied
          for (int k = 0; k < 4; ++k)
            if ((vm >> k) & 1u) f4set(x, k, EF ? __fadd_rn(r[e0 + k], g[e0 + k]) : g[e0 + k]);
        }
        if (EF) {
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
      uint32_t tot = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) tot += __popc(__ballot_sync(0xFFFFFFFFu, (fl >> k) & 1u));
      if (lane == 0) sh_tot[j * (kScanThreads / 32) + warp] = tot;
    }
    if (bad) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)P.large_layers[slot]); }
    __syncthreads();   // sh_tot complete; every thread is done reading this stage
    if (tid == 0 && prod_ok) {   // refill the stage just consumed
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_sub<EF>(P, prod, stage, sg, sr, full, g, r, psi);
      prod_ok = next_sub(P, prod);
    }
    if (warp == 0) {
      const int nseg = kSlotsPerThread * (kScanThreads / 32);   // 32 segments: one per lane
      uint32_t v = lane < nseg ? sh_tot[lane] : 0u, inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t base = s_run;
      if (lane < nseg) sh_tot[lane] = base + inc - v;
      if (lane == 31) sh_tot[nseg] = base + inc;
    }
    __syncthreads();
    uint32_t* cidx = P.cand_idx + (uint64_t)ch * kChunk;
    uint32_t* cval = P.cand_val + (uint64_t)ch * kChunk;
#pragma unroll
    for (int j = 0; j < kSlotsPerThread; ++j) {
      const uint32_t fl = f[j];
      uint32_t pos = sh_tot[j * (kScanThreads / 32) + warp];
#pragma unroll
      for (int k = 0; k < 4; ++k) pos += __popc(__ballot_sync(0xFFFFFFFFu, (fl >> k) & 1u) & lt);
      if (fl) {
        const uint64_t e0 = sb + 4ull * (j * kScanThreads + tid);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((fl >> k) & 1u) { cidx[pos] = (uint32_t)(e0 + k); cval[pos] = __float_as_uint(f4get(a[j], k)); ++pos; }
      }
    }
    if (tid == 0) s_run = sh_tot[kSlotsPerThread * (kScanThreads / 32)];
    if (++stage == kStages) { stage = 0; phase ^= 1u; }
    const bool last_sub = (uint64_t)(cur.sub + 1) * kSub >= hi - P.chunk_base[ch];
    if (last_sub) {
      __syncthreads();   // s_run final, histogram complete
      if (tid == 0) P.chunk_count[ch] = s_run;
      uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
      for (int b = tid; b < kH0; b += kScanThreads) {
        const uint32_t h = sh_hist[b];
        if (h) { atomicAdd(&hrow[b], h); sh_hist[b] = 0; }
      }
      if (tid == 0) s_run = 0;
    }
    __syncthreads();
    if (!next_sub(P, cur)) break;
  }
}

template <bool EF>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r) {
  __shared__ uint32_t sh_hist[kH0];
  __shared__ uint32_t sh_tot[8 * (kScanThreads / 32) + 1];
  scan_chunk<EF, false>(P, blockIdx.x, g, r, sh_hist, sh_tot);
}

template <bool EF>
__global__ void __launch_bounds__(kScanThreads, 2)
rescan_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r) {
  __shared__ uint32_t sh_hist[kH0];
  __shared__ uint32_t sh_tot[8 * (kScanThreads / 32) + 1];
  const uint32_t n = P.counters[0];
  for (uint32_t w = blockIdx.x; w < n; w += gridDim.x) {
    scan_chunk<EF, true>(P, (int)P.refill_list[w], g, r, sh_hist, sh_tot);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- per-layer plan / digit search
// mode 0: after scan -- decide hit/refill, find digit 0 for hits, queue refills
// mode 1: after rescan -- find digit 0 for refilled layers
// mode 2/3: find digit 1/2 for every large layer
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
      if (lane == 0) { S.prefix = bin; S.kleft = k - above; S.total = tot; S.refill = 0; atomicAdd(&P.counters[1], 1u); }
    } else {
      for (int b = lane; b < kH0; b += 32) hrow[b] = 0;
      uint32_t base = 0;
      if (lane == 0) {
        base = atomicAdd(&P.counters[0], (uint32_t)(c1 - c0));
        S.refill = 1;
        S.total = (uint32_t)(P.layer_off[li + 1] - P.layer_off[li]);
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
      // Speculative band for the next call: the key with C = 1.5 k_l candidate keys at or above it
      // (digit-0 resolution, refined with the digit-1 histogram when C falls in T's digit-0 bin).
      // Only a prediction -- the next call checks #candidates >= k_l and refills otherwise.
      const uint32_t C = k + max(k / 2, 32u);
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
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int shift = d == 1 ? 9 : 0;
  const int hs = d == 1 ? 20 : 9;
  const uint32_t mask = d == 1 ? 0x7FFu : 0x1FFu;
  const int hoff = d == 1 ? kH0 : kH0 + kH1;
  for (int ch = gw; ch < P.n_chunks; ch += nwarps) {
    const int slot = P.chunk_slot[ch];
    const uint32_t pre = P.sel[slot].prefix;
    const uint32_t cnt = P.chunk_count[ch];
    const uint32_t* cval = P.cand_val + (uint64_t)ch * kChunk;
    uint32_t* h = P.hist + (uint64_t)slot * kHistRow + hoff;
    for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint32_t key = i < cnt ? cval[i] & 0x7FFFFFFFu : 0u;
      const bool m = i < cnt && (key >> hs) == pre;
      const unsigned act = __ballot_sync(0xFFFFFFFFu, m);
      if (m) {
        const uint32_t bin = (key >> shift) & mask;
        const unsigned peers = __match_any_sync(act, bin);
        if (lane == __ffs(peers) - 1) atomicAdd(&h[bin], (uint32_t)__popc(peers));
      }
    }
  }
}

// per chunk: #(key > T) and #(key == T)
__global__ void count_kernel(DevPlan P) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int ch = gw; ch < P.n_chunks; ch += nwarps) {
    const uint32_t T = P.sel[P.chunk_slot[ch]].prefix;
    const uint32_t cnt = P.chunk_count[ch];
    const uint32_t* cval = P.cand_val + (uint64_t)ch * kChunk;
    uint32_t gt = 0, eq = 0;
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t key = cval[i] & 0x7FFFFFFFu;
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
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int ch = gw; ch < P.n_chunks; ch += nwarps) {
    const int slot = P.chunk_slot[ch];
    const uint32_t T = P.sel[slot].prefix;
    const uint32_t take = P.chunk_take[ch];
    const uint64_t dst0 = P.layer_koff[P.large_layers[slot]] + P.chunk_out[ch];
    const uint32_t cnt = P.chunk_count[ch];
    const uint32_t* cidx = P.cand_idx + (uint64_t)ch * kChunk;
    const uint32_t* cval = P.cand_val + (uint64_t)ch * kChunk;
    uint32_t eq_run = 0, out_run = 0;
    for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool v = i < cnt;
      const uint32_t val = v ? cval[i] : 0u;
      const uint32_t key = val & 0x7FFFFFFFu;
      const bool is_eq = v && key == T;
      const unsigned eqm = __ballot_sync(0xFFFFFFFFu, is_eq);
      const bool sel = v && (key > T || (is_eq && eq_run + __popc(eqm & lt) < take));
      const unsigned sm = __ballot_sync(0xFFFFFFFFu, sel);
      if (sel) {
        const uint32_t idx = cidx[i];
        const uint64_t o = dst0 + out_run + __popc(sm & lt);
        send[o] = idx;
        send[K + o] = val;
        if (EF) r[idx] = 0.0f;
      }
      eq_run += __popc(eqm);
      out_run += __popc(sm);
    }
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
  const int warp_blocks = (P.n_large * 32 + 255) / 256;
  const int pgrid = (P.n_chunks + 7) / 8;   // one warp per chunk: latency hidden by parallelism

  {
    static bool tma_attr[2] = {false, false};
    const size_t smem = (size_t)kStages * kSub * sizeof(float) * (ef ? 2 : 1);
    if (!tma_attr[ef]) {
      e = ef ? cudaFuncSetAttribute(scan_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
             : cudaFuncSetAttribute(scan_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      tma_attr[ef] = true;
    }
    const int grid = std::min(P.n_chunks, sms * 2);
    prof_begin(c, "scan", s, &h);
    if (ef) scan_tma_kernel<true><<<grid, kScanThreads, smem, s>>>(P, grad, residual, (uint64_t)c->psi);
    else scan_tma_kernel<false><<<grid, kScanThreads, smem, s>>>(P, grad, residual, (uint64_t)c->psi);
    prof_end(c, h, s);
  }
  prof_begin(c, "select", s, &h);
  find_kernel<<<warp_blocks, 256, 0, s>>>(P, 0);
  if (ef) rescan_kernel<true><<<sms * 2, kScanThreads, 0, s>>>(P, grad, residual);
  else rescan_kernel<false><<<sms * 2, kScanThreads, 0, s>>>(P, grad, residual);
  find_kernel<<<warp_blocks, 256, 0, s>>>(P, 1);
  digit_kernel<<<pgrid, 256, 0, s>>>(P, 1);
  find_kernel<<<warp_blocks, 256, 0, s>>>(P, 2);
  digit_kernel<<<pgrid, 256, 0, s>>>(P, 2);
  find_kernel<<<warp_blocks, 256, 0, s>>>(P, 3);
  count_kernel<<<pgrid, 256, 0, s>>>(P);
  layer_scan_kernel<<<P.n_large, 256, 0, s>>>(P);
  prof_end(c, h, s);
  prof_begin(c, "emit", s, &h);
  if (ef) emit_kernel<true><<<pgrid, 256, 0, s>>>(P, send, (uint64_t)c->K, residual);
  else emit_kernel<false><<<pgrid, 256, 0, s>>>(P, send, (uint64_t)c->K, residual);
  prof_end(c, h, s);
  c->launches += 11;
  return cudaGetLastError();
}

}  // namespace ld
