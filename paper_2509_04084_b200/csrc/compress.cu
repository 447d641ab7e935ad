// Per-layer top-k compression with error feedback on sm_100a (lowdiff_compress).
//
// What it computes (Alg. 1 line 4 "Comp"; rho = 0.01 sparsification,
// PAPER.md:524; error feedback and per-layer scope from the north star; R-1..R-6):
//   acc = residual + grad; select per layer the k_l largest keys bits(acc) & 0x7FFFFFFF,
//   ties to the lower index; emit index-ascending; residual' = acc with the selection zeroed.
//
// How:
//   small layers (n <= kSmallMax = 4096): one CTA per layer, acc staged in shared memory, 3-digit
//     MSB radix select (11/11/9 key bits) with shared-memory histograms, ordered emit by block scan;
//     on a forked stream, concurrent with the scan.
//   large layers: 16384-element chunks = 16 segments of 1024 elements.
//     scan:   a full-grid streaming kernel (one warp per segment, 128-bit loads of grad and residual,
//             128-bit stores of residual' = acc) -- the pattern measured at ~7.1 TB/s for 2 reads + 1
//             write on this GPU (tools/stream_probe.cu).  Each warp compacts its segment's candidates
//             key >= tau_l (the speculative band predicted by the previous call) in index order with
//             ballots, stages them in shared memory and stores whole 32-entry runs into the segment's
//             bounded slot (cs entries: keys then indices), histogramming the first radix digit (key
//             bits [30:20]) of every candidate on the way.  A segment with more than cs candidates is
//             marked DIRECT: its list is not kept and later passes re-read its 1024 acc values (4 KB)
//             from HBM instead -- exactness never depends on the capacity, which only bounds the
//             scratch at O(K) (cs ~ 12 x the expected candidates per segment: 1 B/param at 1%).
//     prep:   warp per chunk: compacts its stored segment lists in place into one index-ordered
//             chunk list, and histograms the first radix digit (key bits [30:20]) of its candidates.
//     plan:   per layer, #candidates >= k_l means the exact top-k lies inside the band (hit);
//             otherwise a refill: a histogram pass over the layer's acc finds the digit-0 bin of
//             the k-th key, and the layer is rescanned at that bin's lower edge (>= k candidates
//             by construction, about k + the bin's population).
//     digits: two more radix digits over the candidates -> the exact k-th key T and the number of
//             ties at T to take (lowest indices first).
//     count+emit: a warp per chunk counts key > T and key == T, takes its layer offset and the ties
//             taken before it by a decoupled look-back over the layer's earlier chunks, and writes
//             its selected entries at their final positions (residual' zeroing is lazy).
//   HBM traffic in the steady state: 12 B/param + ~(16 + 8 + 8 + 8) B per candidate (~1.5-2 k per
//   layer) + 8 B/entry (+ 4 KB per DIRECT segment and pass).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"
#include "pdl.cuh"

namespace ld {
namespace {

// Large layers select in two windowed digits: all candidates have key >= W (the threshold they
// were taken with), so digit 0 is bin(key) = min(2047, (key - W) >> 11) -- 2047 bins of 2^11 key
// units (half a binade above W) and an overflow bin -- and digit 1 the low 11 bits of key - W:
// the k-th key exactly after two passes (a third, absolute digit of round 1 is gone).  A k-th key in
// the overflow bin (the band was far too low) is treated as a miss and refilled.  (The refill's
// histogram pass and the small layers keep absolute digits: key bits [30:20], [19:9], [8:0].)
constexpr int kH0 = 2048, kH1 = 2048, kH2 = 512;
constexpr int kHistRow = kH0 + kH1;
constexpr int kWinShift = 11;
constexpr uint32_t kWinOver = (uint32_t)kH0 - 1;   // the overflow bin
__device__ __forceinline__ uint32_t win_bin(uint32_t key, uint32_t W) { return min(kWinOver, (key - W) >> kWinShift); }
#ifndef LD_SCAN_WARPS
#define LD_SCAN_WARPS 4
#endif
constexpr int kScanWarps = LD_SCAN_WARPS;           // segments per scan CTA
constexpr int kPiecesPerChunk = kSegsPerChunk / kScanWarps;   // 4 scan CTAs per chunk
#ifndef LD_UNROLL
#define LD_UNROLL 4
#endif
constexpr int kUnroll = LD_UNROLL;                  // candidate rounds in flight per warp
constexpr uint32_t kDirect = 0x80000000u;           // seg_count flag: list not stored, read acc
#ifndef LD_BAND_AIM
#define LD_BAND_AIM 1.5f
#endif
constexpr float kBandAim = LD_BAND_AIM;             // speculative band: candidates admitted / k_l

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
  if (w == 64 || w == 16) {   // the 2048- and 512-bin digits: all of the lane's 128-bit loads in
                              // flight at once (h is 16-byte aligned, top - w a multiple of 16)
    const uint4* h4 = reinterpret_cast<const uint4*>(h + top - w);
    uint4 q[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < w / 4) q[i] = h4[i];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < w / 4) s += (q[i].x + q[i].y) + (q[i].z + q[i].w);
  } else {
#pragma unroll 16
    for (int b = top - 1; b >= top - w; --b) s += h[b];
  }
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
  // second level, warp-parallel: the w bins of lane src (w = 64 or <= 32), highest first, spread
  // over the lanes (2 or 1 per lane), prefix-summed with shuffles
  const int stop = __shfl_sync(0xFFFFFFFFu, top, src);
  const uint32_t base = __shfl_sync(0xFFFFFFFFu, exc, src);
  const uint32_t need = kleft - base;   // >= 1 when src holds the bin
  const int per = w > 32 ? w / 32 : 1;  // bins per lane (w is 64 or a power of two <= 32)
  const int b_hi = stop - 1 - lane * per;
  uint32_t c0 = 0, c1 = 0;
  if (lane * per < w) {
    c0 = h[b_hi];
    if (per == 2) c1 = h[b_hi - 1];
  }
  const uint32_t s2 = c0 + c1;
  uint32_t inc2 = s2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc2, o);
    if (lane >= o) inc2 += y;
  }
  const uint32_t exc2 = inc2 - s2;
  const bool hit = lane * per < w && exc2 < need && need <= inc2;
  const unsigned who2 = __ballot_sync(0xFFFFFFFFu, hit);
  uint32_t bin, above;
  if (who2) {
    const int src2 = __ffs(who2) - 1;
    const bool first = exc2 + c0 >= need;
    bin = first ? (uint32_t)b_hi : (uint32_t)(b_hi - 1);
    above = base + exc2 + (first ? 0u : c0);
    bin = __shfl_sync(0xFFFFFFFFu, bin, src2);
    above = __shfl_sync(0xFFFFFFFFu, above, src2);
  } else {   // kleft exceeds the total (never on a consistent histogram): lowest bin, all counted
    bin = (uint32_t)(stop - w);
    above = base + __shfl_sync(0xFFFFFFFFu, inc2, 31);
  }
  *bin_out = bin;
  *above_out = above;
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

// warp-aggregated histogram increment: lanes with m set add 1 to h[bin] (called by all 32 lanes)
__device__ __forceinline__ void warp_hist_add(uint32_t* h, bool m, uint32_t bin) {
  const unsigned act = __ballot_sync(0xFFFFFFFFu, m);
  if (m) {
    const unsigned peers = __match_any_sync(act, bin);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], (uint32_t)__popc(peers));
  }
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
      __syncwarp();   // every lane has read s_kleft before lane 0 updates it
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

// ---------------------------------------------------------------- large layers: segment compaction
// Lazy residual zeroing: the previous call left residual' = acc at its selection; an element was
// selected iff key > T_prev or (key == T_prev and index < cut_prev), so the scan zeroes it here
// (exactly the +0.0f the eager residual' would hold) instead of a scattered zeroing pass.
__device__ __forceinline__ float lazy_zero(float rv, uint32_t gidx, uint32_t T, uint32_t cut) {
  const uint32_t key = key_of(rv);
  return (key > T || (key == T && gidx < cut)) ? 0.0f : rv;
}

// Candidates of a warp are staged in shared memory and leave in whole 32-entry (256-byte) runs (a
// round produces only a few; storing them straight from the lanes wrote each global sector several
// times).  A candidate is the 64-bit word (acc bits << 32 | global index).
constexpr int kCandBuf = 32 + 32 * 4;   // < 32 staged + one round's worst case

#ifndef LD_SCAN_MINB
#define LD_SCAN_MINB (64 / LD_SCAN_WARPS)
#endif

// One warp's 1024-element segment.  RESCAN = false: acc = r + g (lazy zeros applied), r' = acc
// stored; RESCAN = true: acc re-read (r when EF, else g; the scan of this call left acc there).
// Candidates key >= thr (thr <= 0x7F800000, so every non-finite key is one) are compacted in index
// order into cd[0..cap) (a segment with more than cap keeps only the count: the caller marks it
// DIRECT); HIST: their digit-0 bins are added to h0.  Returns the count.  FULL: the segment lies
// inside the layer (every chunk but a layer's ragged first/last one), so the valid-lane masks and
// the scalar edge path compile away.
template <bool EF, bool RESCAN, bool FULL, bool HIST>
__device__ __forceinline__ uint32_t scan_segment(const float* __restrict__ gc, float* __restrict__ rc,
                                                 uint64_t* __restrict__ cd, uint32_t cap, uint32_t* __restrict__ h0,
                                                 uint64_t* sbuf, uint32_t sb, uint32_t lo, uint32_t hi,
                                                 uint32_t gbase, uint32_t thr, uint32_t lT, uint32_t lcut, int lane,
                                                 unsigned lt, bool& bad) {
  uint32_t run = 0, staged = 0, flushed = 0;   // run = flushed + staged
  auto load = [&](int rd, float4& gq, float4& rq, uint32_t& vq) {
    const uint32_t e0 = sb + 4u * (rd * 32 + lane);
    if (FULL) {
      vq = 0xF;
    } else {
      vq = 0;
      if (e0 >= lo && e0 + 4 <= hi) vq = 0xF;
      else if (e0 + 4 > lo && e0 < hi)
        for (int k = 0; k < 4; ++k) vq |= (e0 + k >= lo && e0 + k < hi) ? 1u << k : 0u;
    }
    if (vq == 0xF) {
      if (RESCAN) {
        gq = *reinterpret_cast<const float4*>((EF ? rc : gc) + e0);
      } else {
        gq = __ldcs(reinterpret_cast<const float4*>(gc + e0));
        if (EF) rq = __ldcs(reinterpret_cast<const float4*>(rc + e0));
      }
    }
  };
  // flush n staged entries (n a multiple of 32, or the final remainder when last)
  auto flush = [&](uint32_t n, bool last) {
    __syncwarp();
    const uint32_t iters = last ? 1u : n / 32u;
    for (uint32_t it = 0; it < iters; ++it) {
      const uint32_t i = it * 32u + lane;
      const bool ok = i < n;
      const uint64_t x = ok ? sbuf[i] : 0ull;
      if (ok && flushed + i < cap) cd[flushed + i] = x;
      if (HIST) warp_hist_add(h0, ok, (uint32_t)(x >> 52) & 0x7FFu);   // key bits [30:20]
    }
    __syncwarp();
  };
  constexpr bool kPF = true;   // issue round r+1's loads before round r is processed
  float4 gn = make_float4(0.f, 0.f, 0.f, 0.f), rn = gn;
  uint32_t vn = 0;
  if (kPF) load(0, gn, rn, vn);
#pragma unroll 1
  for (int rd = 0; rd < kSeg / 128; ++rd) {   // rounds of one float4 x 32 lanes
    float4 gv, rv;
    uint32_t vm;
    if (kPF) {
      gv = gn;
      rv = rn;
      vm = vn;
      if (rd + 1 < kSeg / 128) load(rd + 1, gn, rn, vn);
    } else {
      load(rd, gv, rv, vm);
    }
    const uint32_t e0 = sb + 4u * (rd * 32 + lane);
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (FULL || vm == 0xF) {
      if (!RESCAN && EF) {
        const float4 q = rv;
        const uint32_t k0 = key_of(q.x), k1 = key_of(q.y), k2 = key_of(q.z), k3 = key_of(q.w);
        if ((k0 == lT) | (k1 == lT) | (k2 == lT) | (k3 == lT)) {   // a tie with T_prev: exact rule
          const uint32_t gi = gbase + e0;
          a = make_float4(__fadd_rn(lazy_zero(q.x, gi, lT, lcut), gv.x), __fadd_rn(lazy_zero(q.y, gi + 1, lT, lcut), gv.y),
                          __fadd_rn(lazy_zero(q.z, gi + 2, lT, lcut), gv.z), __fadd_rn(lazy_zero(q.w, gi + 3, lT, lcut), gv.w));
        } else {
          a = make_float4(__fadd_rn(k0 > lT ? 0.0f : q.x, gv.x), __fadd_rn(k1 > lT ? 0.0f : q.y, gv.y),
                          __fadd_rn(k2 > lT ? 0.0f : q.z, gv.z), __fadd_rn(k3 > lT ? 0.0f : q.w, gv.w));
        }
      } else {
        a = gv;
      }
      if (!RESCAN && EF) __stcs(reinterpret_cast<float4*>(rc + e0), a);
    } else if (vm) {   // ragged edge of a layer: scalar
      for (int k = 0; k < 4; ++k)
        if ((vm >> k) & 1u) {
          float y;
          if (RESCAN) y = EF ? rc[e0 + k] : gc[e0 + k];
          else y = EF ? __fadd_rn(lazy_zero(rc[e0 + k], gbase + e0 + k, lT, lcut), gc[e0 + k]) : gc[e0 + k];
          f4set(a, k, y);
          if (!RESCAN && EF) rc[e0 + k] = y;
        }
    }
    // flags + ordered compaction: (round, lane, k) order == index order
    uint32_t fl = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool v = FULL || ((vm >> k) & 1u);
      fl |= (v && key_of(f4get(a, k)) >= thr) ? 1u << k : 0u;
    }
    unsigned bm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) bm[k] = __ballot_sync(0xFFFFFFFFu, (fl >> k) & 1u);
    uint32_t pos = staged;
#pragma unroll
    for (int k = 0; k < 4; ++k) pos += __popc(bm[k] & lt);
    if (fl) {
      const uint32_t gi = gbase + e0;   // global index (Psi < 2^32)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((fl >> k) & 1u) {
          bad |= key_of(f4get(a, k)) >= 0x7F800000u;
          sbuf[pos++] = ((uint64_t)__float_as_uint(f4get(a, k)) << 32) | (gi + k);
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) cnt += __popc(bm[k]);
    run += cnt;
    staged += cnt;
    if (staged >= 32) {   // whole 32-entry runs out; the remainder moves to the front
      const uint32_t full = staged & ~31u;
      flush(full, false);
      const uint32_t rest = staged - full;
      uint64_t x = lane < rest ? sbuf[full + lane] : 0;
      __syncwarp();
      if (lane < rest) sbuf[lane] = x;
      __syncwarp();
      flushed += full;
      staged = rest;
    }
  }
  flush(staged, true);
  return run;
}

// the segment's candidate slot: cs 64-bit candidates
__device__ __forceinline__ uint64_t* seg_slot(const DevPlan& P, uint64_t segid) {
  return P.cand + segid * (uint32_t)P.cs;
}

template <bool EF>
__global__ void __launch_bounds__(kScanWarps * 32, LD_SCAN_MINB)
scan_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r, int lazy) {
  __shared__ uint64_t sbuf_all[kScanWarps][kCandBuf];
  {  // the select chain's per-call state (histograms, candidate totals, counters, look-back states):
     // zeroed here -- it is first read after this grid -- instead of by four memset graph nodes
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t nh = (uint64_t)P.n_large * kHistRow;
    for (uint64_t i = gid; i < nh; i += nthr) P.hist[i] = 0u;
    if (gid < (uint64_t)P.n_large) P.layer_total[gid] = 0u;
    if (gid < 8) P.counters[gid] = 0u;
    for (uint64_t i = gid; i < (uint64_t)P.n_chunks; i += nthr) P.chunk_state[i] = 0ull;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t w = blockIdx.x;
  const int ch = (int)(w / kPiecesPerChunk);
  const int seg = (int)(w % kPiecesPerChunk) * kScanWarps + warp;
  // chunk-local 32-bit offsets keep the register footprint (and so the occupancy that hides HBM
  // latency) at the level of a plain streaming kernel
  const uint64_t cbase = P.chunk_base[ch];
  const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
  const int slot = P.chunk_slot[ch];
  const uint32_t thr = min(P.thr[slot], 0x7F800000u);
  const bool lz = EF && lazy;
  const uint32_t lT = lz ? P.sel_T[slot] : 0xFFFFFFFFu, lcut = lz ? P.sel_cut[slot] : 0u;
  const uint64_t segid = (uint64_t)ch * kSegsPerChunk + seg;
  const uint32_t cs = (uint32_t)P.cs;
  uint64_t* cd = seg_slot(P, segid);
  const uint32_t sb = (uint32_t)seg * kSeg;
  bool bad = false;
  const uint32_t run =
      (sb >= lo && sb + kSeg <= hi)
          ? scan_segment<EF, false, true, false>(g + cbase, r + cbase, cd, cs, nullptr, sbuf_all[warp], sb, lo, hi,
                                                 (uint32_t)cbase, thr, lT, lcut, lane, lt, bad)
          : scan_segment<EF, false, false, false>(g + cbase, r + cbase, cd, cs, nullptr, sbuf_all[warp], sb, lo, hi,
                                                  (uint32_t)cbase, thr, lT, lcut, lane, lt, bad);
  if (lane == 0) {
    P.seg_count[segid] = run > cs ? (run | kDirect) : run;   // layer totals: the select's first pass
  }
  if (bad) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)P.large_layers[slot]); }
}

// A DIRECT segment's acc values, read from HBM: src = r (EF: the scan stored acc there) or g.
// Calls f(ok, key_bits, global_index) for the 4 elements of each lane per 128-element round (all
// lanes, convergent), ok = in the layer and key >= thr.  Unordered across k.
// The chunk geometry and selection arrays the out-of-line helpers need, passed BY VALUE: a
// `const DevPlan&` argument of a __noinline__ function makes every thread copy the whole kernel
// parameter block to local memory at kernel entry (measured: 600 MB of DRAM writes per GPT-2 XL
// count+emit launch).
struct ChunkRefs {
  const uint64_t* base;
  const uint64_t* lo;
  const uint64_t* hi;
  const uint32_t* seg_count;
  uint32_t* sel_cut;
};
__device__ __forceinline__ ChunkRefs chunk_refs(const DevPlan& P) {
  return ChunkRefs{P.chunk_base, P.chunk_lo, P.chunk_hi, P.seg_count, P.sel_cut};
}

template <class F>
__device__ __forceinline__ void visit_direct(const ChunkRefs& R, const float* __restrict__ src, int ch, int seg,
                                             uint32_t thr, int lane, F&& f) {
  const uint64_t cbase = R.base[ch];
  const uint32_t lo = (uint32_t)(R.lo[ch] - cbase), hi = (uint32_t)(R.hi[ch] - cbase);
  const float* s = src + cbase;
  const uint32_t sb = (uint32_t)seg * kSeg;
#pragma unroll 2
  for (int rd = 0; rd < kSeg / 128; ++rd) {
    const uint32_t e0 = sb + 4u * (rd * 32 + lane);
    uint32_t vm = 0;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 >= lo && e0 + 4 <= hi) {
      vm = 0xF;
      a = *reinterpret_cast<const float4*>(s + e0);
    } else if (e0 + 4 > lo && e0 < hi) {
      for (int k = 0; k < 4; ++k)
        if (e0 + k >= lo && e0 + k < hi) { vm |= 1u << k; f4set(a, k, s[e0 + k]); }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t bits = __float_as_uint(f4get(a, k));
      f(((vm >> k) & 1u) && (bits & 0x7FFFFFFFu) >= thr, bits, (uint32_t)cbase + e0 + k);
    }
  }
}

template <class F>
__device__ __forceinline__ void visit_direct(const DevPlan& P, const float* __restrict__ src, int ch, int seg,
                                             uint32_t thr, int lane, F&& f) {
  visit_direct(chunk_refs(P), src, ch, seg, thr, lane, static_cast<F&&>(f));
}

// Refill, pass 1: the digit-0 histogram (key bits [30:20]) of EVERY element of the listed chunks'
// acc (r when EF, else g), one CTA per listed chunk at a time (persistent grid).  Each thread keeps
// four 128-bit loads in flight (16 per chunk); the counts go straight to a shared-memory histogram
// (same-bin lanes serialise in the atomic unit, cheaper than aggregating them first) that is added
// to the layer's histogram row (zeroed by the plan).  Find mode 5 then picks the k-th key's bin.
// CTA-level (256 threads); sh: kH0 words of shared memory.
__device__ __forceinline__ void refill_hist_chunk(const DevPlan& P, const float* __restrict__ src, int ch,
                                                  uint32_t* sh) {
  constexpr int kV = kChunk / 4 / 256;   // float4 per thread per chunk (16)
  {
    const uint64_t cbase = P.chunk_base[ch];
    const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
    const float* sp = src + cbase;
    for (int b = threadIdx.x; b < kH0; b += 256) sh[b] = 0;
    __syncthreads();
#pragma unroll 1
    for (int v0 = 0; v0 < kV; v0 += 4) {
      float4 a[4];
      uint32_t vm[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t e0 = 4u * ((v0 + u) * 256 + threadIdx.x);
        vm[u] = 0;
        a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e0 >= lo && e0 + 4 <= hi) {
          vm[u] = 0xF;
          a[u] = *reinterpret_cast<const float4*>(sp + e0);
        } else if (e0 + 4 > lo && e0 < hi) {
          for (int k = 0; k < 4; ++k)
            if (e0 + k >= lo && e0 + k < hi) { vm[u] |= 1u << k; f4set(a[u], k, sp[e0 + k]); }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((vm[u] >> k) & 1u) atomicAdd(&sh[(__float_as_uint(f4get(a[u], k)) >> 20) & 0x7FFu], 1u);
    }
    __syncthreads();
    uint32_t* hrow = P.hist + (uint64_t)P.chunk_slot[ch] * kHistRow;
    for (int b = threadIdx.x; b < kH0; b += 256)
      if (sh[b]) atomicAdd(&hrow[b], sh[b]);
    __syncthreads();
  }
}

// Refill, pass 2: segment `seg` of chunk ch is rescanned at its layer's thr_used (acc re-read: r
// when EF, else g) into its slot (warp-level; sbuf: the warp's kCandBuf staging entries).
template <bool EF>
__device__ __forceinline__ void rescan_segment(const DevPlan& P, const float* __restrict__ g, float* __restrict__ r,
                                               int ch, int seg, uint64_t* sbuf, int lane) {
  const unsigned lt = (1u << lane) - 1u;
  {
    const uint64_t cbase = P.chunk_base[ch];
    const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
    const int slot = P.chunk_slot[ch];
    const uint64_t segid = (uint64_t)ch * kSegsPerChunk + seg;
    const uint32_t cs = (uint32_t)P.cs;
    bool bad = false;
    const uint32_t run = scan_segment<EF, true, false, false>(g + cbase, r + cbase, seg_slot(P, segid), cs, nullptr,
                                                              sbuf, (uint32_t)seg * kSeg, lo, hi,
                                                              (uint32_t)cbase, P.thr_used[slot], 0xFFFFFFFFu, 0u,
                                                              lane, lt, bad);
    if (lane == 0) {
      P.seg_count[segid] = run > cs ? (run | kDirect) : run;
      if (run > cs) atomicAdd(&P.counters[5], 1u);   // DIRECT segments (stats)
    }
  }
}

// ---------------------------------------------------------------- chunk prep (warp per chunk)
// Compact the stored segment lists of a chunk in place into one index-ordered list at the chunk's
// region start (a candidate never moves up -- the list offset of segment s is at most s cs -- and
// each round loads before it stores), store its length and DIRECT mask, and histogram the first
// radix digit (key bits [30:20]) of its candidates: the stored ones, and those of its DIRECT
// segments read from acc (src) at the layer's threshold -- in shared memory when all chunks of the
// CTA belong to one layer (chunk slots are monotone), else directly.
// mode 0: every chunk (after the scan); 1: chunks of refilled layers (after their rescan), walking
// the refill list (the layers' chunks, listed contiguously).  One round = items i0 .. i0 + 7 (a warp
// each), CTA-level (256 threads); sh: kH0 words of shared memory, s_tot one more.
__device__ __forceinline__ void chunk_prep_round(const DevPlan& P, const float* __restrict__ src, int mode,
                                                 uint32_t i0, uint32_t n_items, uint32_t* sh, uint32_t* s_tot) {
  const uint32_t* list = P.refill_list;
  const int lane = threadIdx.x & 31;
  {
  const uint32_t i_last = min(n_items, i0 + 8u) - 1u;
  const int c_first = mode == 0 ? (int)i0 : (int)list[i0];
  const int c_last = mode == 0 ? (int)i_last : (int)list[i_last];
  const uint32_t item = i0 + (threadIdx.x >> 5);
  const int ch = item <= i_last ? (mode == 0 ? (int)item : (int)list[item]) : c_last;
  const bool uniform = P.chunk_slot[c_first] == P.chunk_slot[c_last];
  if (uniform) {
    __syncthreads();   // the previous round's flush has read sh
    for (int b = threadIdx.x; b < kH0; b += 256) sh[b] = 0;
    if (threadIdx.x == 0) *s_tot = 0;
    __syncthreads();
  }
  const int slot = P.chunk_slot[ch];
  const bool active = item <= i_last;
  if (active) {
    uint32_t* h0 = uniform ? sh : P.hist + (uint64_t)slot * kHistRow;
    // the threshold the chunk's candidates were taken with: the scan's band (mode 0) or the refill's
    const uint32_t thr = mode == 0 ? min(P.thr[slot], 0x7F800000u) : P.thr_used[slot];
    const uint32_t sc = lane < kSegsPerChunk ? P.seg_count[(uint64_t)ch * kSegsPerChunk + lane] : 0u;
    const bool direct = (sc & kDirect) != 0u;
    const uint32_t c = direct ? 0u : sc;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t so = inc - c;                                  // lanes 0..15: segment offsets
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, inc, 31);
    const unsigned dm = __ballot_sync(0xFFFFFFFFu, direct) & 0xFFFFu;
    const uint32_t cs = (uint32_t)P.cs;
    uint64_t* cd = seg_slot(P, (uint64_t)ch * kSegsPerChunk);
    for (uint32_t base = 0; base < total; base += 32 * kUnroll) {
      uint64_t v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint32_t cc = base + u * 32 + lane;
        int s = 0;   // segment of candidate cc: max{s : so[s] <= cc}, by shuffles over lanes 0..15
#pragma unroll
        for (int step = 8; step; step >>= 1) {
          const uint32_t t = __shfl_sync(0xFFFFFFFFu, so, s + step);
          if (t <= cc) s += step;
        }
        const uint32_t sos = __shfl_sync(0xFFFFFFFFu, so, s);
        v[u] = cc < total ? cd[(uint32_t)s * cs + (cc - sos)] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint32_t cc = base + u * 32 + lane;
        if (cc < total) cd[cc] = v[u];
        const uint32_t bin = win_bin((uint32_t)(v[u] >> 32) & 0x7FFFFFFFu, thr);   // windowed digit 0
        if (uniform) { if (cc < total) atomicAdd(&h0[bin], 1u); }
        else warp_hist_add(h0, cc < total, bin);
      }
    }
    uint32_t dcnt = 0;   // DIRECT segments: their candidates read from acc
    for (unsigned m = dm; m; m &= m - 1) {
      visit_direct(P, src, ch, __ffs(m) - 1, thr, lane, [&](bool ok, uint32_t bits, uint32_t) {
        const uint32_t bin = win_bin(bits & 0x7FFFFFFFu, thr);
        if (uniform) { if (ok) atomicAdd(&h0[bin], 1u); }
        else warp_hist_add(h0, ok, bin);
        dcnt += ok;
      });
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dcnt += __shfl_xor_sync(0xFFFFFFFFu, dcnt, o);
    if (lane == 0) {
      P.chunk_count[ch] = total;
      P.chunk_dm[ch] = dm;
      if (dm && mode == 0) atomicAdd(&P.counters[5], (uint32_t)__popc(dm));   // DIRECT segments (stats)
      if (uniform) atomicAdd(s_tot, total + dcnt);
      else atomicAdd(&P.layer_total[slot], total + dcnt);   // per-layer candidate count
    }
  }
  if (uniform) {
    __syncthreads();
    uint32_t* hrow = P.hist + (uint64_t)P.chunk_slot[c_first] * kHistRow;
    for (int b = threadIdx.x; b < kH0; b += 256)
      if (sh[b]) atomicAdd(&hrow[b], sh[b]);
    if (threadIdx.x == 0 && *s_tot) atomicAdd(&P.layer_total[P.chunk_slot[c_first]], *s_tot);
  }
  }
}

// chunk prep of every chunk after the scan (mode 0)
__global__ void __launch_bounds__(256) chunk_prep_kernel(DevPlan P, const float* __restrict__ src) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t sh[kH0];
  __shared__ uint32_t s_tot;
  for (uint32_t i0 = blockIdx.x * 8u; i0 < (uint32_t)P.n_chunks; i0 += gridDim.x * 8u)
    chunk_prep_round(P, src, 0, i0, (uint32_t)P.n_chunks, sh, &s_tot);
}

// ---------------------------------------------------------------- per-layer plan / digit search
__device__ __forceinline__ uint32_t layer_candidates(const DevPlan& P, int slot) {
  return *reinterpret_cast<volatile const uint32_t*>(P.layer_total + slot);
}

// queue every chunk of the layer for a refill (zeroes the layer's digit-0 histogram, which the
// refill's histogram pass then fills with every element of the layer)
__device__ void queue_refill(const DevPlan& P, int slot, int c0, int c1, int lane) {
  uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
  for (int b = lane; b < kH0; b += 32) hrow[b] = 0;
  if (lane == 0) {
    P.layer_total[slot] = 0;   // the refill's chunk_prep recounts every chunk
    P.trace[slot] = 1u;
  }
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(&P.counters[0], (uint32_t)(c1 - c0));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  for (int c = c0 + lane; c < c1; c += 32) P.refill_list[base + (c - c0)] = (uint32_t)c;
}

// mode 0: after the scan -- hit: digit 0; miss: queue a refill
// mode 5: after the refill's histogram pass -- the refill threshold: the lower edge of the digit-0
//         bin holding the k-th key (every element at or above it is a candidate: >= k of them)
// mode 1: after the refill's rescan + prep -- digit 0 (a hit by construction)
// mode 2: digit 1 for every large layer -> the exact k-th key, and the next call's band
// (warp-level: one large layer per warp)
__device__ void find_layer(const DevPlan& P, int slot, int mode, int lane) {
  const int li = P.large_layers[slot];
  const uint32_t k = P.layer_k[li];
  LayerSel& S = P.sel[slot];
  uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
  const int c0 = P.large_chunk0[slot], c1 = P.large_chunk0[slot + 1];
  if (mode == 0) {
    const uint32_t tot = layer_candidates(P, slot);
    uint32_t bin = kWinOver, above = 0;
    if (tot >= k) warp_find_bin(hrow, kH0, k, &bin, &above);
    if (tot >= k && bin < kWinOver) {   // a k-th key in the overflow bin is refilled like a miss
      if (lane == 0) {
        S.prefix = bin; S.kleft = k - above; S.total = tot; S.refill = 0;
        P.trace[slot] = 0;
        P.thr_used[slot] = min(P.thr[slot], 0x7F800000u);   // the scan's band (DIRECT re-reads)
        // adapt the band: the previous call chose it to admit `band` x k keys of ITS distribution;
        // under error feedback the accumulated values drift upward between calls, so the band
        // admitted tot / k x k now.  Aim the next band at kBandAim x k_l admitted.
        const float b = S.band > 0.f ? S.band : kBandAim;
        S.band = fminf(4.f, fmaxf(1.02f, b * kBandAim * (float)k / (float)tot));
        S.alpha = fminf(0.5f, S.alpha + 0.05f);   // drift share of the threshold: recover slowly
        atomicAdd(&P.counters[1], 1u);
        atomicAdd(&P.counters[3], tot);
      }
    } else {
      // missed (or the k-th key lies in the window's overflow bin): the refill histograms every
      // element of the layer (refill_hist_kernel), then rescans at the digit-0 bin of the k-th key
      // (mode 5): the new window base W = that bin's lower edge, so T lies within 2^20 above W.
      queue_refill(P, slot, c0, c1, lane);
      if (lane == 0) {
        S.refill = 1;
        S.total = (uint32_t)(P.layer_off[li + 1] - P.layer_off[li]);
        S.alpha *= 0.5f;                          // the drift prediction overshot
        atomicAdd(&P.counters[2], 1u);
      }
    }
  } else if (mode == 5) {
    if (S.refill != 1) return;
    uint32_t bin, above;
    warp_find_bin(hrow, kH0, k, &bin, &above);   // the full digit-0 histogram of the layer
    __syncwarp();
    for (int b = lane; b < kH0; b += 32) hrow[b] = 0;   // chunk_prep (mode 1) histograms the candidates
    if (lane == 0) P.thr_used[slot] = bin << 20;        // keys >= bin << 20: above + h[bin] >= k of them
  } else if (mode == 1) {
    if (S.refill != 1) return;
    const uint32_t tot = layer_candidates(P, slot);
    if (tot < k) {   // impossible: the rescan admits exactly the elements the histogram counted
      if (lane == 0) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)li); }
      return;
    }
    uint32_t bin, above;
    warp_find_bin(hrow, kH0, k, &bin, &above);
    if (lane == 0) { S.prefix = bin; S.kleft = k - above; S.total = tot; }
  } else {   // mode 2: digit 1 -> the exact k-th key T and the ties to take; the next call's band
    const uint32_t* h = hrow + kH0;
    uint32_t bin, above;
    warp_find_bin(h, kH1, S.kleft, &bin, &above);
    const uint32_t W = P.thr_used[slot];
    const uint32_t T = W + (S.prefix << kWinShift) + bin;
    // Speculative band for the next call: the key with C = band x k_l candidate keys at or above
    // it (digit-0 resolution, refined with the digit-1 histogram when C falls in T's digit-0 bin).
    // Only a prediction -- the next call checks #candidates >= k_l and refills otherwise.
    const float band = S.band > 0.f ? S.band : kBandAim;
    const uint32_t C = max(k + 32u, (uint32_t)fminf((float)k * band, 4.0e9f));
    // (a refilled layer's fallback is its refill threshold, which admitted >= k_l this call)
    uint32_t nt = S.refill ? W : P.thr[slot];
    if (S.total >= C) {
      uint32_t b0, a0;
      warp_find_bin(hrow, kH0, C, &b0, &a0);
      if (b0 == S.prefix) {
        uint32_t b1, a1;
        warp_find_bin(h, kH1, C - a0, &b1, &a1);
        nt = W + (b0 << kWinShift) + b1;
      } else {
        nt = W + (b0 << kWinShift);
      }
    }
    // drift share: under error feedback the k-th key moved from T_{t-1} (sel_T, still the previous
    // call's) to T_t; lead the next band by alpha x the smaller of this drift and the previous
    // call's, so a T that alternates (periodic inputs) gets no lead.
    const uint32_t t_prev = P.sel_T[slot];
    const uint32_t d_now = (t_prev != 0xFFFFFFFFu && T > t_prev) ? T - t_prev : 0u;
    const uint32_t d = min(d_now, S.drift);
    uint32_t na = nt;
    if (d > 0 && nt != 0xFFFFFFFFu) {
      const float a = fmaxf(0.f, fminf(0.5f, S.alpha));
      na = nt + (uint32_t)(a * (float)d);
      na = min(na, 0x7F800000u);
    }
    if (lane == 0) {
      S.next_thr = na; S.next_safe = nt; S.drift = d_now;
      S.prefix = T; S.kleft -= above;
    }
  }
}

__global__ void __launch_bounds__(256) find_kernel(DevPlan P, int mode) {
  pdl_wait();
  pdl_trigger();
  const int slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (slot < P.n_large) find_layer(P, slot, mode, threadIdx.x & 31);
}

// Grid-wide barrier of a co-resident grid (refill_kernel): counter `bar` is zeroed per call with the
// other counters; barrier n (1, 2, ...) releases when every CTA has arrived n times.
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    const uint32_t target = n * gridDim.x;
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// The refill of the layers find mode 0 queued, one launch for the whole sequence:
// histogram pass -> refill threshold (find mode 5) -> rescan at it -> chunk prep -> find mode 1,
// phases separated by grid barriers (the grid is co-resident: a cooperative launch sized by the
// occupancy).  Nothing queued -- the steady state -- is one early exit, not five empty launches.
template <bool EF>
__global__ void __launch_bounds__(256) refill_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r,
                                                     const float* __restrict__ src) {
  pdl_wait();
  pdl_trigger();
  const uint32_t n = P.counters[0];   // chunks queued (written by find mode 0, before this grid)
  if (n == 0) return;
  __shared__ __align__(16) uint64_t smem[8 * kCandBuf];   // 10 KB: staging (rescan) or histogram
  __shared__ uint32_t s_tot;
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + warp, nw = gridDim.x * 8;
  uint32_t* bar = P.counters + 6;
  for (uint32_t w = blockIdx.x; w < n; w += gridDim.x) refill_hist_chunk(P, src, (int)P.refill_list[w], sh);
  grid_barrier(bar, 1);
  for (int slot = gw; slot < P.n_large; slot += nw) find_layer(P, slot, 5, lane);
  grid_barrier(bar, 2);
  for (uint32_t w = blockIdx.x; w < 2 * n; w += gridDim.x)   // half a chunk (8 segments) per CTA round
    rescan_segment<EF>(P, g, r, (int)P.refill_list[w >> 1], (int)(w & 1) * 8 + warp, smem + warp * kCandBuf, lane);
  grid_barrier(bar, 3);
  for (uint32_t i0 = blockIdx.x * 8u; i0 < n; i0 += gridDim.x * 8u) chunk_prep_round(P, src, 1, i0, n, sh, &s_tot);
  grid_barrier(bar, 4);
  for (int slot = gw; slot < P.n_large; slot += nw) find_layer(P, slot, 1, lane);
}


// digit 1 histogram (the low 11 bits of key - W) over the candidates in the k-th key's windowed
// digit-0 bin (the chunk list + its DIRECT segments' acc): warp per chunk, 8 chunks per CTA
// aggregated in shared memory when they belong to one layer
__global__ void __launch_bounds__(256) digit_kernel(DevPlan P, const float* __restrict__ src) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t sh[kH1];
  const int lane = threadIdx.x & 31;
  const int c_first = blockIdx.x * 8;
  const int c_last = min(P.n_chunks, c_first + 8) - 1;
  const int ch = c_first + (threadIdx.x >> 5);
  const bool uniform = P.chunk_slot[c_first] == P.chunk_slot[c_last];
  if (uniform) {
    for (int b = threadIdx.x; b < kH1; b += 256) sh[b] = 0;
    __syncthreads();
  }
  if (ch <= c_last) {
    const int slot = P.chunk_slot[ch];
    const uint32_t pre = P.sel[slot].prefix;
    const uint32_t W = P.thr_used[slot];
    uint32_t* h = uniform ? sh : P.hist + (uint64_t)slot * kHistRow + kH0;
    const uint32_t cnt = P.chunk_count[ch];
    const uint64_t* cd = seg_slot(P, (uint64_t)ch * kSegsPerChunk);
    auto add = [&](bool ok, uint32_t key) {
      const bool m = ok && win_bin(key, W) == pre;
      const uint32_t bin = (key - W) & 0x7FFu;
      if (uniform) { if (m) atomicAdd(&h[bin], 1u); }
      else warp_hist_add(h, m, bin);
    };
    for (uint32_t base = 0; base < cnt; base += 32 * kUnroll) {
      uint32_t key[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint32_t i = base + u * 32 + lane;
        key[u] = i < cnt ? (uint32_t)(cd[i] >> 32) & 0x7FFFFFFFu : 0u;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) add(base + u * 32 + lane < cnt, key[u]);
    }
    for (unsigned m = P.chunk_dm[ch]; m; m &= m - 1)
      visit_direct(P, src, ch, __ffs(m) - 1, W, lane,
                   [&](bool ok, uint32_t bits, uint32_t) { add(ok, bits & 0x7FFFFFFFu); });
  }
  if (uniform) {
    __syncthreads();
    uint32_t* hg = P.hist + (uint64_t)P.chunk_slot[c_first] * kHistRow + kH0;
    for (int b = threadIdx.x; b < kH1; b += 256)
      if (sh[b]) atomicAdd(&hg[b], sh[b]);
  }
}

// Ordered emit of a chunk with a DIRECT segment (warp): its segments in index order -- the stored
// ones from its compacted run Lc (segment after segment), the DIRECT ones from acc.  dst0 = output
// offset of its first entry; it takes `take` of its ties (lowest index first).
__device__ __noinline__ void emit_dirty_chunk(ChunkRefs P, const float* __restrict__ src, int ch, const uint64_t* Lc,
                                 uint32_t* __restrict__ send, uint64_t K, uint64_t dst0, uint32_t T, uint32_t take,
                                 bool last_tie_chunk, int slot, int lane) {
  const unsigned lt = (1u << lane) - 1u;
  uint32_t eq_run = 0, out_run = 0;
  const uint32_t sc = lane < kSegsPerChunk ? P.seg_count[(uint64_t)ch * kSegsPerChunk + lane] : 0u;
  const uint32_t stored = (sc & kDirect) ? 0u : sc;
  uint32_t inc = stored;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  const uint32_t so = inc - stored;
  const uint64_t cbase = P.base[ch];
  const uint32_t lo = (uint32_t)(P.lo[ch] - cbase), hi = (uint32_t)(P.hi[ch] - cbase);
  for (int s = 0; s < kSegsPerChunk; ++s) {
    const uint32_t c = __shfl_sync(0xFFFFFFFFu, sc, s);
    if (!(c & kDirect)) {
      const uint64_t* cv = Lc + __shfl_sync(0xFFFFFFFFu, so, s);
      for (uint32_t b = 0; b < c; b += 32) {
        const uint32_t i = b + lane;
        const bool ok = i < c;
        const uint64_t x = ok ? cv[i] : 0ull;
        const uint32_t val = (uint32_t)(x >> 32), idx = (uint32_t)x, key = val & 0x7FFFFFFFu;
        const bool is_eq = ok && key == T;
        const unsigned eqm = __ballot_sync(0xFFFFFFFFu, is_eq);
        const bool sel = ok && (key > T || (is_eq && eq_run + __popc(eqm & lt) < take));
        const unsigned sm = __ballot_sync(0xFFFFFFFFu, sel);
        if (sel) {
          const uint64_t o = dst0 + out_run + __popc(sm & lt);
          send[o] = idx;
          send[K + o] = val;
        }
        if (last_tie_chunk && is_eq && eq_run + __popc(eqm & lt) == take - 1) P.sel_cut[slot] = idx + 1;
        eq_run += __popc(eqm);
        out_run += __popc(sm);
      }
      continue;
    }
    // direct: each lane holds 4 consecutive elements per round; order = (lane, k).  Every selected
    // element has key >= T >= the threshold, so no threshold test is needed here.
    const float* sp = src + cbase;
    const uint32_t sb = (uint32_t)s * kSeg;
    for (int rd = 0; rd < kSeg / 128; ++rd) {
      const uint32_t e0 = sb + 4u * (rd * 32 + lane);
      uint32_t bits[4] = {0, 0, 0, 0}, vm = 0;
      if (e0 >= lo && e0 + 4 <= hi) {
        const float4 x = *reinterpret_cast<const float4*>(sp + e0);
        bits[0] = __float_as_uint(x.x); bits[1] = __float_as_uint(x.y);
        bits[2] = __float_as_uint(x.z); bits[3] = __float_as_uint(x.w);
        vm = 0xF;
      } else if (e0 + 4 > lo && e0 < hi) {
        for (int k = 0; k < 4; ++k)
          if (e0 + k >= lo && e0 + k < hi) { vm |= 1u << k; bits[k] = __float_as_uint(sp[e0 + k]); }
      }
      uint32_t eqf = 0, gtf = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t key = bits[k] & 0x7FFFFFFFu;
        eqf |= (((vm >> k) & 1u) && key == T) ? 1u << k : 0u;
        gtf |= (((vm >> k) & 1u) && key > T) ? 1u << k : 0u;
      }
      const uint32_t ne = __popc(eqf);   // ties before each element: earlier lanes' + this lane's earlier
      uint32_t einc = ne;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, einc, o);
        if (lane >= o) einc += y;
      }
      const uint32_t ebase = eq_run + einc - ne;
      uint32_t self = gtf, tie_k = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((eqf >> k) & 1u) {
          if (ebase + tie_k < take) self |= 1u << k;
          if (last_tie_chunk && ebase + tie_k == take - 1) P.sel_cut[slot] = (uint32_t)cbase + e0 + k + 1;
          ++tie_k;
        }
      const uint32_t ns = __popc(self);
      uint32_t sinc = ns;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, sinc, o);
        if (lane >= o) sinc += y;
      }
      uint64_t o = dst0 + out_run + (sinc - ns);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((self >> k) & 1u) {
          send[o] = (uint32_t)cbase + e0 + k;
          send[K + o] = bits[k];
          ++o;
        }
      eq_run += __shfl_sync(0xFFFFFFFFu, einc, 31);
      out_run += __shfl_sync(0xFFFFFFFFu, sinc, 31);
    }
  }
}

// (key > T, key == T) counts of the chunk's DIRECT segments (dm), per lane, packed eq << 32 | gt;
// out of line, so the common path of count_emit keeps its 32-register budget (returned by value:
// pointers to the caller's counters would put them in local memory for every thread)
__device__ __noinline__ uint64_t count_direct(ChunkRefs P, const float* __restrict__ src, int ch, unsigned dm,
                                              uint32_t T, int lane) {
  uint32_t g = 0, e = 0;
  for (unsigned m = dm; m; m &= m - 1)
    visit_direct(P, src, ch, __ffs(m) - 1, 0u, lane, [&](bool ok, uint32_t bits, uint32_t) {
      const uint32_t key = bits & 0x7FFFFFFFu;
      g += ok && key > T;
      e += ok && key == T;
    });
  return ((uint64_t)e << 32) | g;
}

// count + layer scan + emit in one kernel (warp per chunk): the chunk's #(key > T) and #(key == T)
// (list + DIRECT segments), then a decoupled look-back over the earlier chunks of its layer (their
// published counts, 32 per round) gives the ties taken before it and its output offset, then the
// ordered emit (the list's second read hits L1/L2; a chunk with a DIRECT segment is emitted
// segment by segment).  The layer's first chunk also does the per-layer bookkeeping.
#ifndef LD_EMIT_MINB
#define LD_EMIT_MINB 8
#endif
__global__ void __launch_bounds__(256, LD_EMIT_MINB) count_emit_kernel(DevPlan P, const float* __restrict__ src,
                                                              uint32_t* __restrict__ send, uint64_t K) {
  pdl_wait();
  pdl_trigger();
  const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ch >= P.n_chunks) return;   // whole warps
  const unsigned lt = (1u << lane) - 1u;
  const int slot = P.chunk_slot[ch];
  const int c0 = P.large_chunk0[slot];
  const uint32_t T = P.sel[slot].prefix, need = P.sel[slot].kleft;
  const uint32_t cnt = P.chunk_count[ch];
  const unsigned dmask = P.chunk_dm[ch];
  const uint64_t* cd = seg_slot(P, (uint64_t)ch * kSegsPerChunk);
  uint32_t gt = 0, eq = 0;
  for (uint32_t base = 0; base < cnt; base += 32 * kUnroll) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t i = base + u * 32 + lane;
      if (i < cnt) {
        const uint32_t key = (uint32_t)(cd[i] >> 32) & 0x7FFFFFFFu;
        gt += key > T;
        eq += key == T;
      }
    }
  }
  if (dmask) {
    const uint64_t d = count_direct(chunk_refs(P), src, ch, dmask, T, lane);
    gt += (uint32_t)d;
    eq += (uint32_t)(d >> 32);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    gt += __shfl_xor_sync(0xFFFFFFFFu, gt, o);
    eq += __shfl_xor_sync(0xFFFFFFFFu, eq, o);
  }
  // per-layer counts < 2^31, so (eq << 31 | gt) words add without carries between the fields
  const unsigned long long mine = ((unsigned long long)eq << 31) | gt;
  unsigned long long before = 0;
  if (ch == c0) {
    if (lane == 0) atomicExch(P.chunk_state + ch, kInc | mine);
  } else {
    if (lane == 0) atomicExch(P.chunk_state + ch, kAgg | mine);
    int p = ch - 1;
    for (;;) {
      const int q = p - lane;   // lane 0: the nearest earlier chunk
      const unsigned long long w =
          q >= c0 ? *reinterpret_cast<volatile unsigned long long*>(P.chunk_state + q) : kInc;
      if (__any_sync(0xFFFFFFFFu, (w >> 62) == 0ull)) continue;   // not published yet
      const unsigned inc = __ballot_sync(0xFFFFFFFFu, (w >> 62) == 2ull);
      const int stop = inc ? __ffs(inc) - 1 : 31;
      unsigned long long v = lane <= stop ? (w & kVal) : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      before += v;
      if (inc) break;
      p -= 32;
    }
    if (lane == 0) {
      __threadfence();
      atomicExch(P.chunk_state + ch, kInc | (before + mine));
    }
  }
  const uint32_t gt_b = (uint32_t)(before & 0x7FFFFFFFull), eq_b = (uint32_t)(before >> 31);
  const uint32_t take_b = min(eq_b, need);       // ties are taken in chunk order, then index order
  const uint32_t take = min(eq, need - take_b);
  const bool last_tie_chunk = take > 0 && take_b + take == need;
  if (ch == c0 && lane == 0) {
    P.sel_T[slot] = T;
    // speculative band for the next call: the drift-led threshold (may exceed T),
    // never below the band without the lead capped at this call's T
    const uint32_t ns = P.sel[slot].next_safe;
    const uint32_t sf = ns <= T ? ns : T;
    P.thr[slot] = max(sf, P.sel[slot].next_thr);
  }
  const uint64_t dst0 = P.layer_koff[P.large_layers[slot]] + gt_b + take_b;
  if (dmask) {
    emit_dirty_chunk(chunk_refs(P), src, ch, cd, send, K, dst0, T, take, last_tie_chunk, slot, lane);
    return;
  }
  uint32_t eq_run = 0, out_run = 0;
  for (uint32_t base = 0; base < cnt; base += 32 * kUnroll) {
    uint64_t v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t i = base + u * 32 + lane;
      v[u] = i < cnt ? cd[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const bool ok = base + u * 32 + lane < cnt;
      const uint32_t val = (uint32_t)(v[u] >> 32), idx = (uint32_t)v[u];
      const uint32_t key = val & 0x7FFFFFFFu;
      const bool is_eq = ok && key == T;
      const unsigned eqm = __ballot_sync(0xFFFFFFFFu, is_eq);
      const bool sel = ok && (key > T || (is_eq && eq_run + __popc(eqm & lt) < take));
      const unsigned sm = __ballot_sync(0xFFFFFFFFu, sel);
      if (sel) {
        const uint64_t o = dst0 + out_run + __popc(sm & lt);
        send[o] = idx;
        send[K + o] = val;
      }
      if (last_tie_chunk && is_eq && eq_run + __popc(eqm & lt) == take - 1) P.sel_cut[slot] = idx + 1;
      eq_run += __popc(eqm);
      out_run += __popc(sm);
    }
  }
}

// residual' = 0 at the last selection of the large layers (lowdiff_residual_materialize): a
// streaming pass applying the lazy rule; small layers are always zeroed eagerly
__global__ void materialize_kernel(DevPlan P, float* __restrict__ r) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x;
  const int ch = (int)(w / kPiecesPerChunk);
  if (ch >= P.n_chunks) return;
  const int seg = (int)(w % kPiecesPerChunk) * kScanWarps + warp;
  const uint64_t cbase = P.chunk_base[ch];
  const uint64_t lo = P.chunk_lo[ch], hi = P.chunk_hi[ch];
  const int slot = P.chunk_slot[ch];
  const uint32_t T = P.sel_T[slot], cut = P.sel_cut[slot];
  for (int i = lane; i < kSeg; i += 32) {
    const uint64_t e = cbase + (uint64_t)seg * kSeg + i;
    if (e >= lo && e < hi) {
      const uint32_t key = key_of(r[e]);
      if (key > T || (key == T && (uint32_t)e < cut)) r[e] = 0.0f;   // selected last call -> +0
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

// per-segment candidate capacity: ~11.5 x the expected candidates of a 1024-element segment at the
// band's ~1.5 k_l, a multiple of 8 in [32, 1024]: <= 1 B/param of scratch at 1 % -- unless the whole
// slot array fits in kSlotFloorBytes anyway (small models), then up to a whole segment, so that a
// segment never overflows into the slower DIRECT path (ResNet-50: 25 K segments -> 1024 slots,
// 205 MB; GPT-2 XL and BERT-large keep the O(K) bound)
constexpr double kSlotFloorBytes = 256.0 * (1 << 20);
int compress_seg_capacity(uint32_t ppm, uint64_t n_segments) {
  const double want = 11.5 * kSeg * (double)ppm / 1e6;   // 1% density: 120 slots (0.94 B/param)
  const double floor_cs = n_segments ? kSlotFloorBytes / (8.0 * (double)n_segments) : (double)kSeg;
  int cs = ((int)std::max(want, std::min(floor_cs, (double)kSeg)) + 7) & ~7;
  return cs < 32 ? 32 : cs > kSeg ? kSeg : cs;
}

// lowdiff_compress: small layers (forked stream) | scan -> chunk prep -> plan -> refill (histogram,
// threshold, rescan, prep, plan) -> digit 1 -> digit 2 -> count+emit, join.
// The refill kernels exit at once when nothing was queued; the CUDA-graph form captures the same
// sequence.  Short kernels use programmatic dependent launch (pdl.cuh).
cudaError_t launch_compress(lowdiff_ctx* c, const float* grad, float* residual, uint32_t* send, cudaStream_t s) {
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
    // the small layers touch disjoint elements and send entries from the large-layer path, so
    // they run on a forked stream, concurrently with the scan, and join at the end
    const bool fork = P.n_large && c->aux;
    cudaStream_t ss = fork ? c->aux : s;
    if (fork) {
      if ((e = cudaEventRecord(c->ev_fork, s)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(c->aux, c->ev_fork, 0)) != cudaSuccess) return e;
    }
    prof_begin(c, "small_layer", ss, &h);
    if (ef) small_layer_kernel<true><<<P.n_small, kSmallThreads, smem, ss>>>(P, grad, residual, send, (uint64_t)c->K);
    else small_layer_kernel<false><<<P.n_small, kSmallThreads, smem, ss>>>(P, grad, residual, send, (uint64_t)c->K);
    prof_end(c, h, ss);
    c->launches += 1;
    if (fork && (e = cudaEventRecord(c->ev_join, c->aux)) != cudaSuccess) return e;
  }
  if (!P.n_large) {
    c->lazy_residual = nullptr;
    return cudaGetLastError();
  }
  // (the per-call state -- digit histograms, candidate totals, counters, look-back states -- is
  // zeroed by the scan kernel itself)
  const int layer_blocks = (P.n_large * 32 + 255) / 256;     // warp per large layer
  const int chunk_blocks = (P.n_chunks + 7) / 8;              // warp per chunk
  const unsigned scan_grid = (unsigned)P.n_chunks * kPiecesPerChunk;   // full grid: no tail loop
  const int uK = kScanWarps * 32;
  const float* src = ef ? residual : grad;   // where acc lives after the scan (DIRECT re-reads)
  // lazy residual zeroing applies only to the residual buffer whose selection is pending
  const int lazy = (ef && c->lazy_residual == residual) ? 1 : 0;
  prof_begin(c, "scan", s, &h);
  if (ef) scan_kernel<true><<<scan_grid, uK, 0, s>>>(P, grad, residual, lazy);
  else scan_kernel<false><<<scan_grid, uK, 0, s>>>(P, grad, residual, 0);
  prof_end(c, h, s);
  int hs;
  prof_begin(c, "select", s, &hs);
  const bool pdl = !c->prof;   // programmatic launches (pdl.cuh); profiling events sit between kernels
  if ((e = launch_pdl(pdl, chunk_prep_kernel, chunk_blocks, 256, 0, s, P, src)) != cudaSuccess) return e;
  if ((e = launch_pdl(pdl, find_kernel, layer_blocks, 256, 0, s, P, 0)) != cudaSuccess) return e;
  // refill of the missed layers: histogram pass, threshold, rescan at it, prep, plan (one launch)
  static int refill_grid[2] = {0, 0};
  if (!refill_grid[ef]) {
    int per_sm = 0;
    e = ef ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refill_kernel<true>, 256, 0)
           : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refill_kernel<false>, 256, 0);
    if (e != cudaSuccess) return e;
    refill_grid[ef] = num_sms() * std::max(1, std::min(per_sm, 4));
  }
  e = ef ? launch_pdl_ex(pdl, true, refill_kernel<true>, refill_grid[1], 256, 0, s, P, grad, residual, src)
         : launch_pdl_ex(pdl, true, refill_kernel<false>, refill_grid[0], 256, 0, s, P, grad, residual, src);
  if (e != cudaSuccess) return e;
  if ((e = launch_pdl(pdl, digit_kernel, chunk_blocks, 256, 0, s, P, src)) != cudaSuccess) return e;
  if ((e = launch_pdl(pdl, find_kernel, layer_blocks, 256, 0, s, P, 2)) != cudaSuccess) return e;
  prof_end(c, hs, s);
  prof_begin(c, "emit", s, &h);
  if ((e = launch_pdl(pdl, count_emit_kernel, chunk_blocks, 256, 0, s, P, src, send, (uint64_t)c->K)) != cudaSuccess)
    return e;
  prof_end(c, h, s);
  if (P.n_small && c->aux && (e = cudaStreamWaitEvent(s, c->ev_join, 0)) != cudaSuccess) return e;   // join
  c->launches += 7;
  c->lazy_residual = ef ? residual : nullptr;   // this call's large-layer selection is now pending
  return cudaGetLastError();
}

cudaError_t launch_materialize(lowdiff_ctx* c, float* residual, cudaStream_t s) {
  DevPlan& P = c->plan;
  if (!P.n_large || c->lazy_residual == nullptr) return cudaSuccess;
  materialize_kernel<<<(unsigned)P.n_chunks * kPiecesPerChunk, kScanWarps * 32, 0, s>>>(P, residual);
  c->launches += 1;
  if (residual == c->lazy_residual) c->lazy_residual = nullptr;   // zeros are in place now
  return cudaGetLastError();
}

}  // namespace ld
