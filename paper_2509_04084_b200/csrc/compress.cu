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
//     select: ONE persistent cooperative kernel (grid barriers between phases, no launch gaps):
//             plan -- per layer, #candidates >= k_l means the exact top-k lies inside the band (hit);
//                     otherwise a refill: level 1 rescans the layer at a lower ("safe") threshold,
//                     level 2 histograms all of its elements directly (no candidate storage);
//             two more radix digits over the candidates (or the DIRECT segments' acc) -> the exact
//             k-th key T and the number of ties at T to take (lowest indices first);
//             count+emit -- a warp per chunk counts key > T and key == T, obtains its layer offset
//             and the ties taken before it by a decoupled look-back over the layer's earlier chunks,
//             and writes its selected entries at their final positions (residual' zeroing is lazy).
//   HBM traffic in the steady state: 12 B/param + ~(4 + 4 + 4 + 8) B per candidate (~1.5-2 k per
//   layer) + 8 B/entry.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"
#include "pdl.cuh"

namespace cg = cooperative_groups;

namespace ld {
namespace {

constexpr int kH0 = 2048, kH1 = 2048, kH2 = 512;   // digit sizes: key bits [30:20] [19:9] [8:0]
constexpr int kHistRow = kH0 + kH1 + kH2;
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
constexpr int kSelThreads = 256;                    // select kernel: 8 warps per CTA
constexpr int kSelWarps = kSelThreads / 32;
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
  constexpr bool kPF = !RESCAN;   // issue round r+1's loads before round r is processed
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
    if (run > cs) P.dlist[atomicAdd(&P.counters[5], 1u)] = (uint32_t)segid;   // DIRECT, level 0
  }
  if (bad) { atomicAdd(&P.err[0], 1u); atomicMin(&P.err[1], (uint32_t)P.large_layers[slot]); }
}

// A DIRECT segment's acc values, read from HBM: src = r (EF: the scan stored acc there) or g.
// Calls f(ok, key_bits, global_index) for the 4 elements of each lane per 128-element round (all
// lanes, convergent), ok = in the layer and key >= thr.  Unordered across k.
template <class F>
__device__ __forceinline__ void visit_direct(const DevPlan& P, const float* __restrict__ src, int ch, int seg,
                                             uint32_t thr, int lane, F&& f) {
  const uint64_t cbase = P.chunk_base[ch];
  const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
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

// ---------------------------------------------------------------- per-layer plan / digit search
#ifndef LD_L1_DROP
#define LD_L1_DROP (1u << 21)
#endif
constexpr uint32_t kL1Drop = LD_L1_DROP;   // level-1 threshold step below a missed band (key units)

__device__ __forceinline__ uint32_t vload(const uint32_t* p) { return *reinterpret_cast<volatile const uint32_t*>(p); }

// queue a refill of the layer at `level` (1: rescan at thr_used, 2: every element, read directly)
__device__ void queue_refill(const DevPlan& P, int slot, int level, int lane) {
  uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
  for (int b = lane; b < kH0; b += 32) hrow[b] = 0;
  if (lane == 0) {
    P.layer_total[slot] = 0;   // the rescan recounts
    const uint32_t at = atomicAdd(&P.counters[level == 1 ? 0 : 4], 1u);
    (level == 1 ? P.refill_list : P.refill_list2)[at] = (uint32_t)slot;
    P.trace[slot] = (uint32_t)level;
  }
}

// mode 0: after the first pass -- hit: digit 0; miss: queue a level-1 (or level-2) refill
// mode 1: after a rescan -- level 1 hit: digit 0; level 1 still short: queue level 2; level 2: digit 0
// mode 2/3: digit 1/2 (mode 2 also predicts the next call's band)
__device__ void find_layer(const DevPlan& P, int slot, int mode, int lane) {
  const int li = P.large_layers[slot];
  const uint32_t k = P.layer_k[li];
  LayerSel& S = P.sel[slot];
  uint32_t* hrow = P.hist + (uint64_t)slot * kHistRow;
  if (mode == 0) {
    const uint32_t tot = vload(P.layer_total + slot);
    if (tot >= k) {
      uint32_t bin, above;
      warp_find_bin(hrow, kH0, k, &bin, &above);
      if (lane == 0) {
        S.prefix = bin; S.kleft = k - above; S.total = tot; S.refill = 0;
        P.thr_used[slot] = min(P.thr[slot], 0x7F800000u);
        P.trace[slot] = 0;
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
      // missed.  Level 1 rescans at the safe threshold (this distribution's band, without the
      // drift share) when that is lower than the one that missed, else at the missed threshold
      // lowered by a quarter binade (x0.75-0.875 in value); level 2 (every element) only when
      // neither exists.
      const uint32_t th = P.thr[slot], ts = P.thr_safe[slot];
      uint32_t l1 = 0xFFFFFFFFu;
      if (ts < th) l1 = ts;
      else if (th != 0xFFFFFFFFu && th > kL1Drop) l1 = min(th, 0x7F800000u) - kL1Drop;
      const int level = l1 != 0xFFFFFFFFu ? 1 : 2;
      if (lane == 0) {
        P.thr_used[slot] = level == 1 ? min(l1, 0x7F800000u) : 0u;
        S.refill = (uint32_t)level;
        S.total = (uint32_t)(P.layer_off[li + 1] - P.layer_off[li]);
        S.alpha *= 0.5f;                          // the drift prediction overshot
        if (level == 2) S.band = S.band > 0.f ? fminf(4.f, S.band * 2.f) : kBandAim;   // widen
        atomicAdd(&P.counters[2], 1u);
      }
      queue_refill(P, slot, level, lane);
    }
  } else if (mode == 1) {
    const uint32_t tot = vload(P.layer_total + slot);
    if (S.refill == 1 && tot < k) {
      if (lane == 0) {
        P.thr_used[slot] = 0u;
        S.refill = 2;
        S.band = S.band > 0.f ? fminf(4.f, S.band * 2.f) : kBandAim;
      }
      queue_refill(P, slot, 2, lane);
    } else {
      uint32_t bin, above;
      warp_find_bin(hrow, kH0, k, &bin, &above);
      if (lane == 0) { S.prefix = bin; S.kleft = k - above; S.total = tot; }
    }
  } else {
    const int nb = mode == 2 ? kH1 : kH2;
    const uint32_t* h = hrow + (mode == 2 ? kH0 : kH0 + kH1);
    uint32_t bin, above;
    warp_find_bin(h, nb, S.kleft, &bin, &above);
    if (mode == 2) {
      // Speculative band for the next call: the key with C = band x k_l candidate keys at or above
      // it (digit-0 resolution, refined with the digit-1 histogram when C falls in T's digit-0
      // bin).  Only a prediction -- the next call checks #candidates >= k_l and refills otherwise.
      const float band = S.band > 0.f ? S.band : kBandAim;
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
      // drift share: under error feedback the k-th key moved from T_{t-1} (sel_T, still the previous
      // call's) to T_t (>= the digit-1 prefix); lead the next band by alpha x the smaller of this
      // drift and the previous call's, so a T that alternates gets no lead
      const uint32_t t_lo = ((S.prefix << 11) | bin) << 9;
      const uint32_t t_prev = P.sel_T[slot];
      const uint32_t d_now = (t_prev != 0xFFFFFFFFu && t_lo > t_prev) ? t_lo - t_prev : 0u;
      const uint32_t d = min(d_now, S.drift);
      uint32_t na = nt;
      if (d > 0 && nt != 0xFFFFFFFFu) {
        const float a = fmaxf(0.f, fminf(0.5f, S.alpha));
        na = nt + (uint32_t)(a * (float)d);
        na = min(na, 0x7F800000u);
      }
      if (lane == 0) { S.next_thr = na; S.next_safe = nt; S.drift = d_now; }
    }
    if (lane == 0) { S.prefix = (S.prefix << (mode == 2 ? 11 : 9)) | bin; S.kleft -= above; }
  }
}

// Rescan one segment of a refilled layer: level 1 stores the candidates >= thr_used (bounded, as
// the scan); level 2 stores nothing (every element is a candidate, read directly later).  Both add
// the digit-0 bins and the count to the CTA's shared histogram h0 / counter cnt_sh.
template <bool EF>
__device__ void rescan_segment(const DevPlan& P, const float* __restrict__ g, float* __restrict__ r, int slot,
                               int ch, int seg, int level, uint64_t* sbuf, uint32_t* h0, uint32_t* cnt_sh, int lane) {
  const uint64_t segid = (uint64_t)ch * kSegsPerChunk + seg;
  if (level == 2) {
    uint32_t cnt = 0;
    visit_direct(P, EF ? r : g, ch, seg, 0u, lane, [&](bool ok, uint32_t bits, uint32_t) {
      warp_hist_add(h0, ok, (bits >> 20) & 0x7FFu);
      cnt += ok;
    });
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    if (lane == 0) {
      P.seg_count[segid] = cnt | kDirect;
      if (cnt) atomicAdd(cnt_sh, cnt);
      P.dlist[atomicAdd(&P.counters[5], 1u)] = (uint32_t)segid | (2u << 30);   // DIRECT, level 2
    }
    return;
  }
  const uint64_t cbase = P.chunk_base[ch];
  const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
  const uint32_t cs = (uint32_t)P.cs;
  const uint32_t sb = (uint32_t)seg * kSeg;
  const unsigned lt = (1u << lane) - 1u;
  bool bad = false;
  const uint32_t run = scan_segment<EF, true, false, true>(g + cbase, r + cbase, seg_slot(P, segid), cs, h0, sbuf, sb,
                                                           lo, hi, (uint32_t)cbase, P.thr_used[slot], 0xFFFFFFFFu, 0u,
                                                           lane, lt, bad);
  if (lane == 0) {
    P.seg_count[segid] = run > cs ? (run | kDirect) : run;
    if (run) atomicAdd(cnt_sh, run);
    if (run > cs) P.dlist[atomicAdd(&P.counters[5], 1u)] = (uint32_t)segid | (1u << 30);   // DIRECT, level 1
  }
}

// ---------------------------------------------------------------- the persistent select kernel
// One cooperative launch after the scan (grid = co-resident CTAs), phases separated by grid
// barriers.  CTA b owns the contiguous chunk range [cb, ce) for the streaming phases and walks it
// in WINDOWS of at most kWin chunks of one layer.  The first pass COMPACTS each window in place:
// its 16 kWin segment counts go to shared memory and are prefix-summed, the stored candidates are
// read as one flat, index-ordered list (item j -> its segment by binary search over the prefix) and
// written back contiguously at the window's start (a candidate never moves up; each round loads
// before it stores), histogramming digit 0 on the way.  Every later pass then streams the window's
// contiguous list with 128-bit loads, many in flight per thread.  DIRECT segments (more candidates
// than their slot, or level-2 layers) stay out of the list and are read from acc by warps.
// Histograms aggregate per window in shared memory; the per-chunk counts are prefix-summed per
// layer run inside the CTA, and only the CTA's last run is published (tail) for later CTAs of the
// same layer (reduce-then-scan); the ordered emit scans the window's flags block-wide.
constexpr int kWin = kSelThreads;     // chunks per window (one per thread at setup)
constexpr int kStreamV = 4;           // 128-bit loads (2 candidates each) in flight per thread and round
constexpr int kStreamItems = 2 * kStreamV;

struct SelShared {
  uint32_t hist[kH0];
  uint32_t pre[kWin * kSegsPerChunk];   // compaction: exclusive prefix of the window's stored segment counts
  uint32_t cst[kWin + 1];               // window-relative start of each chunk's compacted candidates
  uint32_t dm[kWin];                    // DIRECT-segment bitmask per chunk
  uint32_t cw0[kWin], cw1[kWin];        // per chunk: counts (count pass) / window starts (emit)
  uint32_t take[kWin];                  // emit: ties to take | 0x80000000 if the layer's last tie is here
  uint32_t dst[kWin];                   // emit: output offset of the chunk's first entry
  uint32_t sw[33];
  uint32_t cnt, lvl;
  unsigned long long head;
};

// per-chunk metadata written by the select kernel (global, [n_chunks] each): cpos = absolute offset
// (in candidates) of the chunk's compacted stored list, ccnt its length, cgt / ceq its counts of
// key > T / key == T (stored + DIRECT), cgtb / ceqb their exclusive prefixes inside the CTA's range
struct ChunkMeta {
  uint32_t *cpos, *ccnt, *cgt, *ceq, *cgtb, *ceqb;
};
__device__ __forceinline__ ChunkMeta chunk_meta(const DevPlan& P) {
  uint32_t* b = reinterpret_cast<uint32_t*>(P.chunk_state);
  const uint32_t n = (uint32_t)P.n_chunks;
  return ChunkMeta{b, b + n, b + 2 * n, b + 3 * n, b + 4 * n, b + 5 * n};
}

// iterate the CTA's range in windows of one layer: body(a, n, slot)
template <class B>
__device__ __forceinline__ void for_windows(const DevPlan& P, int cb, int ce, B&& body) {
  for (int a = cb; a < ce;) {
    const int slot = P.chunk_slot[a];
    const int z = min(min(ce, P.large_chunk0[slot + 1]), a + kWin);
    body(a, z - a, slot);
    a = z;
  }
}

// window setup after compaction: sh.cst (window-relative chunk starts), sh.dm (DIRECT masks);
// returns the window's stored total
__device__ uint32_t win_meta(const DevPlan& P, const ChunkMeta& M, int a, int n, SelShared& sh) {
  const int t = threadIdx.x;
  const uint32_t wbase = (uint32_t)a * kSegsPerChunk * (uint32_t)P.cs;
  if (t < n) {
    sh.cst[t] = M.cpos[a + t] - wbase;
    uint32_t dm = 0;
    const uint4* q = reinterpret_cast<const uint4*>(P.seg_count + (uint64_t)(a + t) * kSegsPerChunk);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 v = q[i];
      dm |= (((v.x & kDirect) ? 1u : 0u) | ((v.y & kDirect) ? 2u : 0u) | ((v.z & kDirect) ? 4u : 0u) |
             ((v.w & kDirect) ? 8u : 0u)) << (4 * i);
    }
    sh.dm[t] = dm;
    if (t == n - 1) sh.cst[n] = M.cpos[a + t] + M.ccnt[a + t] - wbase;
  }
  __syncthreads();
  return sh.cst[n];
}

// chunk (window-relative) of compacted item j: the largest c with cst[c] <= j (a non-empty chunk)
__device__ __forceinline__ int win_chunk(const SelShared& sh, int n, uint32_t j) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sh.cst[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// the window's compacted candidates L[0, total), kStreamItems contiguous per thread per round:
// f(ok, val_bits, idx, j) -- all threads call f equally often (warp-convergent)
template <class F>
__device__ __forceinline__ void win_stream(const uint64_t* __restrict__ L, uint32_t total, F&& f) {
  for (uint32_t r0 = 0; r0 < total; r0 += kSelThreads * kStreamItems) {
    const uint32_t j0 = r0 + threadIdx.x * kStreamItems;
    uint64_t v[kStreamItems];
    if (j0 + kStreamItems <= total) {
      const uint4* q = reinterpret_cast<const uint4*>(L + j0);
#pragma unroll
      for (int u = 0; u < kStreamV; ++u) {
        const uint4 x = __ldcg(q + u);
        v[2 * u] = ((uint64_t)x.y << 32) | x.x;
        v[2 * u + 1] = ((uint64_t)x.w << 32) | x.z;
      }
    } else {
#pragma unroll
      for (int u = 0; u < kStreamItems; ++u) v[u] = j0 + u < total ? L[j0 + u] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kStreamItems; ++u) f(j0 + u < total, (uint32_t)(v[u] >> 32), (uint32_t)v[u], j0 + u);
  }
}

// Every valid DIRECT segment of the call, grid-wide, one segment per CTA round (thread t reads the
// segment's float4 t): f(ok, key_bits, idx, chunk, slot) for each thread's 4 elements (CTA-uniform
// control flow).  An entry is valid when its level equals the layer's final refill level (entries
// of a layer that was rescanned afterwards are stale); any_level: every entry (the first pass, before
// this call's plan).  thr: the layer's threshold of that level.
static_assert(kSeg == 4 * kSelThreads, "direct_all: one float4 of the segment per thread");
template <class F>
__device__ __forceinline__ void direct_all(const DevPlan& P, const float* __restrict__ src, bool any_level, F&& f) {
  const uint32_t nd = vload(P.counters + 5);
  const int t = threadIdx.x;
  for (uint32_t e = blockIdx.x; e < nd; e += gridDim.x) {
    const uint32_t w = P.dlist[e];
    const uint32_t segid = w & 0x3FFFFFFFu, lvl = w >> 30;
    const int ch = (int)(segid / kSegsPerChunk), seg = (int)(segid % kSegsPerChunk);
    const int slot = P.chunk_slot[ch];
    if (!any_level && lvl != P.sel[slot].refill) continue;   // uniform over the CTA
    const uint32_t thr = any_level ? min(P.thr[slot], 0x7F800000u) : P.thr_used[slot];
    const uint64_t cbase = P.chunk_base[ch];
    const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
    const float* sp = src + cbase;
    const uint32_t e0 = (uint32_t)seg * kSeg + 4u * (uint32_t)t;   // kSeg = 4 x kSelThreads
    uint32_t vm = 0;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 >= lo && e0 + 4 <= hi) {
      vm = 0xF;
      a = *reinterpret_cast<const float4*>(sp + e0);
    } else if (e0 + 4 > lo && e0 < hi) {
      for (int k = 0; k < 4; ++k)
        if (e0 + k >= lo && e0 + k < hi) { vm |= 1u << k; f4set(a, k, sp[e0 + k]); }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t bits = __float_as_uint(f4get(a, k));
      f(((vm >> k) & 1u) && (bits & 0x7FFFFFFFu) >= thr, bits, (uint32_t)cbase + e0 + k, ch, slot);
    }
  }
}

// In-place compaction of window (a, n) + digit-0 histogram of its stored candidates into the
// layer's global row and their count into layer_total; per-chunk cpos / ccnt (and cgt / ceq
// zeroed).  The window's segment slots are contiguous, so its compacted list starts at
// seg_slot(a * 16): a candidate never moves up, and each round loads before it stores.
__device__ void compact_window(const DevPlan& P, const ChunkMeta& M, int a, int n, int slot, bool hist,
                               SelShared& sh, int lane) {
  const int t = threadIdx.x;
  if (hist)
    for (int i = t; i < kH0; i += kSelThreads) sh.hist[i] = 0;
  if (t == 0) sh.cnt = 0;
  uint32_t c[kSegsPerChunk], sum = 0;
  if (t < n) {
    const uint4* q = reinterpret_cast<const uint4*>(P.seg_count + (uint64_t)(a + t) * kSegsPerChunk);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 v = q[i];
      c[4 * i] = v.x; c[4 * i + 1] = v.y; c[4 * i + 2] = v.z; c[4 * i + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < kSegsPerChunk; ++i) {
      c[i] = (c[i] & kDirect) ? 0u : c[i];
      sum += c[i];
    }
  }
  uint32_t total;
  uint32_t run = block_excl_scan(sum, sh.sw, &total);   // (its barriers also order the zeroing)
  const uint32_t cs = (uint32_t)P.cs;
  if (t < n) {
    M.cpos[a + t] = (uint32_t)a * kSegsPerChunk * cs + run;
    M.ccnt[a + t] = sum;
    M.cgt[a + t] = 0;
    M.ceq[a + t] = 0;
#pragma unroll
    for (int i = 0; i < kSegsPerChunk; ++i) { sh.pre[t * kSegsPerChunk + i] = run; run += c[i]; }
  }
  __syncthreads();
  const int nseg = n * kSegsPerChunk;
  uint64_t* L = seg_slot(P, (uint64_t)a * kSegsPerChunk);
  constexpr int U = kStreamItems;
  for (uint32_t r0 = 0; r0 < total; r0 += kSelThreads * U) {
    const uint32_t j0 = r0 + t * U;
    uint64_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = 0ull;
    if (j0 < total) {
      int lo = 0, hi = nseg;   // segment of j0: the largest s with pre[s] <= j0
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sh.pre[mid] <= j0) lo = mid; else hi = mid;
      }
      int s = lo;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u;
        if (j < total) {
          while (s + 1 < nseg && sh.pre[s + 1] <= j) ++s;
          v[u] = L[(uint32_t)s * cs + (j - sh.pre[s])];
        }
      }
    }
    __syncthreads();   // every source of this round is read before any of its destinations is written
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = j0 + u < total;
      if (ok) L[j0 + u] = v[u];
      if (hist) warp_hist_add(sh.hist, ok, (uint32_t)(v[u] >> 52) & 0x7FFu);
    }
    __syncthreads();
  }
  if (hist) {
    uint32_t* hg = P.hist + (uint64_t)slot * kHistRow;
    for (int i = t; i < kH0; i += kSelThreads)
      if (sh.hist[i]) atomicAdd(&hg[i], sh.hist[i]);
    if (t == 0 && total) atomicAdd(&P.layer_total[slot], total);   // stored candidates admitted
    __syncthreads();
  }
}

// digit d = 1 / 2 histogram (key bits [19:9] / [8:0]) of the window's stored candidates matching the prefix
__device__ void digit_window(const DevPlan& P, const ChunkMeta& M, int d, int a, int n, int slot, SelShared& sh) {
  const int nb = d == 1 ? kH1 : kH2, shift = d == 1 ? 9 : 0, hs = d == 1 ? 20 : 9;
  const uint32_t mask = d == 1 ? 0x7FFu : 0x1FFu;
  for (int i = threadIdx.x; i < nb; i += kSelThreads) sh.hist[i] = 0;
  const uint32_t total = win_meta(P, M, a, n, sh);
  const uint32_t pre = P.sel[slot].prefix;
  win_stream(seg_slot(P, (uint64_t)a * kSegsPerChunk), total, [&](bool ok, uint32_t bits, uint32_t, uint32_t) {
    const uint32_t key = bits & 0x7FFFFFFFu;
    warp_hist_add(sh.hist, ok && (key >> hs) == pre, (key >> shift) & mask);
  });
  __syncthreads();
  uint32_t* hg = P.hist + (uint64_t)slot * kHistRow + (d == 1 ? kH0 : kH0 + kH1);
  for (int i = threadIdx.x; i < nb; i += kSelThreads)
    if (sh.hist[i]) atomicAdd(&hg[i], sh.hist[i]);
  __syncthreads();
}

// Ordered emit of a chunk with a DIRECT segment (warp): its segments in index order -- the stored
// ones from its compacted run Lc (segment after segment), the DIRECT ones from acc.  dst0 = output
// offset of its first entry; it takes `take` of its ties (lowest index first).
__device__ void emit_dirty_chunk(const DevPlan& P, const float* __restrict__ src, int ch, const uint64_t* Lc,
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
  const uint64_t cbase = P.chunk_base[ch];
  const uint32_t lo = (uint32_t)(P.chunk_lo[ch] - cbase), hi = (uint32_t)(P.chunk_hi[ch] - cbase);
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

// phase timestamps of the select kernel (block 0, %globaltimer ns): lowdiff_compress_phases
__device__ __forceinline__ void phase_mark(const DevPlan& P, int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.phase_ns[i] = t;
  }
}

// the CTA that owns chunk ch in the select's static partition (cb(b) = floor(n_chunks b / G))
__device__ __forceinline__ int owner_cta(int ch, int n_chunks, int G) {
  int b = (int)(((int64_t)ch * G) / n_chunks);
  while (b + 1 < G && (int)((int64_t)n_chunks * (b + 1) / G) <= ch) ++b;
  while (b > 0 && (int)((int64_t)n_chunks * b / G) > ch) --b;
  return b;
}

#ifndef LD_SEL_MINB
#define LD_SEL_MINB 3
#endif

template <bool EF>
__global__ void __launch_bounds__(kSelThreads, LD_SEL_MINB)
select_kernel(DevPlan P, const float* __restrict__ g, float* __restrict__ r, uint32_t* __restrict__ send, uint64_t K) {
  __shared__ uint64_t sbuf_all[kSelWarps][kCandBuf];
  __shared__ SelShared sh;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, t = threadIdx.x;
  const int gw = blockIdx.x * kSelWarps + warp, nw = gridDim.x * kSelWarps;
  const float* src = EF ? r : g;
  const ChunkMeta M = chunk_meta(P);
  const int cb = (int)((int64_t)P.n_chunks * blockIdx.x / gridDim.x);
  const int ce = (int)((int64_t)P.n_chunks * (blockIdx.x + 1) / gridDim.x);
  if (blockIdx.x == 0 && t < 16) P.phase_ns[t] = 0;   // phases not run stay 0
  __syncthreads();
  phase_mark(P, 0);
  // 1. compact every window in place + digit 0 of its stored candidates; digit 0 of the DIRECT
  //    segments' candidates grid-wide
  for_windows(P, cb, ce, [&](int a, int n, int slot) { compact_window(P, M, a, n, slot, true, sh, lane); });
  {
    uint32_t cnt = 0;
    int cur_slot = -1;
    direct_all(P, src, true, [&](bool ok, uint32_t bits, uint32_t, int, int slot) {
      warp_hist_add(P.hist + (uint64_t)slot * kHistRow, ok, (bits >> 20) & 0x7FFu);
      if (slot != cur_slot) {   // (uniform over the CTA: one segment per round)
        if (cur_slot >= 0) {
#pragma unroll
          for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
          if (lane == 0 && cnt) atomicAdd(&P.layer_total[cur_slot], cnt);
          cnt = 0;
        }
        cur_slot = slot;
      }
      cnt += ok;
    });
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    if (lane == 0 && cnt && cur_slot >= 0) atomicAdd(&P.layer_total[cur_slot], cnt);
  }
  grid.sync();
  phase_mark(P, 1);
  // 2. plan: per large layer, hit or refill
  for (int slot = gw; slot < P.n_large; slot += nw) find_layer(P, slot, 0, lane);
  grid.sync();
  phase_mark(P, 2);
  // 3. refills: level 1 (rescan at the safe threshold, stored), then level 2 (every element, DIRECT).
  // list 1: layers queued at level 1 by the plan; list 2: queued at level 2 by the plan, or still
  // short after their level-1 rescan (appended by find_layer mode 1 in pass 0)
  for (int pass = 0; pass < 2; ++pass) {
    const uint32_t n_ref = vload(P.counters + (pass == 0 ? 0 : 4));
    if (n_ref == 0) continue;   // uniform: every thread reads the same value after the barrier
    const uint32_t* list = pass == 0 ? P.refill_list : P.refill_list2;
    for (uint32_t i = 0; i < n_ref; ++i) {   // layer by layer; its segments over the whole grid
      const int slot = (int)list[i];
      const int c0 = P.large_chunk0[slot], c1 = P.large_chunk0[slot + 1];
      const int nseg = (c1 - c0) * kSegsPerChunk;
      for (int b = t; b < kH0; b += kSelThreads) sh.hist[b] = 0;
      if (t == 0) sh.cnt = 0;
      __syncthreads();
      for (int s = gw; s < nseg; s += nw)
        rescan_segment<EF>(P, g, r, slot, c0 + s / kSegsPerChunk, s % kSegsPerChunk, pass + 1, sbuf_all[warp],
                           sh.hist, &sh.cnt, lane);
      __syncthreads();
      uint32_t* hg = P.hist + (uint64_t)slot * kHistRow;
      for (int b = t; b < kH0; b += kSelThreads)
        if (sh.hist[b]) atomicAdd(&hg[b], sh.hist[b]);
      if (t == 0 && sh.cnt) atomicAdd(&P.layer_total[slot], sh.cnt);
      __syncthreads();
    }
    grid.sync();
    phase_mark(P, 3 + 2 * pass);
    // re-compact the rescanned windows (their histogram is complete), then plan.  The level is read
    // once per CTA: another CTA's plan below may already escalate the layer (1 -> 2), and every
    // thread of the CTA must take the same branch; an escalated layer is re-compacted in pass 1.
    for_windows(P, cb, ce, [&](int a, int n, int slot) {
      if (t == 0) sh.lvl = P.sel[slot].refill;
      __syncthreads();
      const uint32_t lvl = sh.lvl;
      __syncthreads();
      if (lvl == (uint32_t)(pass + 1)) compact_window(P, M, a, n, slot, false, sh, lane);
    });
    for (uint32_t i = gw; i < n_ref; i += nw) find_layer(P, (int)list[i], 1, lane);
    grid.sync();
    phase_mark(P, 4 + 2 * pass);
  }
  // 4. digits 1 and 2 over the candidates matching the prefix
  for (int d = 1; d <= 2; ++d) {
    const int shift = d == 1 ? 9 : 0, hs = d == 1 ? 20 : 9;
    const uint32_t mask = d == 1 ? 0x7FFu : 0x1FFu;
    for_windows(P, cb, ce, [&](int a, int n, int slot) { digit_window(P, M, d, a, n, slot, sh); });
    direct_all(P, src, false, [&](bool ok, uint32_t bits, uint32_t, int, int slot) {
      const uint32_t key = bits & 0x7FFFFFFFu;
      warp_hist_add(P.hist + (uint64_t)slot * kHistRow + (d == 1 ? kH0 : kH0 + kH1),
                    ok && (key >> hs) == P.sel[slot].prefix, (key >> shift) & mask);
    });
    grid.sync();
    phase_mark(P, 5 + 2 * d);
    for (int slot = gw; slot < P.n_large; slot += nw) find_layer(P, slot, d == 1 ? 2 : 3, lane);
    grid.sync();
    phase_mark(P, 6 + 2 * d);
  }
  // 5. counts per chunk (key > T, key == T): stored per window, DIRECT grid-wide (both add)
  for_windows(P, cb, ce, [&](int a, int n, int slot) {
    if (t < n) { sh.cw0[t] = 0; sh.cw1[t] = 0; }
    const uint32_t total = win_meta(P, M, a, n, sh);
    const uint32_t T = P.sel[slot].prefix;
    int cc = 0;
    uint32_t last_j0 = 0xFFFFFFFFu;
    win_stream(seg_slot(P, (uint64_t)a * kSegsPerChunk), total, [&](bool ok, uint32_t bits, uint32_t, uint32_t j) {
      if (ok) {   // items are contiguous per thread: the chunk of the first by binary search, then advance
        const uint32_t j0 = j - (j % kStreamItems);
        if (j0 != last_j0) { cc = win_chunk(sh, n, j); last_j0 = j0; }
        while (cc + 1 < n && sh.cst[cc + 1] <= j) ++cc;
      }
      const uint32_t key = bits & 0x7FFFFFFFu;
      const bool gt = ok && key > T, eq = ok && key == T;
      const unsigned act = __ballot_sync(0xFFFFFFFFu, gt || eq);
      if (gt || eq) {
        const unsigned peers = __match_any_sync(act, cc);
        const unsigned ng = __popc(__ballot_sync(act, gt) & peers), ne = __popc(__ballot_sync(act, eq) & peers);
        if (lane == __ffs(peers) - 1) {
          if (ng) atomicAdd(&sh.cw0[cc], ng);
          if (ne) atomicAdd(&sh.cw1[cc], ne);
        }
      }
    });
    __syncthreads();
    if (t < n) {
      if (sh.cw0[t]) atomicAdd(&M.cgt[a + t], sh.cw0[t]);
      if (sh.cw1[t]) atomicAdd(&M.ceq[a + t], sh.cw1[t]);
    }
    __syncthreads();
  });
  {
    uint32_t gtc = 0, eqc = 0;
    int cur = -1;
    auto flush = [&]() {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        gtc += __shfl_xor_sync(0xFFFFFFFFu, gtc, o);
        eqc += __shfl_xor_sync(0xFFFFFFFFu, eqc, o);
      }
      if (lane == 0 && cur >= 0) {
        if (gtc) atomicAdd(&M.cgt[cur], gtc);
        if (eqc) atomicAdd(&M.ceq[cur], eqc);
      }
      gtc = eqc = 0;
    };
    direct_all(P, src, false, [&](bool ok, uint32_t bits, uint32_t, int ch, int slot) {
      if (ch != cur) { flush(); cur = ch; }   // (uniform over the CTA)
      const uint32_t key = bits & 0x7FFFFFFFu, T = P.sel[slot].prefix;
      gtc += ok && key > T;
      eqc += ok && key == T;
    });
    flush();
  }
  grid.sync();
  phase_mark(P, 11);
  // 6. in-CTA exclusive scan of the counts, restarting at every layer boundary; the CTA's last
  //    run's total is published for the CTAs after it (reduce-then-scan)
  if (warp == 0) {
    unsigned long long carry = 0;
    int cur = -1;
    for (int a = cb; a < ce; a += 32) {
      const int ch = a + lane;
      const bool in = ch < ce;
      const int slot = in ? P.chunk_slot[ch] : -1;
      const unsigned long long v = in ? (((unsigned long long)M.ceq[ch] << 31) | M.cgt[ch]) : 0ull;
      // segmented inclusive scan (segments = layer runs; slots ascend with the chunk index):
      // (x, fx) + (y, fy) = (fy ? y : x + y, fx | fy)
      const int prev = __shfl_up_sync(0xFFFFFFFFu, slot, 1);
      bool f = in && (lane == 0 ? slot != cur : slot != prev);
      unsigned long long inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        const bool fy = __shfl_up_sync(0xFFFFFFFFu, f, o);
        if (lane >= o) {
          if (!f) inc += y;
          f = f || fy;
        }
      }
      if (!f) inc += carry;   // no run start in [round start, lane]: continues the previous round's run
      const unsigned long long exc = inc - v;
      if (in) {
        M.cgtb[ch] = (uint32_t)(exc & 0x7FFFFFFFull);
        M.ceqb[ch] = (uint32_t)(exc >> 31);
      }
      const int last = min(31, ce - 1 - a);
      carry = __shfl_sync(0xFFFFFFFFu, inc, last);
      cur = __shfl_sync(0xFFFFFFFFu, slot, last);
    }
    if (lane == 0) {
      P.tail_agg[blockIdx.x] = ce > cb ? carry : 0ull;        // the CTA's last run: its layer's partial sum
      P.tail_slot[blockIdx.x] = ce > cb ? (uint32_t)cur : 0xFFFFFFFEu;   // no chunks: transparent
    }
  }
  grid.sync();
  phase_mark(P, 12);
  // the CTA's first layer may have started in earlier CTAs: their published tails of that layer;
  // the full "before" counts of every chunk of the range are then written back (cgtb / ceqb)
  if (warp == 0) {
    unsigned long long head = 0;
    if (ce > cb) {
      const uint32_t slot0 = (uint32_t)P.chunk_slot[cb];
      if (P.large_chunk0[slot0] < cb) {
        for (int b = (int)blockIdx.x - 1; b >= 0; b -= 32) {
          const int q = b - lane;
          const uint32_t ts = q >= 0 ? P.tail_slot[q] : 0u;
          const bool same = q >= 0 && (ts == slot0 || ts == 0xFFFFFFFEu);
          const unsigned stop = __ballot_sync(0xFFFFFFFFu, !same);
          const int n_same = stop ? __ffs(stop) - 1 : 32;
          unsigned long long v = lane < n_same ? P.tail_agg[q] : 0ull;
#pragma unroll
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
          head += v;
          if (stop) break;
        }
      }
    }
    if (lane == 0) sh.head = head;
  }
  __syncthreads();
  {
    const unsigned long long head = sh.head;
    const int first_run_end = ce > cb ? min(ce, P.large_chunk0[P.chunk_slot[cb] + 1]) : cb;
    if (head)
      for (int ch = cb + t; ch < first_run_end; ch += kSelThreads) {
        const unsigned long long b = (((unsigned long long)M.ceqb[ch] << 31) | M.cgtb[ch]) + head;
        M.cgtb[ch] = (uint32_t)(b & 0x7FFFFFFFull);
        M.ceqb[ch] = (uint32_t)(b >> 31);
      }
  }
  const bool any_direct = vload(P.counters + 5) != 0;
  if (any_direct) grid.sync();   // the dirty-chunk emit below reads other CTAs' chunks (uniform)
  // 7. ordered emit: clean chunks block-parallel over the window's compacted list (flags scanned
  //    block-wide); chunks with a DIRECT segment by a warp each, grid-wide
  for_windows(P, cb, ce, [&](int a, int n, int slot) {
    const uint32_t T = P.sel[slot].prefix, need = P.sel[slot].kleft;
    uint32_t wgt = 0, weq = 0;
    if (t < n) {
      const int ch = a + t;
      const uint32_t gt_b = M.cgtb[ch], eq_b = M.ceqb[ch];
      const uint32_t take_b = min(eq_b, need);       // ties are taken in chunk order, then index order
      const uint32_t take = min(M.ceq[ch], need - take_b);
      const bool last_tie = take > 0 && take_b + take == need;
      sh.take[t] = take | (last_tie ? 0x80000000u : 0u);
      sh.dst[t] = (uint32_t)(P.layer_koff[P.large_layers[slot]] + gt_b + take_b);
      wgt = M.cgt[ch];
      weq = M.ceq[ch];
      if (ch == P.large_chunk0[slot]) {
        P.sel_T[slot] = T;
        // speculative band for the next call: the drift-led threshold (may exceed T)
        // and the safe one (never above this call's T) that a level-1 refill falls back to
        const uint32_t ns = P.sel[slot].next_safe;
        const uint32_t sf = ns <= T ? ns : T;
        P.thr_safe[slot] = sf;
        P.thr[slot] = max(sf, P.sel[slot].next_thr);
      }
    }
    const uint32_t total = win_meta(P, M, a, n, sh);
    if (t < n && sh.dm[t] != 0) { wgt = 0; weq = 0; }   // dirty chunks: emitted below
    uint32_t tot2;
    const uint32_t wsg = block_excl_scan(wgt, sh.sw, &tot2);
    const uint32_t wse = block_excl_scan(weq, sh.sw, &tot2);
    if (t < n) { sh.cw0[t] = wsg; sh.cw1[t] = wse; }
    __syncthreads();
    const uint64_t* L = seg_slot(P, (uint64_t)a * kSegsPerChunk);
    uint32_t g_run = 0, e_run = 0;   // clean gt / eq items of the window before this round
    for (uint32_t r0 = 0; r0 < total; r0 += kSelThreads * kStreamItems) {
      const uint32_t j0 = r0 + t * kStreamItems;
      uint64_t v[kStreamItems];
      if (j0 + kStreamItems <= total) {
        const uint4* q = reinterpret_cast<const uint4*>(L + j0);
#pragma unroll
        for (int u = 0; u < kStreamV; ++u) {
          const uint4 x = __ldcg(q + u);
          v[2 * u] = ((uint64_t)x.y << 32) | x.x;
          v[2 * u + 1] = ((uint64_t)x.w << 32) | x.z;
        }
      } else {
#pragma unroll
        for (int u = 0; u < kStreamItems; ++u) v[u] = j0 + u < total ? L[j0 + u] : 0ull;
      }
      const int c0 = j0 < total ? win_chunk(sh, n, j0) : 0;
      int c = c0;
      uint32_t lg = 0, le = 0, skip = 0;
#pragma unroll
      for (int u = 0; u < kStreamItems; ++u) {
        const uint32_t j = j0 + u;
        const bool ok = j < total;
        if (ok)
          while (c + 1 < n && sh.cst[c + 1] <= j) ++c;
        const bool cl = ok && sh.dm[c] == 0;
        skip |= cl ? 0u : 1u << u;
        const uint32_t key = (uint32_t)(v[u] >> 32) & 0x7FFFFFFFu;
        lg += cl && key > T;
        le += cl && key == T;
      }
      uint32_t rtot;
      const uint32_t rex = block_excl_scan((le << 16) | lg, sh.sw, &rtot);
      uint32_t gbw = g_run + (rex & 0xFFFFu), ebw = e_run + (rex >> 16);   // before this thread's items
      c = c0;
#pragma unroll
      for (int u = 0; u < kStreamItems; ++u) {
        const uint32_t j = j0 + u;
        if (j < total)
          while (c + 1 < n && sh.cst[c + 1] <= j) ++c;
        const bool ok = !((skip >> u) & 1u);
        const uint32_t val = (uint32_t)(v[u] >> 32), key = val & 0x7FFFFFFFu;
        const bool gt = ok && key > T, eq = ok && key == T;
        if (gt || eq) {
          const uint32_t gb = gbw - sh.cw0[c], eb = ebw - sh.cw1[c];   // before it, inside its chunk
          const uint32_t tk = sh.take[c] & 0x7FFFFFFFu;
          if (gt || eb < tk) {
            const uint32_t o = sh.dst[c] + gb + min(eb, tk);
            send[o] = (uint32_t)v[u];
            send[K + o] = val;
          }
          if (eq && (sh.take[c] >> 31) && eb == tk - 1) P.sel_cut[slot] = (uint32_t)v[u] + 1;
        }
        gbw += gt;
        ebw += eq;
      }
      g_run += rtot & 0xFFFFu;
      e_run += rtot >> 16;
    }
    __syncthreads();
  });
  if (any_direct) {   // chunks with a DIRECT segment: the entry of the chunk's first DIRECT segment emits it
    const uint32_t nd = vload(P.counters + 5);
    for (uint32_t e = gw; e < nd; e += nw) {
      const uint32_t w = P.dlist[e];
      const uint32_t segid = w & 0x3FFFFFFFu, lvl = w >> 30;
      const int ch = (int)(segid / kSegsPerChunk), seg = (int)(segid % kSegsPerChunk);
      const int slot = P.chunk_slot[ch];
      if (lvl != P.sel[slot].refill) continue;
      const uint32_t sc = lane < kSegsPerChunk ? P.seg_count[(uint64_t)ch * kSegsPerChunk + lane] : 0u;
      const unsigned dmask = __ballot_sync(0xFFFFFFFFu, (sc & kDirect) != 0u) & 0xFFFFu;
      if (__ffs(dmask) - 1 != seg) continue;
      const uint32_t T = P.sel[slot].prefix, need = P.sel[slot].kleft;
      const uint32_t take_b = min(M.ceqb[ch], need);
      const uint32_t take = min(M.ceq[ch], need - take_b);
      const bool last_tie = take > 0 && take_b + take == need;
      const uint64_t dst0 = P.layer_koff[P.large_layers[slot]] + M.cgtb[ch] + take_b;
      emit_dirty_chunk(P, src, ch, P.cand + M.cpos[ch], send, K, dst0, T, take, last_tie, slot, lane);
    }
  }
  __syncthreads();
  phase_mark(P, 15);
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

// per-segment candidate capacity: ~12 x the expected candidates of a 1024-element segment at the
// band's ~1.5 k_l (a power of two in [32, 1024]); 1 B/param of scratch at 1% density
int compress_seg_capacity(uint32_t ppm) {
  const double want = 12.0 * kSeg * (double)ppm / 1e6;
  int cs = 32;
  while (cs < 1024 && cs < want) cs <<= 1;
  return cs;
}

// co-resident CTAs of the select kernel (cooperative launch), at most 4 per SM
static unsigned select_grid(bool ef) {
  static int occ[2] = {0, 0};
  if (!occ[ef]) {
    int o = 0;
    if (ef) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, select_kernel<true>, kSelThreads, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, select_kernel<false>, kSelThreads, 0);
    occ[ef] = std::max(1, std::min(4, o));
  }
  return (unsigned)std::min(kMaxSelGrid, num_sms() * occ[ef]);
}

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
    // they run on a forked stream, concurrently with the scan, and join before the select
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
  // per-call state: digit histograms, per-layer candidate totals, counters
  if ((e = cudaMemsetAsync(P.hist, 0, compress_hist_bytes(P.n_large), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(P.layer_total, 0, (size_t)P.n_large * 4, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(P.counters, 0, 8 * sizeof(uint32_t), s)) != cudaSuccess) return e;
  const unsigned scan_grid = (unsigned)P.n_chunks * kPiecesPerChunk;
  // lazy residual zeroing applies only to the residual buffer whose selection is pending
  const int lazy = (ef && c->lazy_residual == residual) ? 1 : 0;
  prof_begin(c, "scan", s, &h);
  if (ef) scan_kernel<true><<<scan_grid, kScanWarps * 32, 0, s>>>(P, grad, residual, lazy);
  else scan_kernel<false><<<scan_grid, kScanWarps * 32, 0, s>>>(P, grad, residual, 0);
  prof_end(c, h, s);
  if (P.n_small && c->aux && (e = cudaStreamWaitEvent(s, c->ev_join, 0)) != cudaSuccess) return e;   // join
  prof_begin(c, "select", s, &h);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(select_grid(ef));
    cfg.blockDim = dim3(kSelThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint64_t K = (uint64_t)c->K;
    e = ef ? cudaLaunchKernelEx(&cfg, select_kernel<true>, P, grad, residual, send, K)
           : cudaLaunchKernelEx(&cfg, select_kernel<false>, P, grad, residual, send, K);
    if (e != cudaSuccess) return e;
  }
  prof_end(c, h, s);
  c->launches += 2;
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
