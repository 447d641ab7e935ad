// Merge (decompress) and fused multi-step replay on sm_100a.
//
// merge  -- Alg. 1 line 7 "Comp^-1" after the allgather "Sync":
//           G[j] = ((+0 + v_0[j]) + v_1[j] + ... + v_{N-1}[j]) / N, rank order, IEEE divide
//           (R-8).  Tile-gather: every CTA owns a tile of the dense output, sums the
//           entries that fall in it rank by rank in shared memory (indices are unique within a
//           rank, so a rank's adds never collide) and writes the tile once with 128-bit stores.
//           No atomics -> bit-deterministic for any N.  The per-(block, tile) entry ranges come
//           from one linear pass over the (globally ascending) index lists.
// replay -- Alg. 1 recovery loop, Eq. 1 update, dense Adam
//           (R-10) or SGD (R-12), fused over steps: every CTA keeps its tile of (p, m, v) in
//           registers, rebuilds G_t for the tile in shared memory exactly as the merge does,
//           applies the update with block t's stored scalars, and writes the tile once at the
//           end.  Per element this is the sequential recurrence, in order -- bit-identical to
//           applying the steps one by one (the paper's log-n pairwise merge, is not
//           exact for Adam; R-16).
// All float operations are explicit round-to-nearest intrinsics (no FMA contraction, no
// fast-math, denormals preserved; R-20/R-21).
#include <cuda_runtime.h>

#include "ieee_fast.cuh"
#include "internal.h"
#include "pdl.cuh"

namespace ld {
namespace {

// start[b][t - T0] = lower_bound(idx_b, t * 2^tile_shift) for t = T0..T1 (idx_b ascending).
// Entry e owns the tiles (tile(idx[e-1]), tile(idx[e])]; grid.y walks the blocks (no 64-bit division).
// ranges (optional, u32[2 * n_blocks]): only entries [a_b, b_b) of block b are valid (the rest of
// the block was not uploaded); the tiles before the first valid entry get a_b, those after the last
// get b_b.  Entries outside the range lie outside the element range being replayed.
#ifndef LD_TS_UNROLL
#define LD_TS_UNROLL 4
#endif
__global__ void tile_start_kernel(const uint32_t* __restrict__ blocks, int64_t n_blocks, uint64_t stride,
                                  uint32_t K, int tile_shift, uint32_t T0, uint32_t T1,
                                  const uint32_t* __restrict__ ranges, uint32_t* __restrict__ start) {
  pdl_trigger();   // the merge may be scheduled now (it waits for this grid before reading start)
  const uint32_t W = T1 - T0 + 1;
  for (int64_t b = blockIdx.y; b < n_blocks; b += gridDim.y) {
    const uint32_t* idx = blocks + (uint64_t)b * stride;
    uint32_t* st = start + (uint64_t)b * W;
    const uint32_t ea = ranges ? __ldg(ranges + 2 * b) : 0u;
    const uint32_t eb = ranges ? __ldg(ranges + 2 * b + 1) : K;
    auto owned = [&](uint32_t e, uint32_t prev, uint32_t cur) {   // the tiles entry e starts
      uint32_t t_lo = e == ea ? T0 : (prev >> tile_shift) + 1;
      uint32_t t_hi = e == eb ? T1 : (cur >> tile_shift);
      t_lo = max(t_lo, T0);
      t_hi = min(t_hi, T1);
      for (uint32_t t = t_lo; t <= t_hi; ++t) st[t - T0] = e;
    };
    const uint32_t nthr = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
    // entries [ea, eb) are real, eb is the sentinel (the tiles after the last entry).  The 16-byte
    // aligned middle [p0, p1) goes four entries per 128-bit load, LD_TS_UNROLL groups in flight per
    // thread (one 32-bit entry at a time left the replay's index pass latency-bound: 4.7 ms for 100
    // GPT-2 XL blocks, 1.3 TB/s; four 32-bit loads in flight 3.1 ms); the unaligned head (< 4
    // entries), the tail and the sentinel go one entry per thread.
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(idx + ea) >> 2) & 3u);
    const uint32_t p0 = min(eb, ea + ((4u - mis) & 3u));
    const uint32_t ng = (eb - p0) / 4u, p1 = p0 + 4u * ng;
    for (uint32_t e = ea + tid; e < p0; e += nthr) owned(e, e == ea ? 0u : __ldg(idx + e - 1), __ldg(idx + e));
    for (uint32_t e = p1 + tid; e <= eb; e += nthr) owned(e, e == ea ? 0u : __ldg(idx + e - 1), e == eb ? 0u : __ldg(idx + e));
    const uint4* v4 = reinterpret_cast<const uint4*>(idx + p0);
    uint32_t gi = tid;
    for (; gi + (LD_TS_UNROLL - 1) * nthr < ng; gi += LD_TS_UNROLL * nthr) {
      uint4 cur[LD_TS_UNROLL];
      uint32_t prev[LD_TS_UNROLL];
#pragma unroll
      for (int q = 0; q < LD_TS_UNROLL; ++q) {
        const uint32_t g = gi + q * nthr, e = p0 + 4u * g;
        cur[q] = __ldg(v4 + g);
        prev[q] = e == ea ? 0u : __ldg(idx + e - 1);
      }
#pragma unroll
      for (int q = 0; q < LD_TS_UNROLL; ++q) {
        const uint32_t e = p0 + 4u * (gi + q * nthr);
        owned(e, prev[q], cur[q].x);
        owned(e + 1, cur[q].x, cur[q].y);
        owned(e + 2, cur[q].y, cur[q].z);
        owned(e + 3, cur[q].z, cur[q].w);
      }
    }
    for (; gi < ng; gi += nthr) {
      const uint4 c = __ldg(v4 + gi);
      const uint32_t e = p0 + 4u * gi;
      owned(e, e == ea ? 0u : __ldg(idx + e - 1), c.x);
      owned(e + 1, c.x, c.y);
      owned(e + 2, c.y, c.z);
      owned(e + 3, c.z, c.w);
    }
  }
}

// G = S / N.  DIV = 0: no division (sum mode, or N = 1 where x / 1 == x bit for bit);
// DIV = 1: N is a power of two, so x / N == x * 2^-log2(N) exactly (both are the correctly rounded
// value of the same real number, subnormals included); DIV = 2: IEEE division.
template <int DIV>
__device__ __forceinline__ float mean_of(float s, float n, float inv) {
  if (DIV == 0) return s;
  if (DIV == 1) return __fmul_rn(s, inv);
  return __fdiv_rn(s, n);
}

int div_mode(bool mean, int world) {
  if (!mean || world == 1) return 0;
  return (world & (world - 1)) == 0 ? 1 : 2;
}

template <int DIV>
__global__ void __launch_bounds__(256)
merge_kernel(const uint32_t* __restrict__ gathered, int world, uint64_t K, const uint32_t* __restrict__ start,
             int64_t n_tiles, uint64_t psi, float* __restrict__ dense) {
  __shared__ __align__(128) float acc[kMergeTile];
  const int64_t t = blockIdx.x;
  const uint64_t j0 = (uint64_t)t * kMergeTile;
  const int len = (int)min((uint64_t)kMergeTile, psi - j0);
  float4* acc4 = reinterpret_cast<float4*>(acc);
  for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  pdl_wait();
  __syncthreads();
  for (int r = 0; r < world; ++r) {
    const uint32_t* idx = gathered + (uint64_t)r * 2 * K;
    const uint32_t* val = idx + K;
    const uint32_t* st = start + (uint64_t)r * (n_tiles + 1) + t;
    const uint32_t a = st[0], b = st[1];
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const uint32_t j = idx[e] - (uint32_t)j0;
      acc[j] = __fadd_rn(acc[j], __uint_as_float(val[e]));
    }
    __syncthreads();
  }
  const float n = (float)world, inv = 1.0f / (float)world;
  if (DIV == 0 && len == kMergeTile) {
    // the finished tile leaves through one bulk copy (TMA engine, SASS UBLKCP): one thread issues
    // it after the CTA barrier of the last rank and waits only until the engine has read the
    // shared memory (0.990 -> 0.962 ms per GPT-2 XL merge against 128-bit stores by every thread)
    if (threadIdx.x == 0) {
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(acc);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(dense + j0), "r"(src), "n"(kMergeTile * 4) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    return;
  }
  if (len == kMergeTile) {
    float4* out = reinterpret_cast<float4*>(dense + j0);
    for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) {
      float4 v = acc4[q];
      v = make_float4(mean_of<DIV>(v.x, n, inv), mean_of<DIV>(v.y, n, inv), mean_of<DIV>(v.z, n, inv),
                      mean_of<DIV>(v.w, n, inv));
      out[q] = v;
    }
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) dense[j0 + i] = mean_of<DIV>(acc[i], n, inv);
  }
}


#ifndef LD_REPLAY_MINB
#define LD_REPLAY_MINB 6   // resident CTAs per SM the replay is compiled for (128 threads: 80 registers)
#endif

struct AdamK { float b1, c1, b2, c2, eps, nz; };   // nz = -0.0f (ieee_fast.cuh: opaque -0 addend)

// Fused n-step replay.  Each warp owns a contiguous kWarpSpan-element region of the CTA's tile and
// lane l the elements j0 + wb + 4*(l + 32*i) + q (i < kReplaySlots, q < 4): the per-step G_t of the
// region is built in the warp's own slice of shared memory, so a step needs only __syncwarp --
// no CTA barrier (barrier stalls were 17% of the 256-thread version's samples).  128 threads x 4
// slots: the per-step fixed work (zeroing, entry loops) is amortised over 16 elements per thread
// (measured 249 -> 214 ms for 100 GPT-2 XL steps against 256 x 2, 357 ms for 512 x 1).
// MAXW >= min(world, 8): ranks whose first-round entries are prefetched in registers.
// SGD keeps only p per element and its step is a couple of operations, so the per-step fixed work
// dominates: it runs 64 threads x 32 elements per tile instead (100 GPT-2 XL steps 69 -> 53 ms).
template <int OPT> struct ReplayShape {
  static constexpr int threads = OPT == LOWDIFF_SGD ? 64 : kReplayThreads;
  static constexpr int slots = kReplayTile / (4 * threads);        // float4 slots per lane
  static constexpr int span = kReplayTile / (threads / 32);         // elements per warp
  static constexpr int minb = OPT == LOWDIFF_SGD ? 14 : LD_REPLAY_MINB;
};

struct ReplayArgs {
  const uint32_t* diffs;
  int world;
  uint64_t K;
  int64_t n_steps;
  const uint32_t* start;
  int64_t n_tiles;
  const float* scal;
  AdamK ak;
  uint64_t lo, hi;
  int64_t tile0;
  float *p, *m, *v;
  uint32_t* fix_list;        // [n_tiles * warps] (tile << 8 | region) of regions to re-run exactly
  unsigned int* fix_count;
};

// cp.async of one 32-bit word global -> shared (LDGSTS): the prefetched entries of the next step land
// in shared memory without holding registers (a register prefetch was spilled by ptxas right after its
// load -- an STL waiting on the LDG, 11% of the kernel's stall samples)
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// The replay of one warp's region (region `wreg` of tile tl of the window), G_t built in the warp's
// shared-memory slice Gw.  SAFE = false: Adam's sqrt / division take the branch-free fast
// sequences (ieee_fast.cuh) with their operand windows folded into a WinAcc; if any operand of any
// step left the windows, nothing is written and the region is queued for an exact re-run
// (replay_fix_kernel).  SAFE = true: the intrinsics throughout (that re-run, or an eps outside the
// fast window).  Either way the written bits are the sequential R-11 recurrence.
// Sw: the warp's staging words in shared memory, u32[2 * MAXW * 32 + 4] (first-round idx | val |
// the step's lr, r1, r2)
template <int OPT, int DIV, int MAXW, bool SAFE>
__device__ __forceinline__ void replay_region(const ReplayArgs& A, int64_t tl, int wreg, float* Gw, uint32_t* Sw,
                                              int lane) {
  // elements [lo, hi) are replayed; p, m, v hold exactly that range (p[0] is element lo)
  constexpr int kReplaySlots = ReplayShape<OPT>::slots, kWarpSpan = ReplayShape<OPT>::span;
  static_assert(kWarpSpan == 128 * kReplaySlots, "one float4 per lane per slot");
  const uint32_t* __restrict__ diffs = A.diffs;
  const int world = A.world;
  const uint64_t K = A.K;
  const int64_t n_steps = A.n_steps;
  const uint32_t* __restrict__ start = A.start;
  const float* __restrict__ scal = A.scal;
  const AdamK ak = A.ak;
  const uint64_t lo = A.lo, hi = A.hi;
  float* __restrict__ p = A.p;
  float* __restrict__ m = A.m;
  float* __restrict__ v = A.v;
  const int64_t t = A.tile0 + tl;
  const uint64_t j0 = (uint64_t)t * kReplayTile;
  const uint32_t wb = (uint32_t)wreg * kWarpSpan;           // the warp's region: [j0 + wb, j0 + wb + span)
  const uint32_t jw = (uint32_t)j0 + wb;                    // Psi < 2^32
  float4* G4w = reinterpret_cast<float4*>(Gw);
  // state in element pairs (f32x2: FADD2/FMUL2/FFMA2 do both halves in one instruction, each
  // rounded exactly like the scalar operation): pair x = 2 i + h holds elements 2h, 2h+1 of slot i
  f32x2 P2[2 * kReplaySlots], M2[2 * kReplaySlots], V2[2 * kReplaySlots];
  bool neg_v = false;   // a negative initial v (not -0) is outside the fast windows
#pragma unroll
  for (int i = 0; i < kReplaySlots; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float pe[2], me[2], ve[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint64_t j = (uint64_t)jw + 4 * (lane + 32 * i) + 2 * h + e;
        const bool in = j >= lo && j < hi;
        pe[e] = in ? p[j - lo] : 0.f;
        me[e] = (OPT == LOWDIFF_ADAM && in) ? m[j - lo] : 0.f;
        ve[e] = (OPT == LOWDIFF_ADAM && in) ? v[j - lo] : 0.f;
        neg_v |= __float_as_uint(ve[e]) > 0x80000000u;
      }
      P2[2 * i + h] = pk2(pe[0], pe[1]);
      M2[2 * i + h] = pk2(me[0], me[1]);
      V2[2 * i + h] = pk2(ve[0], ve[1]);
    }
  }
  const AdamK2 k2 = make_adamk2(ak.b1, ak.c1, ak.b2, ak.c2, ak.eps, ak.nz);
  const float n = (float)world, inv = 1.0f / (float)world;
  const uint64_t tstride = (uint64_t)(A.n_tiles + 1);   // n_tiles = tiles in the window
  WinAcc win = win_init();
  // Software pipeline over steps: lane r (< 32) holds rank r's entry range of this tile for the
  // current step (ra_c, rb_c) and the next (ra_n, rb_n); the ranges of step s+2 and the first
  // round of step s+1's entries (entry a_r + lane of every rank < MAXW, by cp.async into the warp's
  // staging words Sw) are loaded while step s computes.
  const int wr = world < 32 ? world : 32;
  uint32_t ra_c = 0, rb_c = 0, ra_n = 0, rb_n = 0;
  if (lane < wr) {
    ra_c = __ldg(start + (uint64_t)lane * tstride + tl);
    rb_c = __ldg(start + (uint64_t)lane * tstride + tl + 1);
    if (n_steps > 1) {
      const uint32_t* st1 = start + ((uint64_t)world + lane) * tstride + tl;
      ra_n = __ldg(st1);
      rb_n = __ldg(st1 + 1);
    }
  }
  // per-step strides, advanced incrementally (no 64-bit products in the step loop)
  const uint64_t bstride = (uint64_t)world * 2 * K;          // u32 of the blocks of one step
  const uint64_t sstride = (uint64_t)world * tstride;        // u32 of the start table of one step
  const uint32_t* st2 = start + 2 * sstride + (uint64_t)lane * tstride + tl;   // step s + 2, rank `lane`
  const float* sc_n = scal + 3;                              // scalars of step s + 1 (then s + 2 ...)
  // kCpa (several ranks per step): the prefetched first round and the step's three scalars go to the
  // warp's staging words Sw by cp.async -- with 2 x MAXW prefetch registers ptxas spilled each
  // prefetched word right after its load (an STL waiting on the LDG: 11% of the stall samples) and
  // moved the scalars to uniform registers right after theirs.  Measured, 100 GPT-2 XL steps: 8 ranks
  // per step over 1/8 of Psi 95.9 -> 77.8 ms; 1 rank 189.5 -> 193.7 ms, so one rank keeps registers.
#ifndef LD_CPA_E_MIN
#define LD_CPA_E_MIN 2
#endif
#ifndef LD_CPA_S_MIN
#define LD_CPA_S_MIN 2
#endif
  constexpr bool kCpa = MAXW >= LD_CPA_E_MIN, kCpaS = MAXW >= LD_CPA_S_MIN;
  uint32_t* Ssc = Sw + 2 * MAXW * 32;
  uint32_t pj[MAXW], pv[MAXW];          // !kCpa: the first round in registers
  float lr = 0.f, r1 = 0.f, r2 = 0.f;   // !kCpa: the scalars of the prefetched step
  auto load_entries = [&](const uint32_t* blk, uint32_t ra, uint32_t rb, const float* sc) {   // first round of a step
    if (kCpaS) {
      if (lane < 3) cp_async4(Ssc + lane, reinterpret_cast<const uint32_t*>(sc) + lane);
    } else {
      lr = __ldg(sc);
      r1 = __ldg(sc + 1);
      r2 = __ldg(sc + 2);
    }
#pragma unroll
    for (int r = 0; r < MAXW; ++r) {
      if (!kCpa) {
        pj[r] = 0xFFFFFFFFu;
        pv[r] = 0u;
      }
      if (r < world) {
        const uint32_t e = __shfl_sync(0xFFFFFFFFu, ra, r) + lane;
        const uint32_t eb = __shfl_sync(0xFFFFFFFFu, rb, r);
        if (e < eb) {
          const uint32_t* idx = blk + (uint64_t)r * 2 * K;
          if (kCpa) {
            cp_async4(Sw + r * 32 + lane, idx + e);
            cp_async4(Sw + (MAXW + r) * 32 + lane, idx + K + e);
          } else {
            pj[r] = __ldg(idx + e) - jw;   // >= kWarpSpan (wrapped) when outside the warp's region
            pv[r] = __ldg(idx + K + e);
          }
        }
      }
    }
    if (kCpa || kCpaS) asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const uint32_t* blk = diffs;                               // step s
  load_entries(blk, ra_c, rb_c, scal);
#pragma unroll 1
  for (int64_t s = 0; s < n_steps; ++s) {
#pragma unroll
    for (int i = 0; i < kReplaySlots; ++i) G4w[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kCpa || kCpaS) asm volatile("cp.async.wait_all;" ::: "memory");   // this step's first round and scalars are in Sw
    __syncwarp();
    const float slr = kCpaS ? __uint_as_float(Ssc[0]) : lr, sr1 = kCpaS ? __uint_as_float(Ssc[1]) : r1,
                sr2 = kCpaS ? __uint_as_float(Ssc[2]) : r2;
    // rank by rank from +0: the rank-order sum of DESIGN.md R-8 (indices unique within a rank)
#pragma unroll
    for (int r = 0; r < MAXW; ++r) {
      if (r < world) {
        if (!kCpa && pj[r] < (uint32_t)kWarpSpan) Gw[pj[r]] = __fadd_rn(Gw[pj[r]], __uint_as_float(pv[r]));
        const uint32_t a = __shfl_sync(0xFFFFFFFFu, ra_c, r), b = __shfl_sync(0xFFFFFFFFu, rb_c, r);
        if (kCpa && a + lane < b) {
          const uint32_t jl = Sw[r * 32 + lane] - jw;   // >= kWarpSpan (wrapped) outside the region
          if (jl < (uint32_t)kWarpSpan) Gw[jl] = __fadd_rn(Gw[jl], __uint_as_float(Sw[(MAXW + r) * 32 + lane]));
        }
        const uint32_t* idx = blk + (uint64_t)r * 2 * K;
        for (uint32_t e = a + 32 + lane; e < b; e += 32) {
          const uint32_t jl = __ldg(idx + e) - jw;
          if (jl < (uint32_t)kWarpSpan) Gw[jl] = __fadd_rn(Gw[jl], __uint_as_float(__ldg(idx + K + e)));
        }
        __syncwarp();
      }
    }
    for (int r = MAXW; r < world; ++r) {   // ranks beyond the register window
      uint32_t a, b;
      if (r < 32) {
        a = __shfl_sync(0xFFFFFFFFu, ra_c, r);
        b = __shfl_sync(0xFFFFFFFFu, rb_c, r);
      } else {
        const uint32_t* st = start + ((uint64_t)s * world + r) * tstride + tl;
        a = __ldg(st);
        b = __ldg(st + 1);
      }
      const uint32_t* idx = blk + (uint64_t)r * 2 * K;
      for (uint32_t e = a + lane; e < b; e += 32) {
        const uint32_t jl = __ldg(idx + e) - jw;
        if (jl < (uint32_t)kWarpSpan) Gw[jl] = __fadd_rn(Gw[jl], __uint_as_float(__ldg(idx + K + e)));
      }
      __syncwarp();
    }
    // prefetch for the next steps while this one computes
    uint32_t na = 0, nb = 0;
    if (s + 1 < n_steps) {
      load_entries(blk + bstride, ra_n, rb_n, sc_n);
      sc_n += 3;
    }
    if (lane < wr && s + 2 < n_steps) {
      na = __ldg(st2);
      nb = __ldg(st2 + 1);
    }
    st2 += sstride;
    blk += bstride;
    const f32x2 LR = pk2(slr, slr), R1 = pk2(sr1, sr1), R2 = pk2(sr2, sr2), R2N = pk2(-sr2, -sr2);
#pragma unroll
    for (int i = 0; i < kReplaySlots; ++i) {   // float4 slots: 2 independent element pairs each
      const float4 gv = G4w[lane + 32 * i];
      const f32x2 g01 = pk2(mean_of<DIV>(gv.x, n, inv), mean_of<DIV>(gv.y, n, inv));
      const f32x2 g23 = pk2(mean_of<DIV>(gv.z, n, inv), mean_of<DIV>(gv.w, n, inv));
      if (OPT == LOWDIFF_ADAM) {
        // m = b1*m + c1*g ; v = b2*v + c2*(g*g) ; mh = m*r1 ; vh = v*r2
        // d = sqrt(vh) + eps ; u = mh / d ; p = p - lr*u          (R-11)
        f32x2 u0, u1;
        if (SAFE) {
          u0 = adam2_u_exact(M2[2 * i], V2[2 * i], g01, k2, R1, R2, ak.eps);
          u1 = adam2_u_exact(M2[2 * i + 1], V2[2 * i + 1], g23, k2, R1, R2, ak.eps);
        } else {
          u0 = adam2_u_agg(M2[2 * i], V2[2 * i], g01, k2, R1, R2N, win);
          u1 = adam2_u_agg(M2[2 * i + 1], V2[2 * i + 1], g23, k2, R1, R2N, win);
        }
        P2[2 * i] = sub_prod2(P2[2 * i], LR, u0, k2.nz);
        P2[2 * i + 1] = sub_prod2(P2[2 * i + 1], LR, u1, k2.nz);
      } else {
        P2[2 * i] = sub_prod2(P2[2 * i], LR, g01, k2.nz);
        P2[2 * i + 1] = sub_prod2(P2[2 * i + 1], LR, g23, k2.nz);
      }
    }
    ra_c = ra_n;
    rb_c = rb_n;
    ra_n = na;
    rb_n = nb;
    __syncwarp();   // every lane has read this step's G before the next step zeroes and adds
  }
  if (OPT == LOWDIFF_ADAM && !SAFE) {
    if (__any_sync(0xFFFFFFFFu, neg_v | win_bad(win))) {   // rare: re-run the region exactly
      if (lane == 0) A.fix_list[atomicAdd(A.fix_count, 1u)] = (uint32_t)(tl << 8) | (uint32_t)wreg;
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < kReplaySlots; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t j = (uint64_t)jw + 4 * (lane + 32 * i) + q;
      const int x = 2 * i + (q >> 1);
      if (j >= lo && j < hi) {
        p[j - lo] = (q & 1) ? hi2(P2[x]) : lo2(P2[x]);
        if (OPT == LOWDIFF_ADAM) {
          m[j - lo] = (q & 1) ? hi2(M2[x]) : lo2(M2[x]);
          v[j - lo] = (q & 1) ? hi2(V2[x]) : lo2(V2[x]);
        }
      }
    }
  }
}

// Measured (B200, 100 GPT-2 XL steps, tools/run_replay_ab.sh): Adam, 1 rank per step: 6 CTAs/SM
// (80 registers) 196 ms, 7 (72, spills) 199 ms, 5 (96) 207 ms, 8 (64) 216 ms, 256 threads x 8
// elements 227-245 ms; 8 ranks per step (MAXW 8): 7 CTAs/SM 96.5 ms, 6 99.5 ms, 5 108 ms.  Re-run
// on the final code (cp.async staging, chained window minima): 1 rank 6 / 7 / 5 CTAs/SM 185.4 /
// 190.2 / 198.1 ms; 8 ranks 7 / 8 / 6 CTAs/SM 78.6 / 79.8 / 79.0 ms (before the index-pass change;
// DESIGN.md 4.3).
template <int OPT, int DIV, int MAXW, bool SAFE>
__global__ void __launch_bounds__(ReplayShape<OPT>::threads,
                                  OPT == LOWDIFF_ADAM && MAXW >= 8 ? ReplayShape<OPT>::minb + 1 : ReplayShape<OPT>::minb)
replay_kernel(ReplayArgs A) {
  __shared__ __align__(16) float G[kReplayTile];
  __shared__ uint32_t S[ReplayShape<OPT>::threads / 32][2 * MAXW * 32 + 4];
  const int warp = threadIdx.x >> 5;
  replay_region<OPT, DIV, MAXW, SAFE>(A, blockIdx.x, warp, G + warp * ReplayShape<OPT>::span, S[warp],
                                      threadIdx.x & 31);
}

// the exact re-run of the regions replay_kernel queued (Adam only): one warp per queued region
template <int DIV, int MAXW>
__global__ void __launch_bounds__(ReplayShape<LOWDIFF_ADAM>::threads)
replay_fix_kernel(ReplayArgs A) {
  __shared__ __align__(16) float G[kReplayTile];
  constexpr int kWarps = ReplayShape<LOWDIFF_ADAM>::threads / 32;
  __shared__ uint32_t S[kWarps][2 * MAXW * 32 + 4];
  const int warp = threadIdx.x >> 5;
  const unsigned n = *A.fix_count;
  for (unsigned i = blockIdx.x * kWarps + warp; i < n; i += gridDim.x * kWarps) {
    const uint32_t item = A.fix_list[i];
    replay_region<LOWDIFF_ADAM, DIV, MAXW, true>(A, (int64_t)(item >> 8), (int)(item & 0xFFu),
                                                 G + warp * ReplayShape<LOWDIFF_ADAM>::span, S[warp], threadIdx.x & 31);
  }
}

// Live optimizer step from the gathered blocks (lowdiff_exchange_update): the merge's
// tile gather into shared memory, then one streaming pass over the tile's p, m, v with 128-bit
// loads/stores, the R-11 Adam / R-12 SGD on each element (same operations and order as the replay
// kernel, so the same bits), two float4 groups in flight per thread.  G never reaches HBM:
// 24 B/param (Adam) + 8 N B/entry instead of merge 4 B/param + dense step 28 B/param.
template <int OPT, int DIV>
__global__ void __launch_bounds__(256)
update_kernel(const uint32_t* __restrict__ gathered, int world, uint64_t K, const uint32_t* __restrict__ start,
              int64_t n_tiles, uint64_t psi, AdamK ak, float lr, float r1, float r2, float* __restrict__ p,
              float* __restrict__ m, float* __restrict__ v) {
  __shared__ float acc[kMergeTile];
  const int64_t t = blockIdx.x;
  const uint64_t j0 = (uint64_t)t * kMergeTile;
  const int len = (int)min((uint64_t)kMergeTile, psi - j0);
  float4* acc4 = reinterpret_cast<float4*>(acc);
  for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  for (int r = 0; r < world; ++r) {
    const uint32_t* idx = gathered + (uint64_t)r * 2 * K;
    const uint32_t* val = idx + K;
    const uint32_t* st = start + (uint64_t)r * (n_tiles + 1) + t;
    const uint32_t a = st[0], b = st[1];
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const uint32_t j = idx[e] - (uint32_t)j0;
      acc[j] = __fadd_rn(acc[j], __uint_as_float(val[e]));
    }
    __syncthreads();
  }
  const float n = (float)world, inv = 1.0f / (float)world;
  const bool eps_ok = ak.eps >= 0x1p-60f && ak.eps <= 0x1p59f;
  auto step1 = [&](float g, float& P, float& M, float& V) {
    opt_step1<OPT == LOWDIFF_ADAM>(g, P, M, V, ak.b1, ak.c1, ak.b2, ak.c2, ak.eps, eps_ok, lr, r1, r2);
  };
  if (len == kMergeTile) {
    float4* p4 = reinterpret_cast<float4*>(p + j0);
    float4* m4 = reinterpret_cast<float4*>(m + j0);
    float4* v4 = reinterpret_cast<float4*>(v + j0);
#pragma unroll 2
    for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) {
      float4 P = __ldcs(p4 + q), M, V;
      if (OPT == LOWDIFF_ADAM) { M = __ldcs(m4 + q); V = __ldcs(v4 + q); }
      const float4 gv = acc4[q];
      const float g[4] = {mean_of<DIV>(gv.x, n, inv), mean_of<DIV>(gv.y, n, inv), mean_of<DIV>(gv.z, n, inv),
                          mean_of<DIV>(gv.w, n, inv)};
      step1(g[0], P.x, M.x, V.x);
      step1(g[1], P.y, M.y, V.y);
      step1(g[2], P.z, M.z, V.z);
      step1(g[3], P.w, M.w, V.w);
      __stcs(p4 + q, P);
      if (OPT == LOWDIFF_ADAM) { __stcs(m4 + q, M); __stcs(v4 + q, V); }
    }
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      float P = p[j0 + i], M = 0.f, V = 0.f;
      if (OPT == LOWDIFF_ADAM) { M = m[j0 + i]; V = v[j0 + i]; }
      step1(mean_of<DIV>(acc[i], n, inv), P, M, V);
      p[j0 + i] = P;
      if (OPT == LOWDIFF_ADAM) { m[j0 + i] = M; v[j0 + i] = V; }
    }
  }
}

int num_sms2() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

size_t merge_scratch_bytes(int64_t psi, int world, int64_t n_blocks) {
  (void)world;
  const int64_t n_tiles = (psi + kMergeTile - 1) / kMergeTile;
  return (size_t)n_blocks * (n_tiles + 1) * sizeof(uint32_t);
}

size_t replay_scratch_bytes(int64_t psi, int world, int64_t n_steps) {
  const int64_t n_tiles = (psi + kReplayTile - 1) / kReplayTile;
  return (size_t)n_steps * world * (n_tiles + 1) * sizeof(uint32_t) + (size_t)n_steps * 3 * sizeof(float) + 256 +
         (size_t)n_tiles * 4 * sizeof(uint32_t);   // + the exact-re-run queue
}

cudaError_t launch_tile_start(const uint32_t* block, uint64_t K, int64_t psi, uint32_t* start, cudaStream_t s) {
  const int64_t n_tiles = (psi + kMergeTile - 1) / kMergeTile;
  const unsigned gx = (unsigned)std::min<uint64_t>((K + 256) / 256, (uint64_t)num_sms2() * 16);
  tile_start_kernel<<<dim3(gx, 1), 256, 0, s>>>(block, 1, 2 * K, (uint32_t)K, kMergeTileShift, 0u, (uint32_t)n_tiles,
                                                 nullptr, start);
  return cudaGetLastError();
}

namespace {
// warp-cooperative lower_bound over an ascending u32 array: 32 probes per round
__device__ uint32_t warp_lower_bound(const uint32_t* __restrict__ a, uint32_t n, uint32_t key) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = n;   // the answer lies in [lo, hi]
  while (hi - lo > 32) {
    const uint32_t span = hi - lo;
    const uint32_t p = lo + (uint32_t)(((uint64_t)span * (uint32_t)(lane + 1)) / 33u);
    const bool below = __ldg(a + p) < key;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, below);
    const int c = __popc(m);   // probes below the key (a prefix of the lanes: a is ascending)
    const uint32_t nlo = c ? __shfl_sync(0xFFFFFFFFu, p, c - 1) + 1 : lo;
    const uint32_t nhi = c < 32 ? __shfl_sync(0xFFFFFFFFu, p, c < 32 ? c : 31) : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint32_t p = lo + (uint32_t)lane;
  const bool below = p < hi && __ldg(a + p) < key;
  return lo + (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, below));
}

// ranges[2b], ranges[2b+1] = the entries of block b inside tiles [T0, T1) (warp per block)
__global__ void window_range_kernel(const uint32_t* __restrict__ blocks, int n_blocks, uint64_t stride, uint32_t K,
                                    int shift, uint32_t T0, uint32_t T1, uint32_t* __restrict__ ranges) {
  const int b = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (b >= n_blocks) return;
  const uint32_t* idx = blocks + (uint64_t)b * stride;
  const uint64_t jlo = (uint64_t)T0 << shift, jhi = (uint64_t)T1 << shift;
  const uint32_t ea = warp_lower_bound(idx, K, jlo > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)jlo);
  const uint32_t eb = jhi > 0xFFFFFFFFull ? K : warp_lower_bound(idx, K, (uint32_t)jhi);
  if ((threadIdx.x & 31) == 0) {
    ranges[2 * b] = ea;
    ranges[2 * b + 1] = eb;
  }
}
}  // namespace

// the start table of tiles T0..T1 reading only the entries that fall in them (a window-range search
// first: a shard's table no longer streams every rank's whole index list)
cudaError_t launch_tile_window(const uint32_t* blocks, int n_blocks, uint64_t K, int shift, uint32_t T0, uint32_t T1,
                               uint32_t* start, uint32_t* ranges, cudaStream_t s) {
  window_range_kernel<<<(n_blocks * 32 + 127) / 128, 128, 0, s>>>(blocks, n_blocks, 2 * K, (uint32_t)K, shift, T0, T1,
                                                                   ranges);
  // entries in the window: ~ K (T1 - T0) / (all tiles) per block; size the grid for the window
  const uint64_t per = std::max<uint64_t>(1, K);
  const unsigned gx = (unsigned)std::min<uint64_t>((per + 256) / 256, (uint64_t)num_sms2() * 16);
  tile_start_kernel<<<dim3(gx, (unsigned)n_blocks), 256, 0, s>>>(blocks, n_blocks, 2 * K, (uint32_t)K, shift, T0, T1,
                                                                  ranges, start);
  return cudaGetLastError();
}

cudaError_t launch_merge(lowdiff_ctx* c, int world, const uint32_t* gathered, float* dense, cudaStream_t s) {
  const int64_t psi = c->psi;
  const uint64_t K = (uint64_t)c->K;
  const int64_t n_tiles = (psi + kMergeTile - 1) / kMergeTile;
  const size_t need = merge_scratch_bytes(psi, world, world);
  if (c->merge_scratch_bytes < need) {
    if (c->merge_scratch) cudaFree(c->merge_scratch);
    c->merge_scratch = nullptr;
    c->scratch_gen += 1;   // captured graphs that baked in the old buffer are rebuilt
    c->merge_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&c->merge_scratch, need);
    if (e != cudaSuccess) return e;
    c->merge_scratch_bytes = need;
  }
  uint32_t* start = static_cast<uint32_t*>(c->merge_scratch);
  const int sms = num_sms2();
  int h;
  prof_begin(c, "merge", s, &h);
  {
    const unsigned gx = (unsigned)std::min<uint64_t>((K + 256) / 256, (uint64_t)sms * 16);
    tile_start_kernel<<<dim3(gx, (unsigned)world), 256, 0, s>>>(gathered, world, 2 * K, (uint32_t)K,
                                                                 kMergeTileShift, 0u, (uint32_t)n_tiles, nullptr,
                                                                 start);
  }
  const unsigned grid = (unsigned)n_tiles;
  // world 1 takes the same shared-memory tile (DIV 0: x / 1 == x): every element written once with
  // 128-bit stores -- measured 1.030 -> 0.990 ms per GPT-2 XL merge against round 1's global
  // zero-fill + scatter over the L2-resident tile (merge1)
  const int dm = div_mode(c->cfg.mean != 0, world);
  cudaError_t e = launch_pdl(!c->prof, dm == 0 ? merge_kernel<0> : dm == 1 ? merge_kernel<1> : merge_kernel<2>, grid, 256, 0,
                             s, gathered, world, K, start, n_tiles, (uint64_t)psi, dense);
  if (e != cudaSuccess) return e;
  prof_end(c, h, s);
  c->launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_update(lowdiff_ctx* c, int world, const uint32_t* gathered, const lowdiff_step_scalars& sc,
                          float* p, float* m, float* v, cudaStream_t s) {
  const int64_t psi = c->psi;
  const uint64_t K = (uint64_t)c->K;
  const int64_t n_tiles = (psi + kMergeTile - 1) / kMergeTile;
  const size_t need = merge_scratch_bytes(psi, world, world);
  if (c->merge_scratch_bytes < need) {
    if (c->merge_scratch) cudaFree(c->merge_scratch);
    c->merge_scratch = nullptr;
    c->scratch_gen += 1;   // captured graphs that baked in the old buffer are rebuilt
    c->merge_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&c->merge_scratch, need);
    if (e != cudaSuccess) return e;
    c->merge_scratch_bytes = need;
  }
  uint32_t* start = static_cast<uint32_t*>(c->merge_scratch);
  int h;
  prof_begin(c, "update", s, &h);
  {
    const unsigned gx = (unsigned)std::min<uint64_t>((K + 256) / 256, (uint64_t)num_sms2() * 16);
    tile_start_kernel<<<dim3(gx, (unsigned)world), 256, 0, s>>>(gathered, world, 2 * K, (uint32_t)K,
                                                                 kMergeTileShift, 0u, (uint32_t)n_tiles, nullptr,
                                                                 start);
  }
  const AdamK ak{c->cfg.adam.beta1, c->cfg.adam.one_minus_beta1, c->cfg.adam.beta2, c->cfg.adam.one_minus_beta2,
                 c->cfg.adam.eps, -0.0f};
  const unsigned grid = (unsigned)n_tiles;
  const int dm = div_mode(c->cfg.mean != 0, world);
#define LD_UPD(OPT, DIV) \
  update_kernel<OPT, DIV><<<grid, 256, 0, s>>>(gathered, world, K, start, n_tiles, (uint64_t)psi, ak, sc.lr, \
                                               sc.bc1_inv, sc.bc2_inv, p, m, v)
  if (c->cfg.optim == LOWDIFF_ADAM) {
    if (dm == 0) LD_UPD(LOWDIFF_ADAM, 0); else if (dm == 1) LD_UPD(LOWDIFF_ADAM, 1); else LD_UPD(LOWDIFF_ADAM, 2);
  } else {
    if (dm == 0) LD_UPD(LOWDIFF_SGD, 0); else if (dm == 1) LD_UPD(LOWDIFF_SGD, 1); else LD_UPD(LOWDIFF_SGD, 2);
  }
#undef LD_UPD
  prof_end(c, h, s);
  c->launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_replay(lowdiff_ctx* c, int optim, bool mean, const float* consts5, int world, int64_t n_steps,
                          const uint32_t* diffs, const float* scal_dev, uint64_t lo, uint64_t hi,
                          const uint32_t* ranges, float* p, float* m, float* v, cudaStream_t s, uint64_t k_stride) {
  if (lo >= hi) return cudaSuccess;
  const uint64_t K = k_stride ? k_stride : (uint64_t)c->K;
  // the window of tiles that hold [lo, hi): tile0 .. tile0 + n_tiles - 1 (start table: n_tiles + 1)
  const int64_t tile0 = (int64_t)(lo >> kReplayTileShift);
  const int64_t n_tiles = (int64_t)((hi - 1) >> kReplayTileShift) - tile0 + 1;
  // scratch: the start table, then the exact-re-run queue (a count and one word per warp region)
  const size_t sbytes = ((size_t)n_steps * world * (n_tiles + 1) * sizeof(uint32_t) + 15) & ~(size_t)15;
  const size_t fix_words = (size_t)n_tiles * (kReplayTile / (128 * ReplayShape<LOWDIFF_ADAM>::slots));
  const size_t tbytes = sbytes + 16 + fix_words * sizeof(uint32_t);
  if (c->replay_scratch_bytes < tbytes) {
    if (c->replay_scratch) cudaFree(c->replay_scratch);
    c->replay_scratch = nullptr;
    c->replay_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&c->replay_scratch, tbytes);
    if (e != cudaSuccess) return e;
    c->replay_scratch_bytes = tbytes;
  }
  uint32_t* start = static_cast<uint32_t*>(c->replay_scratch);
  unsigned int* fix_count = reinterpret_cast<unsigned int*>(static_cast<char*>(c->replay_scratch) + sbytes);
  uint32_t* fix_list = reinterpret_cast<uint32_t*>(static_cast<char*>(c->replay_scratch) + sbytes + 16);
  const int sms = num_sms2();
  AdamK ak{consts5[0], consts5[1], consts5[2], consts5[3], consts5[4], -0.0f};
  int h;
  prof_begin(c, "replay_index", s, &h);
  {
    const int64_t nb = n_steps * world;
    const unsigned gy = (unsigned)std::min<int64_t>(nb, 65535);
    // ~96 CTAs per SM in total over the blocks: several waves, so the last one's tail is short
    // (measured, C4 shape: 16 per SM 60.5 ms, 48 58.4, 96 58.2, 160 58.0; one wave, 8: 63.7)
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((K + 256) / 256, (int64_t)sms * 96 / gy + 1));
    tile_start_kernel<<<dim3(gx, gy), 256, 0, s>>>(diffs, nb, 2 * K, (uint32_t)K, kReplayTileShift, (uint32_t)tile0,
                                                   (uint32_t)(tile0 + n_tiles), ranges, start);
  }
  prof_end(c, h, s);
  prof_begin(c, "replay", s, &h);
  const unsigned grid = (unsigned)n_tiles;
  const int dm = div_mode(mean, world);
  const bool eps_ok = ak.eps >= 0x1p-60f && ak.eps <= 0x1p59f;   // adam_u_fast's precondition
  const ReplayArgs A{diffs, world, K, n_steps, start, n_tiles, scal_dev, ak, lo, hi, tile0, p, m, v, fix_list,
                     fix_count};
  const bool fix = optim == LOWDIFF_ADAM && eps_ok;   // the fast path may queue regions for a re-run
  if (fix) {
    cudaError_t e = cudaMemsetAsync(fix_count, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
  }
#define LD_REPLAY(OPT, DIV, W)                                                                         \
  do {                                                                                               \
    if (OPT == LOWDIFF_SGD || eps_ok)                                                                \
      replay_kernel<OPT, DIV, W, false><<<grid, ReplayShape<OPT>::threads, 0, s>>>(A);               \
    else                                                                                             \
      replay_kernel<OPT, DIV, W, true><<<grid, ReplayShape<OPT>::threads, 0, s>>>(A);                \
    if (OPT == LOWDIFF_ADAM && eps_ok)                                                               \
      replay_fix_kernel<DIV, W><<<sms * 4, ReplayShape<LOWDIFF_ADAM>::threads, 0, s>>>(A);           \
  } while (0)
#define LD_REPLAY_W(OPT, DIV)                                  \
  do {                                                         \
    if (world == 1) LD_REPLAY(OPT, DIV, 1);                    \
    else if (world == 2) LD_REPLAY(OPT, DIV, 2);               \
    else if (world <= 4) LD_REPLAY(OPT, DIV, 4);               \
    else LD_REPLAY(OPT, DIV, 8);                               \
  } while (0)
  if (optim == LOWDIFF_ADAM) {
    if (dm == 0) LD_REPLAY_W(LOWDIFF_ADAM, 0); else if (dm == 1) LD_REPLAY_W(LOWDIFF_ADAM, 1); else LD_REPLAY_W(LOWDIFF_ADAM, 2);
  } else {
    if (dm == 0) LD_REPLAY_W(LOWDIFF_SGD, 0); else if (dm == 1) LD_REPLAY_W(LOWDIFF_SGD, 1); else LD_REPLAY_W(LOWDIFF_SGD, 2);
  }
#undef LD_REPLAY_W
#undef LD_REPLAY
  prof_end(c, h, s);
  c->launches += fix ? 3 : 2;
  return cudaGetLastError();
}

}  // namespace ld
