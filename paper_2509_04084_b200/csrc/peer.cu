// Peer-memory exchange: the allgather of Alg. 1 line 5 fused into
// the merge of line 7.  Every rank's send blocks live in library-owned device
// buffers that the other ranks map (CUDA IPC over NVLink/NVSwitch, or plain pointers when the
// "ranks" share a device); each rank's merge kernel reads the peers' (idx, val) entries of its
// output tile straight from their HBM, rank by rank, so the gathered buffer is never written to or
// re-read from local HBM and the NVLink transfer overlaps the merge tile by tile.  The arithmetic
// is merge_kernel's (rank-order sum from +0, then / N: DESIGN.md R-8) -> bitwise equal to the
// NCCL path.
//
// Ordering between ranks uses per-rank flag words (u64, system scope):
//   ready[slot]         = epoch of the block now in `slot` (written by its owner after compress and
//                         its tile-start table; st.release.sys after __threadfence_system)
//   done[slot][q]       = last epoch of `slot` that rank q finished reading (written remotely by q)
// A consumer waits for ready >= epoch before reading (ld.acquire.sys); a producer waits for every
// done >= previous epoch before compressing into the slot again (write-after-read).  Every wait
// is bounded (kPeerTimeoutNs): on expiry it counts an error in the waiter's own flag word and
// continues, so a protocol misuse surfaces as LOWDIFF_E_STATE at lowdiff_sync instead of a hang.
#include <cuda_runtime.h>

#include "ieee_fast.cuh"
#include "internal.h"

namespace ld {
namespace {

constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// spin until *p >= want; false on timeout (then counts an error in *err)
__device__ bool wait_geq(const unsigned long long* p, unsigned long long want, unsigned long long* err) {
  if (ld_acquire(p) >= want) return true;
  const unsigned long long t0 = now_ns();
  while (ld_acquire(p) < want) {
    if (now_ns() - t0 > kPeerTimeoutNs) {
      atomicAdd(err, 1ull);
      return false;
    }
    __nanosleep(256);
  }
  return true;
}

__global__ void peer_ready_kernel(unsigned long long* own_flags, int slot, unsigned long long epoch) {
  __threadfence_system();   // the block and its tile-start table (earlier kernels) before the flag
  st_release(own_flags + slot, epoch);
}

// producer side WAR: every rank has finished reading the previous content of `slot`
__global__ void peer_wait_done_kernel(unsigned long long* own_flags, int n_slots, int slot, int world,
                                      unsigned long long epoch) {
  const int q = threadIdx.x;
  if (q < world) wait_geq(own_flags + n_slots + slot * kPeerMaxWorld + q, epoch, own_flags + peer_err_word(n_slots));
}

template <int DIV>
__device__ __forceinline__ float mean_of(float s, float n, float inv) {
  if (DIV == 0) return s;
  if (DIV == 1) return __fmul_rn(s, inv);
  return __fdiv_rn(s, n);
}

template <int DIV>
__global__ void __launch_bounds__(256)
peer_merge_kernel(PeerTable T, uint64_t K, int64_t n_tiles, uint64_t psi, float* __restrict__ dense) {
  __shared__ float acc[kMergeTile];
  const int64_t t = blockIdx.x;
  const uint64_t j0 = (uint64_t)t * kMergeTile;
  const int len = (int)min((uint64_t)kMergeTile, psi - j0);
  if (threadIdx.x < T.world)
    wait_geq(T.flags[threadIdx.x] + T.slot, T.epoch, T.flags[T.self] + peer_err_word(T.n_slots));
  float4* acc4 = reinterpret_cast<float4*>(acc);
  for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  for (int r = 0; r < T.world; ++r) {
    const uint32_t* idx = T.send[r];
    const uint32_t* val = idx + K;
    const uint32_t a = T.start[r][t], b = T.start[r][t + 1];
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const uint32_t j = idx[e] - (uint32_t)j0;
      acc[j] = __fadd_rn(acc[j], __uint_as_float(val[e]));
    }
    __syncthreads();
  }
  const float n = (float)T.world, inv = 1.0f / (float)T.world;
  if (len == kMergeTile) {
    float4* out = reinterpret_cast<float4*>(dense + j0);
    for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) {
      float4 v = acc4[q];
      out[q] = make_float4(mean_of<DIV>(v.x, n, inv), mean_of<DIV>(v.y, n, inv), mean_of<DIV>(v.z, n, inv),
                           mean_of<DIV>(v.w, n, inv));
    }
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) dense[j0 + i] = mean_of<DIV>(acc[i], n, inv);
  }
}

// The live optimizer step straight from the peers' blocks (lowdiff_exchange_peer_update, SURVEY
// NEXT-1 second half): the tile's G is merged in shared memory from every rank's entries read over
// NVLink (as peer_merge_kernel), then one streaming pass applies the R-11 Adam / R-12 SGD to the
// tile's p, m, v (opt_step1: the replay's and update_kernel's operations) -- neither a gathered
// buffer nor the dense G ever exists in HBM.  Local HBM: 24 B/param (Adam; 8 SGD); remote reads:
// 8 B per peer entry falling in the tile.
template <bool ADAM, int DIV>
__global__ void __launch_bounds__(256)
peer_update_kernel(PeerTable T, uint64_t K, int64_t n_tiles, uint64_t psi, PeerOpt o, float* __restrict__ p,
                   float* __restrict__ m, float* __restrict__ v) {
  __shared__ float acc[kMergeTile];
  const int64_t t = blockIdx.x;
  const uint64_t j0 = (uint64_t)t * kMergeTile;
  const int len = (int)min((uint64_t)kMergeTile, psi - j0);
  if (threadIdx.x < T.world)
    wait_geq(T.flags[threadIdx.x] + T.slot, T.epoch, T.flags[T.self] + peer_err_word(T.n_slots));
  float4* acc4 = reinterpret_cast<float4*>(acc);
  for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  for (int r = 0; r < T.world; ++r) {   // rank order from +0 (R-8): no conflicts within a rank
    const uint32_t* idx = T.send[r];
    const uint32_t* val = idx + K;
    const uint32_t a = T.start[r][t], b = T.start[r][t + 1];
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const uint32_t j = idx[e] - (uint32_t)j0;
      acc[j] = __fadd_rn(acc[j], __uint_as_float(val[e]));
    }
    __syncthreads();
  }
  const float n = (float)T.world, inv = 1.0f / (float)T.world;
  const bool eps_ok = o.eps >= 0x1p-60f && o.eps <= 0x1p59f;
  auto step1 = [&](float g, float& P, float& M, float& V) {
    opt_step1<ADAM>(mean_of<DIV>(g, n, inv), P, M, V, o.b1, o.c1, o.b2, o.c2, o.eps, eps_ok, o.lr, o.r1, o.r2);
  };
  if (len == kMergeTile) {
    float4* p4 = reinterpret_cast<float4*>(p + j0);
    float4* m4 = reinterpret_cast<float4*>(m + j0);
    float4* v4 = reinterpret_cast<float4*>(v + j0);
#pragma unroll 2
    for (int q = threadIdx.x; q < kMergeTile / 4; q += blockDim.x) {
      float4 P = __ldcs(p4 + q), M = make_float4(0.f, 0.f, 0.f, 0.f), V = M;
      if (ADAM) { M = __ldcs(m4 + q); V = __ldcs(v4 + q); }
      const float4 gv = acc4[q];
      step1(gv.x, P.x, M.x, V.x);
      step1(gv.y, P.y, M.y, V.y);
      step1(gv.z, P.z, M.z, V.z);
      step1(gv.w, P.w, M.w, V.w);
      __stcs(p4 + q, P);
      if (ADAM) { __stcs(m4 + q, M); __stcs(v4 + q, V); }
    }
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      float P = p[j0 + i], M = 0.f, V = 0.f;
      if (ADAM) { M = m[j0 + i]; V = v[j0 + i]; }
      step1(acc[i], P, M, V);
      p[j0 + i] = P;
      if (ADAM) { m[j0 + i] = M; v[j0 + i] = V; }
    }
  }
}

// consumer side: tell every owner that this rank finished reading `slot` at `epoch`
__global__ void peer_done_kernel(PeerTable T) {
  const int q = threadIdx.x;
  if (q < T.world) st_release(T.flags[q] + T.n_slots + T.slot * kPeerMaxWorld + T.self, T.epoch);
}

}  // namespace

cudaError_t launch_peer_update(const PeerTable& T, uint64_t K, int64_t psi, bool mean, bool adam, const PeerOpt& o,
                               float* p, float* m, float* v, cudaStream_t s) {
  const int64_t n_tiles = (psi + kMergeTile - 1) / kMergeTile;
  const unsigned grid = (unsigned)n_tiles;
  const int dm = (!mean || T.world == 1) ? 0 : ((T.world & (T.world - 1)) == 0 ? 1 : 2);
#define LD_PU(A, D) peer_update_kernel<A, D><<<grid, 256, 0, s>>>(T, K, n_tiles, (uint64_t)psi, o, p, m, v)
  if (adam) {
    if (dm == 0) LD_PU(true, 0); else if (dm == 1) LD_PU(true, 1); else LD_PU(true, 2);
  } else {
    if (dm == 0) LD_PU(false, 0); else if (dm == 1) LD_PU(false, 1); else LD_PU(false, 2);
  }
#undef LD_PU
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  peer_done_kernel<<<1, 32, 0, s>>>(T);
  return cudaGetLastError();
}

cudaError_t launch_peer_ready(unsigned long long* own_flags, int slot, unsigned long long epoch, cudaStream_t s) {
  peer_ready_kernel<<<1, 1, 0, s>>>(own_flags, slot, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait_done(unsigned long long* own_flags, int n_slots, int slot, int world,
                                  unsigned long long epoch, cudaStream_t s) {
  peer_wait_done_kernel<<<1, 32, 0, s>>>(own_flags, n_slots, slot, world, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_merge(const PeerTable& T, uint64_t K, int64_t psi, bool mean, float* dense, cudaStream_t s) {
  const int64_t n_tiles = (psi + kMergeTile - 1) / kMergeTile;
  const unsigned grid = (unsigned)n_tiles;
  const int dm = (!mean || T.world == 1) ? 0 : ((T.world & (T.world - 1)) == 0 ? 1 : 2);
  switch (dm) {
    case 0: peer_merge_kernel<0><<<grid, 256, 0, s>>>(T, K, n_tiles, (uint64_t)psi, dense); break;
    case 1: peer_merge_kernel<1><<<grid, 256, 0, s>>>(T, K, n_tiles, (uint64_t)psi, dense); break;
    default: peer_merge_kernel<2><<<grid, 256, 0, s>>>(T, K, n_tiles, (uint64_t)psi, dense); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  peer_done_kernel<<<1, 32, 0, s>>>(T);
  return cudaGetLastError();
}

}  // namespace ld
