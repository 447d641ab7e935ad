// LowDiff+ CPU replica, host optimizer (NEXT-3): PAPER.md §5.2 "CPU-based asynchronous persistence"
// and Alg. 2 lines 11-13: the snapshotted synced gradient
// G_t is applied to a CPU-resident copy of the model state, M^C_{t+1} = M^C_t + Adam(o_t, G_t);
// that copy is the in-memory checkpoint, persisted asynchronously, and the GPU state is restored
// from it after a software failure.  The worker thread and the ABI entry points
// that drive it are in api.cpp; this file is the arithmetic.
//
// Op order = DESIGN.md R-11, single-precision IEEE operations only: compiled by g++ with
// -ffp-contract=off and without fast-math (Makefile), so the replica equals the device replay
// bit for bit (tests/test_replica.py).  sqrt/div vectorise to sqrtps/divps, which are correctly
// rounded; -fno-math-errno only lets the compiler drop the errno branch of sqrt.  The loop is
// element-wise, so any split over threads gives the same bits.
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "../../include/lowdiff.h"

namespace {

__attribute__((target_clones("avx512f", "avx2", "default")))
void adam_range(const float* __restrict G, float b1, float c1, float b2, float c2, float eps, float lr, float r1,
                float r2, float* __restrict p, float* __restrict m, float* __restrict v, size_t lo, size_t hi) {
  for (size_t j = lo; j < hi; ++j) {
    const float g = G[j];
    const float mj = b1 * m[j] + c1 * g;
    const float vj = b2 * v[j] + c2 * (g * g);
    const float mh = mj * r1;
    const float vh = vj * r2;
    const float d = std::sqrt(vh) + eps;
    const float u = mh / d;
    p[j] = p[j] - lr * u;
    m[j] = mj;
    v[j] = vj;
  }
}

__attribute__((target_clones("avx512f", "avx2", "default")))
void sgd_range(const float* __restrict G, float lr, float* __restrict p, size_t lo, size_t hi) {
  for (size_t j = lo; j < hi; ++j) p[j] = p[j] - lr * G[j];
}

template <class F>
void parallel(size_t n, int threads, F f) {
  // contiguous ranges aligned to 16 elements (64 B) so threads never share a cache line
  threads = std::max(1, std::min(threads, (int)((n + 65535) >> 16)));
  if (threads == 1) { f(0, n); return; }
  const size_t per = ((n + threads - 1) / threads + 15) & ~(size_t)15;
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) {
    const size_t lo = std::min(n, per * t), hi = std::min(n, lo + per);
    if (lo < hi) pool.emplace_back(f, lo, hi);
  }
  f(0, std::min(n, per));
  for (auto& th : pool) th.join();
}

}  // namespace

namespace ld {

void host_adam(int64_t n, const float* G, const lowdiff_adam_consts& a, const lowdiff_step_scalars& s, float* p,
               float* m, float* v, int threads) {
  parallel((size_t)n, threads, [&](size_t lo, size_t hi) {
    adam_range(G, a.beta1, a.one_minus_beta1, a.beta2, a.one_minus_beta2, a.eps, s.lr, s.bc1_inv, s.bc2_inv, p, m, v,
               lo, hi);
  });
}

void host_sgd(int64_t n, const float* G, float lr, float* p, int threads) {
  parallel((size_t)n, threads, [&](size_t lo, size_t hi) { sgd_range(G, lr, p, lo, hi); });
}

}  // namespace ld

extern "C" {

lowdiff_status lowdiff_host_adam_step(int64_t n, const float* G, const lowdiff_adam_consts* consts,
                                      const lowdiff_step_scalars* scalars, float* p, float* m, float* v,
                                      int32_t threads) {
  if (n < 0 || (n > 0 && (!G || !consts || !scalars || !p || !m || !v))) return LOWDIFF_E_INVALID;
  if (n > 0) ld::host_adam(n, G, *consts, *scalars, p, m, v, threads);
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_host_sgd_step(int64_t n, const float* G, float lr, float* p, int32_t threads) {
  if (n < 0 || (n > 0 && (!G || !p))) return LOWDIFF_E_INVALID;
  if (n > 0) ld::host_sgd(n, G, lr, p, threads);
  return LOWDIFF_OK;
}

}  // extern "C"
