// C-ABI implementation of liblowdiff (part 4): LowDiff+ -- layer-wise dense snapshots and the CPU
// replica (Sec. 5; Alg. 2).
#include <dirent.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <thread>

#include "api_util.h"

using namespace ld::api;

namespace ld {
namespace api {

void replica_drain(lowdiff_ctx* c) {
  if (!c->rep_active) return;
  {
    std::unique_lock<std::mutex> lk(c->rep_mu);
    c->rep_done_cv.wait(lk, [&] { return c->rep_q.empty() && !c->rep_busy; });
  }
  // the writer is only joined by the worker or here; the worker is idle now
  if (c->rep_writer.joinable()) c->rep_writer.join();
}

void replica_shutdown(lowdiff_ctx* c) {
  if (c->rep_thread.joinable()) {
    {
      std::lock_guard<std::mutex> g(c->rep_mu);
      c->rep_stop = true;
    }
    c->rep_cv.notify_all();
    c->rep_thread.join();
  }
  if (c->rep_writer.joinable()) c->rep_writer.join();
  c->rep_stop = false;
  c->rep_active = false;
}

}  // namespace api
}  // namespace ld

extern "C" {

lowdiff_status lowdiff_snapshot_layer(lowdiff_ctx* c, int64_t iteration, int32_t first_layer, int32_t n_layers,
                                      const float* grad_bucket, void* producer) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!grad_bucket || first_layer < 0 || n_layers < 1 || first_layer + n_layers > c->cfg.n_layers || iteration < 0)
    return fail(c, LOWDIFF_E_INVALID, "snapshot_layer: bad argument");
  const int buf = (int)(iteration & 1);
  if (!c->snap_host[buf]) {
    CK(cudaHostAlloc((void**)&c->snap_host[buf], (size_t)c->psi * 4, cudaHostAllocDefault));
  }
  if (c->snap_iter[buf] != iteration) {
    const int64_t old = c->snap_iter[buf];
    if (c->rep_active && old >= 0 && old <= c->rep_tail) {
      // the replica worker still has to read iteration `old` from this buffer
      const int64_t t0 = now_ns();
      std::unique_lock<std::mutex> lk(c->rep_mu);
      c->rep_done_cv.wait(lk, [&] { return c->rep_iter.load() >= old; });
      c->rep_stall_ns += now_ns() - t0;
    }
    CK(cudaEventSynchronize(c->snap_done[buf]));   // iteration - 2 finished with this buffer
    c->snap_iter[buf] = iteration;
    c->snap_seen[buf].assign(c->cfg.n_layers, 0);
  }
  for (int l = first_layer; l < first_layer + n_layers; ++l) c->snap_seen[buf][l] = 1;
  cudaStream_t p = static_cast<cudaStream_t>(producer);
  CK(cudaEventRecord(c->ev_tmp, p));
  CK(cudaStreamWaitEvent(c->side, c->ev_tmp, 0));
  const uint64_t lo = c->off[first_layer], hi = c->off[first_layer + n_layers];
  // with an active replica, or when sharded snapshots are on, only this rank's shard of the bucket
  // crosses PCIe (the rest is not read)
  const uint64_t psi = (uint64_t)c->psi, rk = (uint64_t)c->cfg.rank, wd = (uint64_t)c->cfg.world;
  const bool shard = c->rep_active || c->snap_sharded;
  const uint64_t sb = c->rep_active ? c->rep_sb : psi * rk / wd, se = c->rep_active ? c->rep_se : psi * (rk + 1) / wd;
  const uint64_t a = shard ? std::max(lo, sb) : lo;
  const uint64_t z = shard ? std::min(hi, se) : hi;
  int h;
  ld::prof_begin(c, "snapshot_d2h", c->side, &h);
  if (a < z)
    CK(cudaMemcpyAsync(c->snap_host[buf] + a, grad_bucket + (a - lo), (z - a) * 4, cudaMemcpyDeviceToHost, c->side));
  ld::prof_end(c, h, c->side);
  CK(cudaEventRecord(c->snap_done[buf], c->side));
  return LOWDIFF_OK;
}

// Backward-order buckets of >= min_bytes contiguous layers (LowDiff+ snapshot granularity).
lowdiff_status lowdiff_bucket_plan(int32_t n_layers, const int64_t* numel, int64_t min_bytes, int32_t* first,
                                   int32_t* count, int32_t cap, int32_t* n_buckets) {
  if (n_layers < 1 || !numel || min_bytes < 0 || !first || !count || !n_buckets || cap < 0) return LOWDIFF_E_INVALID;
  for (int32_t l = 0; l < n_layers; ++l)
    if (numel[l] < 1) return LOWDIFF_E_INVALID;
  int32_t n = 0, hi = n_layers;   // the bucket being formed ends (exclusive) at layer hi
  int64_t bytes = 0;
  for (int32_t l = n_layers - 1; l >= 0; --l) {
    bytes += 4 * numel[l];
    if (bytes >= min_bytes && l > 0) {
      if (n == cap) return LOWDIFF_E_DIM;
      first[n] = l, count[n] = hi - l, ++n;
      hi = l, bytes = 0;
    }
  }
  // the bucket holding layer 0 takes whatever is left (possibly below min_bytes)
  if (bytes > 0 || n == 0) {
    if (n == cap) return LOWDIFF_E_DIM;
    first[n] = 0, count[n] = hi, ++n;
  }
  *n_buckets = n;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_snapshot_shard(lowdiff_ctx* c, int32_t enable) {
  lowdiff_status st = entry(c);
  if (st) return st;
  c->snap_sharded = enable != 0;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_snapshot_wait(lowdiff_ctx* c, int64_t iteration, const float** host_grad) {
  lowdiff_status st = entry(c);
  if (st) return st;
  const int buf = (int)(iteration & 1);
  if (iteration < 0 || c->snap_iter[buf] != iteration) return fail(c, LOWDIFF_E_STATE, "snapshot_wait: unknown iteration");
  for (uint8_t x : c->snap_seen[buf])
    if (!x) return fail(c, LOWDIFF_E_STATE, "snapshot_wait: some layer of the iteration was not snapshotted");
  CK(cudaEventSynchronize(c->snap_done[buf]));
  if (host_grad) *host_grad = c->snap_host[buf];
  return LOWDIFF_OK;
}

// ---------------------------------------------------------------- LowDiff+ CPU replica (NEXT-3)
// Worker: applies queued snapshot gradients to the host shard in order (ld::host_adam/host_sgd,
// replica.cpp), and hands persist requests to a writer thread through a staging copy.
static void replica_loop(lowdiff_ctx* c) {
  cudaSetDevice(c->device);
  const uint64_t S = c->rep_se - c->rep_sb;
  for (;;) {
    ld::RepJob j;
    {
      std::unique_lock<std::mutex> lk(c->rep_mu);
      c->rep_cv.wait(lk, [&] { return c->rep_stop || !c->rep_q.empty(); });
      if (c->rep_q.empty()) return;
      j = c->rep_q.front();
      c->rep_q.pop_front();
      c->rep_busy = 1;
    }
    cudaError_t e = cudaSuccess;
    if (j.kind == 0) {
      e = cudaEventSynchronize(c->rep_init_done);
    } else if (j.kind == 1) {
      const int buf = (int)(j.iteration & 1);
      e = cudaEventSynchronize(c->snap_done[buf]);
      if (e == cudaSuccess) {
        const int64_t t0 = now_ns();
        const float* G = c->snap_host[buf] + c->rep_sb;
        if (c->cfg.optim == LOWDIFF_ADAM)
          ld::host_adam((int64_t)S, G, c->cfg.adam, j.sc, c->rep_host, c->rep_host + S, c->rep_host + 2 * S,
                        c->rep_threads);
        else
          ld::host_sgd((int64_t)S, G, j.sc.lr, c->rep_host, c->rep_threads);
        c->rep_ns += now_ns() - t0;
      }
    } else if (c->cfg.ckpt_dir && c->cfg.write_files) {
      if (c->rep_writer.joinable()) c->rep_writer.join();
      c->rep_stage.assign(c->rep_host, c->rep_host + 3 * S);
      const int64_t it = j.iteration;
      c->rep_writer = std::thread([c, it]() {
        const int64_t t0 = now_ns();
        std::string err;
        lowdiff_status s2 = write_ldf(c->cfg, c->ckpt_dir, it, (uint64_t)c->psi, c->rep_sb, c->rep_se,
                                      c->rep_stage.data(), &err);
        if (s2) set_deferred(c, s2, err);
        else { c->files_written += 1; c->bytes_written += (int64_t)(100 + 12 * (c->rep_se - c->rep_sb)); }
        c->writer_ns += now_ns() - t0;
      });
    }
    if (e != cudaSuccess) set_deferred(c, LOWDIFF_E_CUDA, std::string("replica: ") + cudaGetErrorString(e));
    {
      std::lock_guard<std::mutex> g(c->rep_mu);
      if (j.kind != 2) c->rep_iter = j.iteration;
      c->rep_busy = 0;
    }
    c->rep_done_cv.notify_all();
  }
}

// drain the queue and the persist writer (worker stays alive)


static void replica_push(lowdiff_ctx* c, const ld::RepJob& j) {
  {
    std::lock_guard<std::mutex> g(c->rep_mu);
    c->rep_q.push_back(j);
  }
  c->rep_cv.notify_one();
}

lowdiff_status lowdiff_replica_init(lowdiff_ctx* c, int64_t iteration, const float* p, const float* m, const float* v,
                                    int32_t threads, void* producer) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!p || iteration < 0 || threads < 1) return fail(c, LOWDIFF_E_INVALID, "replica_init: bad argument");
  if (c->cfg.optim == LOWDIFF_ADAM && (!m || !v)) return fail(c, LOWDIFF_E_INVALID, "replica_init: Adam needs m and v");
  replica_drain(c);
  replica_shutdown(c);
  const uint64_t sb = (uint64_t)c->psi * c->cfg.rank / c->cfg.world;
  const uint64_t se = (uint64_t)c->psi * (c->cfg.rank + 1) / c->cfg.world;
  const uint64_t S = se - sb;
  if (!c->rep_host || c->rep_se - c->rep_sb != S) {
    if (c->rep_host) cudaFreeHost(c->rep_host);
    c->rep_host = nullptr;
    CK(cudaHostAlloc((void**)&c->rep_host, std::max<size_t>(1, 3 * S) * 4, cudaHostAllocDefault));
  }
  if (!c->rep_init_done) CK(cudaEventCreateWithFlags(&c->rep_init_done, cudaEventDisableTiming));
  c->rep_sb = sb;
  c->rep_se = se;
  c->rep_threads = threads;
  cudaStream_t pr = static_cast<cudaStream_t>(producer);
  CK(cudaEventRecord(c->ev_tmp, pr));
  CK(cudaStreamWaitEvent(c->side, c->ev_tmp, 0));
  const float* src[3] = {p, m, v};
  for (int a = 0; a < 3; ++a) {
    if (src[a]) CK(cudaMemcpyAsync(c->rep_host + a * S, src[a] + sb, S * 4, cudaMemcpyDeviceToHost, c->side));
    else std::memset(c->rep_host + a * S, 0, S * 4);
  }
  CK(cudaEventRecord(c->rep_init_done, c->side));
  CK(cudaStreamWaitEvent(pr, c->rep_init_done, 0));
  c->rep_iter = -1;
  c->rep_tail = iteration;
  c->rep_active = true;
  c->rep_thread = std::thread(replica_loop, c);
  replica_push(c, {0, iteration, {0.f, 0.f, 0.f}});
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_replica_step(lowdiff_ctx* c, int64_t iteration, const lowdiff_step_scalars* scalars) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!c->rep_active) return fail(c, LOWDIFF_E_STATE, "replica_step: no replica (call lowdiff_replica_init)");
  if (!scalars) return fail(c, LOWDIFF_E_INVALID, "replica_step: NULL scalars");
  if (iteration != c->rep_tail + 1)
    return fail(c, LOWDIFF_E_STATE, "replica_step: expected iteration " + std::to_string(c->rep_tail + 1));
  const int buf = (int)(iteration & 1);
  if (c->snap_iter[buf] != iteration) return fail(c, LOWDIFF_E_STATE, "replica_step: iteration was not snapshotted");
  for (uint8_t x : c->snap_seen[buf])
    if (!x) return fail(c, LOWDIFF_E_STATE, "replica_step: some layer of the iteration was not snapshotted");
  c->rep_tail = iteration;
  replica_push(c, {1, iteration, *scalars});
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_replica_persist(lowdiff_ctx* c) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!c->rep_active) return fail(c, LOWDIFF_E_STATE, "replica_persist: no replica");
  if (!c->cfg.ckpt_dir) return fail(c, LOWDIFF_E_INVALID, "replica_persist: no ckpt_dir");
  replica_push(c, {2, c->rep_tail, {0.f, 0.f, 0.f}});
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_replica_wait(lowdiff_ctx* c, int64_t* iteration, const float** p, const float** m,
                                    const float** v, int64_t* shard_begin, int64_t* shard_end) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->rep_active) return fail(c, LOWDIFF_E_STATE, "replica_wait: no replica");
  replica_drain(c);
  if ((st = take_deferred(c))) return st;
  const uint64_t S = c->rep_se - c->rep_sb;
  if (iteration) *iteration = c->rep_iter.load();
  if (p) *p = c->rep_host;
  if (m) *m = c->rep_host + S;
  if (v) *v = c->rep_host + 2 * S;
  if (shard_begin) *shard_begin = (int64_t)c->rep_sb;
  if (shard_end) *shard_end = (int64_t)c->rep_se;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_replica_restore(lowdiff_ctx* c, float* p, float* m, float* v, int64_t* iteration, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->rep_active) return fail(c, LOWDIFF_E_STATE, "replica_restore: no replica");
  if (!p || (c->cfg.optim == LOWDIFF_ADAM && (!m || !v))) return fail(c, LOWDIFF_E_INVALID, "replica_restore: bad argument");
  if (c->cfg.world > 1 && !c->comm) return fail(c, LOWDIFF_E_STATE, "replica_restore: world > 1 needs an NCCL context");
  replica_drain(c);
  if ((st = take_deferred(c))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t S = c->rep_se - c->rep_sb;
  float* dst[3] = {p, m, v};
  for (int a = 0; a < 3; ++a)
    if (dst[a] && S) CK(cudaMemcpyAsync(dst[a] + c->rep_sb, c->rep_host + a * S, S * 4, cudaMemcpyHostToDevice, s));
  if (c->comm && (st = bcast_shards(c, dst, s))) return st;   // world 1 with NCCL: a 1-rank broadcast
  CK(cudaStreamSynchronize(s));
  if (iteration) *iteration = c->rep_iter.load();
  // training resumes at rep_iter + 1: drain the persistence of the abandoned steps, then let the next
  // batch_persist start anywhere (its first call retires the abandoned run's files, api.cpp)
  if ((st = lowdiff_sync(c))) return st;
  c->next_iter = -1;
  c->u_next_iter = -1;
  return LOWDIFF_OK;
}

}  // extern "C"
