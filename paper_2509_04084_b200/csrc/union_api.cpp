// C-ABI implementation of liblowdiff (part 3): union-compacted differentials -- compaction
// (union.cu), .ldu persistence, recovery from .ldu (R-29, §4.7).
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

void union_drain(lowdiff_ctx* c) {
  if (!c->u_writer.joinable()) return;
  std::unique_lock<std::mutex> lk(c->u_mu);
  c->u_flush = true;
  c->u_cv.notify_all();
  c->u_cv_idle.wait(lk, [&] { return c->u_q.empty() && !c->u_flush && !c->u_busy; });
}

void union_shutdown(lowdiff_ctx* c) {
  if (c->u_writer.joinable()) {
    {
      std::lock_guard<std::mutex> g(c->u_mu);
      c->u_stop = true;
      c->u_cv.notify_all();
    }
    c->u_writer.join();
  }
  for (auto*& b : c->u_buf) if (b) { cudaFree(b); b = nullptr; }
  if (c->u_cnt_dev) cudaFree(c->u_cnt_dev);
  if (c->u_cnt_host) cudaFreeHost(c->u_cnt_host);
  for (auto e : c->u_ready) if (e) cudaEventDestroy(e);
  if (c->u_stream) cudaStreamDestroy(c->u_stream);
  if (c->union_scratch) cudaFree(c->union_scratch);
}

}  // namespace api
}  // namespace ld

extern "C" {

// ---------------------------------------------------------------- union-compacted differentials (NEXT-4)
// C^U_t: this rank's shard of the synchronised compressed gradient as an index -> value dictionary
// (R-29; union.cu).  .ldu layout: DESIGN.md §3.
lowdiff_status lowdiff_union_compact(lowdiff_ctx* c, int32_t world, const uint32_t* gathered, int64_t begin,
                                     int64_t end, uint32_t* out, int64_t cap, uint64_t* count_dev, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!gathered || !out || !count_dev || world < 1 || world > 65535)
    return fail(c, LOWDIFF_E_INVALID, "union_compact: bad argument");
  if (begin < 0 || end < begin || end > c->psi) return fail(c, LOWDIFF_E_DIM, "union_compact: range outside [0, Psi]");
  const int64_t worst = std::min<int64_t>((int64_t)world * c->K, end - begin);
  if (cap < worst) return fail(c, LOWDIFF_E_INVALID, "union_compact: cap below min(world * K, end - begin)");
  if ((reinterpret_cast<uintptr_t>(out) & 3u) || (reinterpret_cast<uintptr_t>(count_dev) & 7u))
    return fail(c, LOWDIFF_E_INVALID, "union_compact: misaligned buffer");
  CK(ld::launch_union(c, world, c->cfg.mean != 0, gathered, (uint64_t)begin, (uint64_t)end, out, (uint64_t)cap,
                      reinterpret_cast<unsigned long long*>(count_dev), static_cast<cudaStream_t>(stream)));
  return LOWDIFF_OK;
}

struct UBlock { int64_t it; lowdiff_step_scalars sc; std::vector<uint32_t> data; uint64_t n; };   // idx[n] | val[n]

static std::string union_name(const std::string& dir, int rank, int64_t first) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "/ld_union_r%03d_%012lld.ldu", rank, (long long)first);
  return dir + buf;
}

// 80-byte header + hyper (32 B) + layer table (16 B per layer) of a .ldu file; flags bit 2 marks
// an accumulated batch (one block covering n_iters iterations)
static std::vector<uint8_t> ldu_prefix(const lowdiff_ctx* c, int64_t first, uint32_t n_iters, bool accumulated) {
  std::vector<uint8_t> b(112 + 16 * (size_t)c->cfg.n_layers, 0);
  const uint16_t ver = 1,
                 flags = (uint16_t)((c->cfg.error_feedback ? 1 : 0) | (c->cfg.mean ? 2 : 0) | (accumulated ? 4 : 0));
  const uint32_t rk = (uint32_t)c->cfg.rank, wd = (uint32_t)c->cfg.world, nl = (uint32_t)c->cfg.n_layers;
  const uint32_t ppm = c->cfg.density_ppm, opt = (uint32_t)c->cfg.optim;
  const uint64_t psi = (uint64_t)c->psi, K = (uint64_t)c->K, sb = psi * rk / wd, se = psi * (rk + 1) / wd;
  const uint64_t fi = (uint64_t)first;
  std::memcpy(b.data(), "LDU1", 4);
  std::memcpy(b.data() + 4, &ver, 2);
  std::memcpy(b.data() + 6, &flags, 2);
  std::memcpy(b.data() + 8, &rk, 4);
  std::memcpy(b.data() + 12, &wd, 4);
  std::memcpy(b.data() + 16, &fi, 8);
  std::memcpy(b.data() + 24, &n_iters, 4);
  std::memcpy(b.data() + 28, &nl, 4);
  std::memcpy(b.data() + 32, &psi, 8);
  std::memcpy(b.data() + 40, &K, 8);
  std::memcpy(b.data() + 48, &ppm, 4);
  std::memcpy(b.data() + 52, &opt, 4);
  std::memcpy(b.data() + 56, &sb, 8);
  std::memcpy(b.data() + 64, &se, 8);
  std::memcpy(b.data() + 80, &c->cfg.adam, 20);
  for (int l = 0; l < c->cfg.n_layers; ++l) {
    const uint64_t n = (uint64_t)c->numel[l];
    const uint32_t k = c->k[l];
    std::memcpy(b.data() + 112 + 16 * (size_t)l, &n, 8);
    std::memcpy(b.data() + 120 + 16 * (size_t)l, &k, 4);
  }
  return b;
}

// Accumulated batch mode (R-30): tensor addition of the batch's
// dictionaries on the host, in iteration order: A[j] = (j in A ? A[j] : +0) + x.  Both lists are
// index-ascending, so one merge pass per iteration.
struct UAcc {
  int64_t first = -1, last = -1;
  uint32_t n_iters = 0;
  lowdiff_step_scalars sc{};
  std::vector<uint32_t> idx, val, tidx, tval;
};

static void accumulate_into(UAcc& A, const UBlock& B) {
  const uint64_t n = B.n;
  const uint32_t* bi = B.data.data();
  const uint32_t* bv = B.data.data() + n;
  A.tidx.clear();
  A.tval.clear();
  A.tidx.reserve(A.idx.size() + n);
  A.tval.reserve(A.idx.size() + n);
  size_t i = 0, e = 0;
  while (i < A.idx.size() || e < n) {
    if (e == n || (i < A.idx.size() && A.idx[i] < bi[e])) {
      A.tidx.push_back(A.idx[i]);
      A.tval.push_back(A.val[i]);
      ++i;
    } else {
      const bool both = i < A.idx.size() && A.idx[i] == bi[e];
      float before = 0.0f, x;
      if (both) std::memcpy(&before, &A.val[i], 4);
      std::memcpy(&x, &bv[e], 4);
      const float sum = before + x;
      uint32_t u;
      std::memcpy(&u, &sum, 4);
      A.tidx.push_back(bi[e]);
      A.tval.push_back(u);
      ++e;
      if (both) ++i;
    }
  }
  A.idx.swap(A.tidx);
  A.val.swap(A.tval);
  if (A.n_iters == 0) A.first = B.it;
  A.last = B.it;
  A.sc = B.sc;
  A.n_iters += 1;
}

// CRC trailer, *.tmp + rename (parts: everything before the CRC)
static void write_ldu(lowdiff_ctx* c, int64_t first, std::vector<std::pair<const void*, size_t>>& parts) {
  const int64_t t0 = now_ns();
  uint32_t crc = 0xFFFFFFFFu;
  size_t bytes = 4;
  for (auto& q : parts) {
    crc = ld::crc32c_update(crc, q.first, q.second);
    bytes += q.second;
  }
  crc ^= 0xFFFFFFFFu;
  parts.push_back({&crc, 4});
  std::string err;
  lowdiff_status st =
      ld::write_file_atomic(union_name(c->ckpt_dir, c->cfg.rank, first), parts, c->cfg.fsync != 0, &err);
  if (st) set_deferred(c, st, err);
  else { c->u_files += 1; c->u_bytes += (int64_t)bytes; }
  c->writer_ns += now_ns() - t0;
}

static void union_write_accumulated(lowdiff_ctx* c, UAcc& A) {
  if (A.n_iters == 0) return;
  if (c->cfg.ckpt_dir) {
    const std::vector<uint8_t> pre = ldu_prefix(c, A.first, A.n_iters, true);
    std::array<uint8_t, 32> h;
    h.fill(0);
    const uint64_t it = (uint64_t)A.last;
    const uint32_t n = (uint32_t)A.idx.size();
    std::memcpy(h.data(), &it, 8);
    std::memcpy(h.data() + 8, &A.sc, 12);
    std::memcpy(h.data() + 20, &n, 4);
    std::vector<std::pair<const void*, size_t>> parts{{pre.data(), pre.size()}, {h.data(), 32}};
    if (n) {
      parts.push_back({A.idx.data(), 4 * (size_t)n});
      parts.push_back({A.val.data(), 4 * (size_t)n});
    }
    write_ldu(c, A.first, parts);
  }
  A.idx.clear();
  A.val.clear();
  A.n_iters = 0;
  A.first = A.last = -1;
}

static void union_write(lowdiff_ctx* c, std::vector<UBlock>& batch) {
  if (batch.empty()) return;
  if (c->cfg.ckpt_dir) {
    const std::vector<uint8_t> pre = ldu_prefix(c, batch[0].it, (uint32_t)batch.size(), false);
    std::vector<std::array<uint8_t, 32>> heads(batch.size());
    std::vector<std::pair<const void*, size_t>> parts{{pre.data(), pre.size()}};
    for (size_t i = 0; i < batch.size(); ++i) {
      auto& h = heads[i];
      h.fill(0);
      const uint64_t it = (uint64_t)batch[i].it;
      const uint32_t n = (uint32_t)batch[i].n;
      std::memcpy(h.data(), &it, 8);
      std::memcpy(h.data() + 8, &batch[i].sc, 12);
      std::memcpy(h.data() + 20, &n, 4);
      parts.push_back({h.data(), 32});
      if (n) parts.push_back({batch[i].data.data(), 8 * (size_t)n});
    }
    write_ldu(c, batch[0].it, parts);
  }
  batch.clear();
}

static void union_loop(lowdiff_ctx* c) {
  cudaSetDevice(c->device);
  std::vector<UBlock> batch;
  UAcc acc;
  // writes whatever is pending (record batch or accumulated batch)
  auto write_pending = [&] {
    union_write(c, batch);
    union_write_accumulated(c, acc);
  };
  for (;;) {
    ld::UJob j{};
    bool have = false, flush = false;
    {
      std::unique_lock<std::mutex> lk(c->u_mu);
      c->u_cv.wait(lk, [&] { return c->u_stop || c->u_flush || !c->u_q.empty(); });
      if (!c->u_q.empty()) {
        j = c->u_q.front();
        c->u_q.pop_front();
        have = true;
      } else if (c->u_flush) {
        flush = true;
      }
      c->u_busy = 1;
    }
    if (have) {
      UBlock B{j.iteration, j.sc, {}, 0};
      cudaError_t e = cudaEventSynchronize(c->u_ready[j.buf]);
      bool bad = false;
      if (e == cudaSuccess) {
        const unsigned long long n = c->u_cnt_host[2 * j.buf];
        const uint32_t errc = (uint32_t)c->u_cnt_host[2 * j.buf + 1];
        if (errc > c->u_err_seen) {   // a non-finite accumulated gradient reached this iteration
          c->u_err_seen = errc;
          bad = true;
        } else {
          B.n = n;
          B.data.resize(2 * (size_t)n);
          if (n) {
            e = cudaMemcpyAsync(B.data.data(), c->u_buf[j.buf], 4 * (size_t)n, cudaMemcpyDeviceToHost, c->u_stream);
            if (e == cudaSuccess)
              e = cudaMemcpyAsync(B.data.data() + n, c->u_buf[j.buf] + c->u_cap, 4 * (size_t)n, cudaMemcpyDeviceToHost,
                                  c->u_stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(c->u_stream);
          }
        }
      }
      {
        std::lock_guard<std::mutex> g(c->u_mu);
        c->u_inuse[j.buf] = false;
        c->u_cv_free.notify_all();
      }
      if (e != cudaSuccess || bad) {
        set_deferred(c, e != cudaSuccess ? LOWDIFF_E_CUDA : LOWDIFF_E_NUMERIC,
                     e != cudaSuccess ? std::string("union differential copy: ") + cudaGetErrorString(e)
                                      : "non-finite accumulated gradient before union iteration " +
                                            std::to_string(j.iteration));
        write_pending();   // the chain stops before this iteration
      } else {
        c->u_entries += (int64_t)B.n;
        if (j.accumulate) {
          union_write(c, batch);   // a record batch in flight ends where accumulation starts
          const int64_t t0 = now_ns();
          accumulate_into(acc, B);
          c->writer_ns += now_ns() - t0;
          if ((int)acc.n_iters == c->b) union_write_accumulated(c, acc);
        } else {
          union_write_accumulated(c, acc);
          batch.push_back(std::move(B));
          if ((int)batch.size() == c->b) union_write(c, batch);
        }
      }
    } else if (flush) {
      write_pending();
      std::lock_guard<std::mutex> g(c->u_mu);
      c->u_flush = false;
    } else {
      write_pending();
      std::lock_guard<std::mutex> g(c->u_mu);
      c->u_busy = 0;
      c->u_cv_idle.notify_all();
      return;
    }
    std::lock_guard<std::mutex> g(c->u_mu);
    c->u_busy = 0;
    c->u_cv_idle.notify_all();
  }
}

// drain queued union blocks and write the partial batch (lowdiff_sync)


lowdiff_status lowdiff_union_persist(lowdiff_ctx* c, int64_t iteration, const lowdiff_step_scalars* scalars,
                                     const uint32_t* gathered, void* producer) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!scalars || !gathered) return fail(c, LOWDIFF_E_INVALID, "union_persist: NULL argument");
  if (c->u_next_iter >= 0 && iteration != c->u_next_iter)
    return fail(c, LOWDIFF_E_STATE, "union_persist: iteration " + std::to_string(iteration) + " after " +
                                        std::to_string(c->u_next_iter - 1) + " (must be consecutive)");
  if (c->u_next_iter < 0 && c->cfg.write_files) {   // persisting (re)starts here: retire the abandoned run
    if (c->full_writer.joinable()) c->full_writer.join();
    std::string err;
    if ((st = retire_from(c->cfg, iteration, 2 | 4, &err))) return fail(c, st, err);
  }
  const uint64_t psi = (uint64_t)c->psi, rk = (uint64_t)c->cfg.rank, wd = (uint64_t)c->cfg.world;
  const uint64_t sb = psi * rk / wd, se = psi * (rk + 1) / wd;
  if (!c->u_buf[0]) {   // first call: buffers sized for the worst case min(N K, shard)
    c->u_cap = std::max<uint64_t>(1, std::min<uint64_t>(wd * (uint64_t)c->K, se - sb));
    for (auto*& b : c->u_buf) CK(cudaMalloc((void**)&b, 2 * c->u_cap * 4));
    CK(cudaMalloc((void**)&c->u_cnt_dev, 2 * sizeof(unsigned long long)));
    CK(cudaHostAlloc((void**)&c->u_cnt_host, 4 * sizeof(unsigned long long), cudaHostAllocDefault));
    for (auto& e : c->u_ready) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&c->u_stream, cudaStreamNonBlocking));
    c->u_err_seen = c->err_seen.load();
    c->u_writer = std::thread(union_loop, c);
  }
  const int buf = (int)(iteration & 1);
  {
    std::unique_lock<std::mutex> lk(c->u_mu);
    if (c->u_inuse[buf]) {   // the writer still copies iteration - 2 out of this buffer
      const int64_t t0 = now_ns();
      c->u_cv_free.wait(lk, [&] { return !c->u_inuse[buf]; });
      c->stall_ns += now_ns() - t0;
    }
    c->u_inuse[buf] = true;
  }
  cudaStream_t s = static_cast<cudaStream_t>(producer);
  c->u_cnt_host[2 * buf] = 0;
  c->u_cnt_host[2 * buf + 1] = 0;
  CK(ld::launch_union(c, c->cfg.world, c->cfg.mean != 0, gathered, sb, se, c->u_buf[buf], c->u_cap, c->u_cnt_dev + buf, s));
  CK(cudaMemcpyAsync(&c->u_cnt_host[2 * buf], c->u_cnt_dev + buf, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&c->u_cnt_host[2 * buf + 1], c->plan.err, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(c->u_ready[buf], s));
  c->u_next_iter = iteration + 1;
  {
    std::lock_guard<std::mutex> g(c->u_mu);
    c->u_q.push_back(ld::UJob{iteration, *scalars, buf, c->u_accumulate != 0});
    c->u_cv.notify_all();
  }
  return LOWDIFF_OK;
}

// Accumulated batch mode switch (R-30): the union writer first writes the batch in flight
lowdiff_status lowdiff_set_batch_mode(lowdiff_ctx* c, int32_t mode) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (mode != LOWDIFF_BATCH_RECORD && mode != LOWDIFF_BATCH_ACCUMULATED)
    return fail(c, LOWDIFF_E_INVALID, "set_batch_mode: unknown mode");
  if ((mode == LOWDIFF_BATCH_ACCUMULATED) == (c->u_accumulate != 0)) return LOWDIFF_OK;
  union_drain(c);
  c->u_accumulate = mode == LOWDIFF_BATCH_ACCUMULATED;
  return take_deferred(c);
}

// recovery from .ldf + .ldu: the chain rules of lowdiff_recover; the replay is the fused kernel with
// one "rank" per step (the union is already merged and divided: sum mode, G = +0 + value)
static lowdiff_status union_recover_impl(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v,
                                         bool sharded, int64_t* recovered, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->cfg.ckpt_dir) return fail(c, LOWDIFF_E_INVALID, "recover_union: no ckpt_dir");
  if (!p) return fail(c, LOWDIFF_E_INVALID, "recover_union: NULL p");
  if ((st = lowdiff_sync(c))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t world = (uint32_t)c->cfg.world;
  const uint64_t psi = (uint64_t)c->psi, K = (uint64_t)c->K;
  std::map<int64_t, std::map<uint32_t, std::string>> fulls;
  std::vector<std::map<int64_t, std::string>> diffs(world);
  DIR* d = opendir(c->cfg.ckpt_dir);
  if (!d) return fail(c, LOWDIFF_E_IO, std::string("cannot open ") + c->cfg.ckpt_dir);
  while (dirent* de = readdir(d)) {
    unsigned r;
    long long it;
    if (parse_name(de->d_name, "full", "ldf", &r, &it) && r < world)
      fulls[it][r] = std::string(c->cfg.ckpt_dir) + "/" + de->d_name;
    else if (parse_name(de->d_name, "union", "ldu", &r, &it) && r < world)
      diffs[r][it] = std::string(c->cfg.ckpt_dir) + "/" + de->d_name;
  }
  closedir(d);
  int64_t F = -1;
  std::vector<std::string> full_paths;
  for (auto it = fulls.rbegin(); it != fulls.rend(); ++it) {
    if (target >= 0 && it->first > target) continue;
    if (it->second.size() == world) {
      F = it->first;
      for (uint32_t r = 0; r < world; ++r) full_paths.push_back(it->second[r]);
      break;
    }
  }
  if (F < 0) return fail(c, LOWDIFF_E_GAP, "no complete full checkpoint <= target");
  uint32_t optim = 0;
  float consts[5] = {0, 0, 0, 0, 0};
  uint16_t flags = 0;
  if ((st = load_full_shards(c, full_paths, F, sharded, p, m, v, &optim, consts, &flags))) return st;
  // index every needed rank's .ldu files: iteration -> (file, byte offset of its block, count);
  // files are verified (magic, CRC, header fields, block walk) when indexed
  const uint32_t r0 = sharded ? (uint32_t)c->cfg.rank : 0, r1 = sharded ? (uint32_t)c->cfg.rank + 1 : world;
  // replay units: iteration -> (file, byte offset of its block, count, iterations covered: 1, or b
  // for an accumulated batch keyed by its first iteration)
  struct Where { std::string path; size_t off; uint64_t n; int64_t span; };
  std::vector<std::map<int64_t, Where>> where(world);
  for (uint32_t r = r0; r < r1; ++r) {
    for (auto& fe : diffs[r]) {   // ascending first iteration: later files win
      std::vector<uint8_t> buf;
      if (!read_all(fe.second, buf)) return fail(c, LOWDIFF_E_IO, "cannot read " + fe.second);
      const size_t L = (size_t)c->cfg.n_layers;
      if (buf.size() < 116 + 16 * L || std::memcmp(buf.data(), "LDU1", 4) != 0 ||
          lowdiff_crc32c(buf.data(), buf.size() - 4) != rd<uint32_t>(buf.data() + buf.size() - 4) ||
          rd<uint32_t>(buf.data() + 8) != r || rd<uint32_t>(buf.data() + 12) != world ||
          rd<uint32_t>(buf.data() + 28) != (uint32_t)L || rd<uint64_t>(buf.data() + 32) != psi ||
          rd<uint64_t>(buf.data() + 40) != K || rd<uint32_t>(buf.data() + 48) != c->cfg.density_ppm ||
          rd<uint32_t>(buf.data() + 52) != optim || rd<uint64_t>(buf.data() + 56) != psi * r / world ||
          rd<uint64_t>(buf.data() + 64) != psi * (r + 1) / world)
        return fail(c, LOWDIFF_E_CORRUPT, "corrupt union file " + fe.second);
      const uint32_t n_it = rd<uint32_t>(buf.data() + 24);
      const bool accumulated = (rd<uint16_t>(buf.data() + 6) & 4u) != 0;
      size_t off = 112 + 16 * L;
      const uint32_t n_blocks = accumulated ? 1u : n_it;
      if (accumulated && n_it < 1) return fail(c, LOWDIFF_E_CORRUPT, "corrupt union file " + fe.second);
      for (uint32_t i = 0; i < n_blocks; ++i) {
        const int64_t it = accumulated ? fe.first + n_it - 1 : fe.first + i;
        if (off + 32 > buf.size() - 4 || (int64_t)rd<uint64_t>(buf.data() + off) != it)
          return fail(c, LOWDIFF_E_CORRUPT, "corrupt union file " + fe.second);
        const uint64_t n = rd<uint32_t>(buf.data() + off + 20);
        where[r][accumulated ? fe.first : it] = Where{fe.second, off, n, accumulated ? (int64_t)n_it : 1};
        off += 32 + 8 * n;
      }
      if (off != buf.size() - 4) return fail(c, LOWDIFF_E_CORRUPT, "corrupt union file " + fe.second);
    }
  }
  // the chain of replay units F+1, ...: every needed rank holds a unit starting there that covers
  // the same iterations; an accumulated batch is recovered whole or not at all (R-30)
  int64_t last = F;
  std::vector<int64_t> units;
  for (;;) {
    const int64_t t = last + 1;
    bool all = true;
    int64_t span = 0;
    for (uint32_t r = r0; r < r1 && all; ++r) {
      auto f = where[r].find(t);
      all = f != where[r].end();
      if (!all) break;
      if (r == r0) span = f->second.span;
      else if (f->second.span != span)
        return fail(c, LOWDIFF_E_CORRUPT, "ranks disagree on the batch starting at iteration " + std::to_string(t));
    }
    if (!all || (target >= 0 && t + span - 1 > target)) break;
    units.push_back(t);
    last = t + span - 1;
  }
  if (target >= 0 && last < target)
    return fail(c, LOWDIFF_E_GAP, "union chain has a gap (or an accumulated batch boundary) after " + std::to_string(last));
  const uint64_t lo = sharded ? psi * c->cfg.rank / world : 0, hi = sharded ? psi * (c->cfg.rank + 1) / world : psi;
  // replay in chunks of steps: block of step t = idx[Kc] | val[Kc], entries [0, U_t) valid
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  std::map<std::string, std::vector<uint8_t>> cache;
  lowdiff_status result = LOWDIFF_OK;
  const int64_t n_units = (int64_t)units.size();
  for (int64_t u0 = 0; u0 < n_units && result == LOWDIFF_OK;) {
    // grow the chunk of replay steps while its padded size stays within a quarter of free memory
    uint64_t Kc = 1;
    int64_t u1 = u0;
    for (int64_t u = u0; u < n_units; ++u) {
      uint64_t U = 0;
      for (uint32_t r = r0; r < r1; ++r) U += where[r][units[u]].n;
      const uint64_t k2 = std::max<uint64_t>(Kc, U);
      if (u > u0 && (uint64_t)(u - u0 + 1) * 8 * k2 > free_b / 4) break;
      Kc = k2;
      u1 = u;
    }
    const int64_t ns = u1 - u0 + 1;
    std::vector<uint32_t> host((size_t)ns * 2 * Kc, 0u), ranges((size_t)ns * 2, 0u);
    std::vector<lowdiff_step_scalars> scal((size_t)ns);
    for (int64_t u = u0; u <= u1 && result == LOWDIFF_OK; ++u) {
      const int64_t t = units[u];
      uint64_t at = 0;
      for (uint32_t r = r0; r < r1; ++r) {
        const Where& w = where[r][t];
        auto itc = cache.find(w.path);
        if (itc == cache.end()) {
          for (auto jt = cache.begin(); jt != cache.end();) {   // drop files this step no longer uses
            bool used = false;
            for (uint32_t q = r0; q < r1 && !used; ++q) used = where[q][t].path == jt->first;
            jt = used ? std::next(jt) : cache.erase(jt);
          }
          std::vector<uint8_t> buf;
          if (!read_all(w.path, buf)) { result = fail(c, LOWDIFF_E_IO, "cannot read " + w.path); break; }
          itc = cache.emplace(w.path, std::move(buf)).first;
        }
        const uint8_t* blk = itc->second.data() + w.off;
        lowdiff_step_scalars sc;
        std::memcpy(&sc, blk + 8, 12);
        if (r == r0) scal[u - u0] = sc;
        else if (std::memcmp(&sc, &scal[u - u0], 12) != 0) {
          result = fail(c, LOWDIFF_E_CORRUPT, "ranks disagree on the scalars of iteration " + std::to_string(t));
          break;
        }
        const uint64_t sbr = psi * r / world, ser = psi * (r + 1) / world;
        const uint32_t* idx = reinterpret_cast<const uint32_t*>(blk + 32);
        for (uint64_t e = 0; e < w.n; ++e)
          if (idx[e] < sbr || idx[e] >= ser || (e && idx[e] <= idx[e - 1])) {
            result = fail(c, LOWDIFF_E_CORRUPT, "union entries outside their shard or not ascending in " + w.path);
            break;
          }
        if (result) break;
        uint32_t* dst = host.data() + (size_t)(u - u0) * 2 * Kc;
        std::memcpy(dst + at, idx, 4 * w.n);
        std::memcpy(dst + Kc + at, idx + w.n, 4 * w.n);
        at += w.n;
      }
      ranges[2 * (size_t)(u - u0) + 1] = (uint32_t)at;
    }
    if (result) break;
    uint32_t* d_diffs = nullptr;
    uint32_t* d_ranges = nullptr;
    float* scal_dev = nullptr;
    cudaError_t e = cudaMalloc((void**)&d_diffs, host.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&d_ranges, ranges.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&scal_dev, scal.size() * 12);
    if (e == cudaSuccess) e = cudaMemcpy(d_diffs, host.data(), host.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_ranges, ranges.data(), ranges.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(scal_dev, scal.data(), scal.size() * 12, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = ld::launch_replay(c, (int)optim, false, consts, 1, ns, d_diffs, scal_dev, lo, hi, d_ranges, p + lo,
                            m ? m + lo : nullptr, v ? v + lo : nullptr, s, Kc);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (d_diffs) cudaFree(d_diffs);
    if (d_ranges) cudaFree(d_ranges);
    if (scal_dev) cudaFree(scal_dev);
    if (e != cudaSuccess) result = cuda_fail(c, e, "union replay");
    u0 = u1 + 1;
  }
  if (result) return result;
  if (recovered) *recovered = last;
  c->u_next_iter = -1;   // persisting may resume at last + 1 (the abandoned run is retired then)
  c->next_iter = -1;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_recover_union(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int32_t sharded,
                                     int64_t* recovered, void* stream) {
  return union_recover_impl(c, target, p, m, v, sharded != 0, recovered, stream);
}

}  // extern "C"
