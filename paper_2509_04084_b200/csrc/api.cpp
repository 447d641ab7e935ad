// C-ABI implementation of liblowdiff: context, NCCL exchange, reuse queue -> pinned ring ->
// writer thread, full checkpoints, chain scan + recovery, LowDiff+ snapshots.
// The GPU kernels live in compress.cu and merge_replay.cu.  See include/lowdiff.h.
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

#include "internal.h"

using ld::DevPlan;

namespace {

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

lowdiff_status fail(lowdiff_ctx* c, lowdiff_status st, const std::string& msg) {
  std::lock_guard<std::mutex> g(c->err_mu);
  c->last_error = msg;
  if (st == LOWDIFF_E_CUDA || st == LOWDIFF_E_NCCL) c->poisoned = st;
  return st;
}

lowdiff_status cuda_fail(lowdiff_ctx* c, cudaError_t e, const char* what) {
  return fail(c, LOWDIFF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
  } while (0)

lowdiff_status entry(lowdiff_ctx* c) {
  if (!c) return LOWDIFF_E_INVALID;
  if (c->poisoned != LOWDIFF_OK) return c->poisoned;
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  return LOWDIFF_OK;
}

lowdiff_status take_deferred(lowdiff_ctx* c) {
  std::lock_guard<std::mutex> g(c->err_mu);
  lowdiff_status d = c->deferred;
  c->deferred = LOWDIFF_OK;
  return d;
}

void set_deferred(lowdiff_ctx* c, lowdiff_status st, const std::string& msg) {
  std::lock_guard<std::mutex> g(c->err_mu);
  if (c->deferred == LOWDIFF_OK) c->deferred = st;
  c->last_error = msg;
  if (st == LOWDIFF_E_CUDA) c->poisoned = st;
}

// 96-byte .ldf header: shard [sb, se) of p | m | v after `iteration` steps
std::vector<uint8_t> ldf_header(const lowdiff_config& cfg, int64_t iteration, uint64_t psi, uint64_t sb, uint64_t se) {
  std::vector<uint8_t> hdr(96, 0);
  std::memcpy(hdr.data(), "LDF1", 4);
  const uint16_t ver = 1, flags = (uint16_t)((cfg.error_feedback ? 1 : 0) | (cfg.mean ? 2 : 0));
  const uint32_t rk = (uint32_t)cfg.rank, wd = (uint32_t)cfg.world, opt = (uint32_t)cfg.optim;
  const uint64_t itu = (uint64_t)iteration;
  std::memcpy(hdr.data() + 4, &ver, 2);
  std::memcpy(hdr.data() + 6, &flags, 2);
  std::memcpy(hdr.data() + 8, &rk, 4);
  std::memcpy(hdr.data() + 12, &wd, 4);
  std::memcpy(hdr.data() + 16, &itu, 8);
  std::memcpy(hdr.data() + 24, &psi, 8);
  std::memcpy(hdr.data() + 32, &sb, 8);
  std::memcpy(hdr.data() + 40, &se, 8);
  std::memcpy(hdr.data() + 48, &opt, 4);
  std::memcpy(hdr.data() + 64, &cfg.adam, 20);
  return hdr;
}

// write header + body (3 * S floats) + CRC-32C atomically
lowdiff_status write_ldf(const lowdiff_config& cfg, const std::string& dir, int64_t iteration, uint64_t psi,
                         uint64_t sb, uint64_t se, const float* body, std::string* err) {
  const std::vector<uint8_t> hdr = ldf_header(cfg, iteration, psi, sb, se);
  const size_t bytes = 3 * (se - sb) * 4;
  uint32_t crc = ld::crc32c_update(0xFFFFFFFFu, hdr.data(), hdr.size());
  crc = ld::crc32c_update(crc, body, bytes) ^ 0xFFFFFFFFu;
  return ld::write_file_atomic(ld::full_name(dir, cfg.rank, iteration), {{hdr.data(), hdr.size()}, {body, bytes}, {&crc, 4}},
                               cfg.fsync != 0, err);
}

uint64_t k_rule(uint64_t n, uint32_t ppm) {   // DESIGN.md R-3
  uint64_t k = n * ppm / 1000000ull;
  return std::max<uint64_t>(1, std::min(k, n));
}

template <class T>
lowdiff_status upload(lowdiff_ctx* c, const std::vector<T>& h, T** d) {
  void* p = nullptr;
  size_t bytes = std::max<size_t>(1, h.size()) * sizeof(T);
  CK(cudaMalloc(&p, bytes));
  c->dev_allocs.push_back(p);
  if (!h.empty()) CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *d = static_cast<T*>(p);
  return LOWDIFF_OK;
}

lowdiff_status dalloc(lowdiff_ctx* c, size_t bytes, void** d) {
  CK(cudaMalloc(d, std::max<size_t>(bytes, 16)));
  c->dev_allocs.push_back(*d);
  return LOWDIFF_OK;
}

// ---------------------------------------------------------------- chunk plan
lowdiff_status build_plan(lowdiff_ctx* c) {
  const int L = c->cfg.n_layers;
  std::vector<uint64_t> off(L + 1), koff(L);
  std::vector<uint32_t> kk(L);
  std::vector<int32_t> small, large, chunk0, cslot;
  std::vector<uint64_t> cbase, clo, chi;
  for (int l = 0; l < L; ++l) {
    off[l + 1] = off[l] + (uint64_t)c->numel[l];
    kk[l] = (uint32_t)k_rule((uint64_t)c->numel[l], c->cfg.density_ppm);
    koff[l] = l ? koff[l - 1] + kk[l - 1] : 0;
  }
  for (int l = 0; l < L; ++l) {
    const uint64_t lo = off[l], hi = off[l + 1];
    if (hi - lo <= (uint64_t)ld::kSmallMax) { small.push_back(l); continue; }
    const int slot = (int)large.size();
    large.push_back(l);
    chunk0.push_back((int32_t)cslot.size());
    for (uint64_t b = lo & ~3ull; b < hi; b += ld::kChunk) {
      cslot.push_back(slot);
      cbase.push_back(b);
      clo.push_back(std::max(b, lo));
      chi.push_back(std::min(b + ld::kChunk, hi));
    }
  }
  chunk0.push_back((int32_t)cslot.size());
  c->off = off;
  c->koff = koff;
  c->k = kk;
  c->psi = (int64_t)off[L];
  c->K = (int64_t)(koff[L - 1] + kk[L - 1]);

  DevPlan& P = c->plan;
  P.n_layers = L;
  P.n_small = (int)small.size();
  P.n_large = (int)large.size();
  P.n_chunks = (int)cslot.size();
  lowdiff_status st;
  uint64_t* d_off; uint32_t* d_k; uint64_t* d_koff; int32_t *d_small, *d_large, *d_c0, *d_cslot;
  uint64_t *d_cb, *d_clo, *d_chi;
  if ((st = upload(c, off, &d_off)) || (st = upload(c, kk, &d_k)) || (st = upload(c, koff, &d_koff)) ||
      (st = upload(c, small, &d_small)) || (st = upload(c, large, &d_large)) || (st = upload(c, chunk0, &d_c0)) ||
      (st = upload(c, cslot, &d_cslot)) || (st = upload(c, cbase, &d_cb)) || (st = upload(c, clo, &d_clo)) ||
      (st = upload(c, chi, &d_chi)))
    return st;
  P.layer_off = d_off; P.layer_k = d_k; P.layer_koff = d_koff;
  P.small_layers = d_small; P.large_layers = d_large; P.large_chunk0 = d_c0;
  P.chunk_slot = d_cslot; P.chunk_base = d_cb; P.chunk_lo = d_clo; P.chunk_hi = d_chi;
  const size_t nc = (size_t)std::max(1, P.n_chunks), nl = (size_t)std::max(1, P.n_large);
  void* p;
  if ((st = dalloc(c, nc * ld::kChunk * sizeof(uint64_t), &p))) return st; P.cand = (uint64_t*)p;
  if ((st = dalloc(c, nc * ld::kSegsPerChunk * sizeof(uint32_t), &p))) return st; P.seg_count = (uint32_t*)p;
  if ((st = dalloc(c, nc * 4 * 7, &p))) return st;
  P.chunk_count = (uint32_t*)p; P.chunk_gt = P.chunk_count + nc; P.chunk_eq = P.chunk_gt + nc;
  P.chunk_out = P.chunk_eq + nc; P.chunk_take = P.chunk_out + nc; P.refill_list = P.chunk_take + nc;
  P.refill_list2 = P.refill_list + nc;
  if ((st = dalloc(c, nl * (2048 + 2048 + 512) * 4, &p))) return st; P.hist = (uint32_t*)p;
  if ((st = dalloc(c, nl * sizeof(ld::LayerSel), &p))) return st; P.sel = (ld::LayerSel*)p;
  CK(cudaMemset(P.sel, 0, nl * sizeof(ld::LayerSel)));   // band = 0: not yet adapted
  if ((st = dalloc(c, nl * 4, &p))) return st; P.thr = (uint32_t*)p;
  if ((st = dalloc(c, nl * 4, &p))) return st; P.sel_T = (uint32_t*)p;
  if ((st = dalloc(c, nl * 4, &p))) return st; P.layer_total = (uint32_t*)p;
  CK(cudaMemset(P.layer_total, 0, nl * 4));   // then kept zero between calls by layer_scan_kernel
  if ((st = dalloc(c, nl * 4, &p))) return st; P.sel_cut = (uint32_t*)p;
  if ((st = dalloc(c, nl * 4, &p))) return st; P.thr_safe = (uint32_t*)p;
  if ((st = dalloc(c, (size_t)nc * 8, &p))) return st; P.chunk_state = (unsigned long long*)p;
  CK(cudaMemset(P.thr, 0xFF, nl * 4));   // no speculative band before the first call
  CK(cudaMemset(P.thr_safe, 0xFF, nl * 4));
  CK(cudaMemset(P.sel_T, 0xFF, nl * 4));  // no previous k-th key (no drift estimate yet)
  if ((st = dalloc(c, 8 * 4, &p))) return st; P.counters = (uint32_t*)p;
  if ((st = dalloc(c, 4 * 4, &p))) return st; P.err = (uint32_t*)p;
  CK(cudaMemset(P.err, 0, 16));
  CK(cudaMemset(P.err + 1, 0xFF, 4));
  return LOWDIFF_OK;
}

// ---------------------------------------------------------------- writer thread
void write_batch(lowdiff_ctx* c, const std::vector<int>& batch) {
  if (!c->cfg.write_files || batch.empty()) return;
  const int64_t t0 = now_ns();
  std::vector<uint8_t> pre = c->prefix;
  const uint64_t first = (uint64_t)c->slots[batch[0]].iteration;
  const uint32_t n = (uint32_t)batch.size();
  std::memcpy(pre.data() + 16, &first, 8);
  std::memcpy(pre.data() + 24, &n, 4);
  std::vector<std::pair<const void*, size_t>> parts;
  parts.push_back({pre.data(), pre.size()});
  uint32_t crc = ld::crc32c_update(0xFFFFFFFFu, pre.data(), pre.size());
  const size_t blk = 32 + 8 * (size_t)c->K;
  for (int s : batch) {
    parts.push_back({c->slots[s].host, blk});
    crc = ld::crc32c_update(crc, c->slots[s].host, blk);
  }
  crc ^= 0xFFFFFFFFu;
  parts.push_back({&crc, 4});
  std::string err;
  lowdiff_status st = ld::write_file_atomic(ld::batch_name(c->ckpt_dir, c->cfg.rank, (int64_t)first), parts,
                                            c->cfg.fsync != 0, &err);
  if (st != LOWDIFF_OK) {
    set_deferred(c, st, err);
  } else {
    c->files_written += 1;
    size_t tot = 0;
    for (auto& p : parts) tot += p.second;
    c->bytes_written += (int64_t)tot;
  }
  c->writer_ns += now_ns() - t0;
}

void release(lowdiff_ctx* c, std::vector<int>& batch) {
  std::lock_guard<std::mutex> g(c->mu);
  for (int s : batch) c->free_slots.push_back(s);
  batch.clear();
  c->cv_free.notify_all();
}


void writer_loop(lowdiff_ctx* c) {
  std::vector<int> batch;
  cudaSetDevice(c->device);
  for (;;) {
    int slot = -1;
    bool do_flush = false, quit = false;
    {
      std::unique_lock<std::mutex> lk(c->mu);
      c->cv_work.wait(lk, [&] { return c->stop || c->flush_req || !c->queued.empty(); });
      if (!c->queued.empty()) {
        slot = c->queued.front();
        c->queued.pop_front();
        c->writer_busy = 1;
      } else if (c->flush_req) {
        do_flush = true;
        c->writer_busy = 1;
      } else {
        quit = true;
      }
    }
    if (slot >= 0) {
      ld::Slot& S = c->slots[slot];
      cudaError_t e = cudaEventSynchronize(S.done);
      bool drop = false;
      if (e != cudaSuccess) {
        set_deferred(c, LOWDIFF_E_CUDA, std::string("D2H of a differential: ") + cudaGetErrorString(e));
        drop = true;
      } else if (S.err_host[0] > c->err_seen.load()) {
        c->err_seen = S.err_host[0];   // device counter of non-finite events (never reset)
        char msg[160];
        std::snprintf(msg, sizeof msg, "non-finite accumulated gradient before iteration %lld (first layer %u)",
                      (long long)S.iteration, S.err_host[1]);
        set_deferred(c, LOWDIFF_E_NUMERIC, msg);
        drop = true;
      }
      if (drop) {
        write_batch(c, batch);      // keep what is consecutive; the chain stops before this iteration
        release(c, batch);
        std::vector<int> one{slot};
        release(c, one);
      } else {
        batch.push_back(slot);
        if ((int)batch.size() == c->b) {
          write_batch(c, batch);
          release(c, batch);
        }
      }
    } else if (do_flush) {
      write_batch(c, batch);
      release(c, batch);
      std::lock_guard<std::mutex> g(c->mu);
      c->flush_req = false;
    } else if (quit) {
      write_batch(c, batch);
      release(c, batch);
      return;
    }
    std::lock_guard<std::mutex> g(c->mu);
    c->writer_busy = 0;
    c->cv_idle.notify_all();
  }
}

// ---------------------------------------------------------------- chain scan (recovery)
struct Chain {
  int64_t F = -1, last = -1;
  std::vector<std::string> full_paths;                               // [world]
  std::vector<std::map<int64_t, std::pair<std::string, uint32_t>>> where;  // rank -> t -> (file, block)
};

bool parse_name(const char* name, const char* kind, const char* ext, unsigned* rank, long long* it) {
  // ld_<kind>_r%03u_%012lld.<ext>
  char pat[64];
  std::snprintf(pat, sizeof pat, "ld_%s_r%%3u_%%12lld.%%3s", kind);
  char tail[8] = {0};
  if (std::strlen(name) != 3 + std::strlen(kind) + 2 + 3 + 1 + 12 + 1 + std::strlen(ext)) return false;
  if (std::sscanf(name, pat, rank, it, tail) != 3) return false;
  return std::strcmp(tail, ext) == 0;
}

bool read_all(const std::string& path, std::vector<uint8_t>& out) {
  int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) return false;
  struct stat sb;
  if (fstat(fd, &sb) != 0) { ::close(fd); return false; }
  out.resize((size_t)sb.st_size);
  size_t got = 0;
  while (got < out.size()) {
    ssize_t r = ::pread(fd, out.data() + got, out.size() - got, (off_t)got);
    if (r <= 0) { ::close(fd); return false; }
    got += (size_t)r;
  }
  ::close(fd);
  return true;
}

bool read_head(const std::string& path, uint8_t* buf, size_t n, size_t* fsize) {
  int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) return false;
  struct stat sb;
  bool ok = fstat(fd, &sb) == 0 && ::pread(fd, buf, n, 0) == (ssize_t)n;
  *fsize = ok ? (size_t)sb.st_size : 0;
  ::close(fd);
  return ok;
}

template <class T> T rd(const uint8_t* p) { T v; std::memcpy(&v, p, sizeof v); return v; }

lowdiff_status scan_chain(const lowdiff_config& cfg, int64_t target, Chain* ch, std::string* err) {
  const uint32_t world = (uint32_t)cfg.world;
  std::map<int64_t, std::map<uint32_t, std::string>> fulls;
  std::vector<std::map<int64_t, std::string>> diffs(world);
  DIR* d = opendir(cfg.ckpt_dir);
  if (!d) { *err = std::string("cannot open ") + cfg.ckpt_dir; return LOWDIFF_E_IO; }
  while (dirent* de = readdir(d)) {
    unsigned r; long long it;
    if (parse_name(de->d_name, "full", "ldf", &r, &it) && r < world)
      fulls[it][r] = std::string(cfg.ckpt_dir) + "/" + de->d_name;
    else if (parse_name(de->d_name, "diff", "ldb", &r, &it) && r < world)
      diffs[r][it] = std::string(cfg.ckpt_dir) + "/" + de->d_name;
  }
  closedir(d);
  ch->F = -1;
  for (auto it = fulls.rbegin(); it != fulls.rend(); ++it) {
    if (target >= 0 && it->first > target) continue;
    if (it->second.size() == world) {
      ch->F = it->first;
      ch->full_paths.clear();
      for (uint32_t r = 0; r < world; ++r) ch->full_paths.push_back(it->second[r]);
      break;
    }
  }
  if (ch->F < 0) { *err = "no complete full checkpoint <= target"; return LOWDIFF_E_GAP; }
  ch->where.assign(world, {});
  for (uint32_t r = 0; r < world; ++r) {
    for (auto& fe : diffs[r]) {     // ascending first iteration: later files win
      uint8_t h[64];
      size_t fsz = 0;
      if (!read_head(fe.second, h, 64, &fsz) || std::memcmp(h, "LDB1", 4) != 0) {
        *err = "unreadable batch file " + fe.second;
        return LOWDIFF_E_CORRUPT;
      }
      const uint32_t n = rd<uint32_t>(h + 24);
      for (uint32_t i = 0; i < n; ++i) ch->where[r][fe.first + i] = {fe.second, i};
    }
  }
  int64_t last = ch->F;
  for (;;) {
    const int64_t t = last + 1;
    if (target >= 0 && t > target) break;
    bool all = true;
    for (uint32_t r = 0; r < world && all; ++r) all = ch->where[r].count(t) > 0;
    if (!all) break;
    last = t;
  }
  if (target >= 0 && last < target) {
    *err = "differential chain has a gap after iteration " + std::to_string(last);
    return LOWDIFF_E_GAP;
  }
  ch->last = last;
  return LOWDIFF_OK;
}

}  // namespace

// ---------------------------------------------------------------- profiling helpers
namespace ld {
void prof_begin(lowdiff_ctx* c, const char* name, cudaStream_t s, int* handle) {
  *handle = -1;
  if (!c->prof) return;
  ProfRec r{name, nullptr, nullptr};
  // events come from a pool that survives prof_enable: recording stays cheap inside a timed loop
  const size_t need = 2 * (c->prof_recs.size() + 1);
  while (c->prof_pool.size() < need) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    c->prof_pool.push_back(e);
  }
  r.a = c->prof_pool[need - 2];
  r.b = c->prof_pool[need - 1];
  cudaEventRecord(r.a, s);
  c->prof_recs.push_back(r);
  *handle = (int)c->prof_recs.size() - 1;
}
void prof_end(lowdiff_ctx* c, int handle, cudaStream_t s) {
  if (handle < 0 || !c->prof) return;
  cudaEventRecord(c->prof_recs[handle].b, s);
}
}  // namespace ld

// ---------------------------------------------------------------- CUDA graphs
// Launch-latency-bound configurations (small models: ~20 dependent kernels of a few us each) replay
// a captured graph of a call's kernels instead of launching them one by one.  A graph is keyed by
// the call kind, its buffer addresses and the host-side state its launch sequence depends on, and
// is rebuilt when a scratch buffer it baked in is reallocated (scratch_gen).  At most 8 are kept.
template <class F>
static lowdiff_status run_graphed(lowdiff_ctx* c, int kind, const void* a, const void* b, const void* d, int flag,
                                  cudaStream_t s, F&& body) {
  for (auto& g : c->graphs) {
    if (g.kind == kind && g.a == a && g.b == b && g.c == d && g.flag == flag && g.gen == c->scratch_gen) {
      g.last_use = ++c->graph_tick;
      CK(cudaGraphLaunch(g.exec, s));
      c->launches += g.launches;
      return LOWDIFF_OK;
    }
  }
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  const int64_t l0 = c->launches;
  CK(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
  cudaError_t e = body(c->cap_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(c->cap_stream, &graph);
  const int64_t n = c->launches - l0;
  c->launches = l0;
  if (e == cudaSuccess) e = e2;
  cudaGraphExec_t exec = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(c, e, "graph capture");
  // drop graphs of stale scratch, then the least recently used beyond 8
  for (size_t i = 0; i < c->graphs.size();) {
    if (c->graphs[i].gen != c->scratch_gen) {
      cudaGraphExecDestroy(c->graphs[i].exec);
      c->graphs.erase(c->graphs.begin() + (long)i);
    } else {
      ++i;
    }
  }
  if (c->graphs.size() >= 8) {
    auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                [](const ld::GraphEntry& x, const ld::GraphEntry& y) { return x.last_use < y.last_use; });
    cudaGraphExecDestroy(lru->exec);
    c->graphs.erase(lru);
  }
  c->graphs.push_back(ld::GraphEntry{kind, a, b, d, flag, c->scratch_gen, exec, n, ++c->graph_tick});
  CK(cudaGraphLaunch(exec, s));
  c->launches += n;
  return LOWDIFF_OK;
}

extern "C" {

int32_t lowdiff_abi_version(void) { return 1; }

lowdiff_status lowdiff_selftest(int32_t which, uint64_t n, uint64_t seed, uint64_t* mismatches, uint64_t* first_bad) {
  if (!mismatches || !first_bad || which < 0 || which > 3) return LOWDIFF_E_INVALID;
  return ld::run_selftest(which, n, seed, mismatches, first_bad) == cudaSuccess ? LOWDIFF_OK : LOWDIFF_E_CUDA;
}

lowdiff_status lowdiff_nccl_unique_id(void* out128) {
  if (!out128) return LOWDIFF_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return LOWDIFF_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_derive_step_scalars(int64_t t, double lr, double beta1, double beta2,
                                           lowdiff_step_scalars* out) {
  if (!out || t < 1) return LOWDIFF_E_INVALID;
  double b1t = 1.0, b2t = 1.0;   // beta^t by t repeated double products (R-11)
  for (int64_t i = 0; i < t; ++i) { b1t *= beta1; b2t *= beta2; }
  out->lr = (float)lr;
  out->bc1_inv = (float)(1.0 / (1.0 - b1t));
  out->bc2_inv = (float)(1.0 / (1.0 - b2t));
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_derive_adam_consts(double beta1, double beta2, double eps, lowdiff_adam_consts* out) {
  if (!out) return LOWDIFF_E_INVALID;
  out->beta1 = (float)beta1;
  out->one_minus_beta1 = (float)(1.0 - beta1);
  out->beta2 = (float)beta2;
  out->one_minus_beta2 = (float)(1.0 - beta2);
  out->eps = (float)eps;
  return LOWDIFF_OK;
}

uint32_t lowdiff_crc32c(const void* data, size_t len) {
  return ld::crc32c_update(0xFFFFFFFFu, data, len) ^ 0xFFFFFFFFu;
}

static lowdiff_status validate_cfg(const lowdiff_config* cfg) {
  if (!cfg || cfg->n_layers <= 0 || !cfg->numel) return LOWDIFF_E_INVALID;
  if (cfg->density_ppm < 1 || cfg->density_ppm > 1000000) return LOWDIFF_E_INVALID;
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return LOWDIFF_E_INVALID;
  if (cfg->optim != LOWDIFF_SGD && cfg->optim != LOWDIFF_ADAM) return LOWDIFF_E_INVALID;
  uint64_t psi = 0;
  for (int l = 0; l < cfg->n_layers; ++l) {
    if (cfg->numel[l] <= 0) return LOWDIFF_E_DIM;
    psi += (uint64_t)cfg->numel[l];
  }
  if (psi >= (1ull << 32)) return LOWDIFF_E_DIM;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_create(const lowdiff_config* cfg, lowdiff_ctx** out) {
  if (!out) return LOWDIFF_E_INVALID;
  *out = nullptr;
  lowdiff_status st = validate_cfg(cfg);
  if (st) return st;
  lowdiff_ctx* c = new lowdiff_ctx();
  c->cfg = *cfg;
  c->numel.assign(cfg->numel, cfg->numel + cfg->n_layers);
  c->cfg.numel = c->numel.data();
  c->cfg.nccl_unique_id = nullptr;
  if (cfg->ckpt_dir) c->ckpt_dir = cfg->ckpt_dir;
  c->cfg.ckpt_dir = cfg->ckpt_dir ? c->ckpt_dir.c_str() : nullptr;
  c->device = cfg->device;
  c->b = std::max(1, cfg->batch_size);
  c->R = cfg->ring_slots > 0 ? std::max(cfg->ring_slots, c->b) : 2 * c->b;
  auto bail = [&](lowdiff_status s) { lowdiff_destroy(c); return s; };
  if ((st = entry(c))) return bail(st);
  if ((st = build_plan(c))) return bail(st);
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_tmp, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_side_all, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->last_d2h, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->full_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->full_staged, cudaEventDisableTiming) != cudaSuccess)
    return bail(LOWDIFF_E_CUDA);
  for (int i = 0; i < 2; ++i)
    if (cudaEventCreateWithFlags(&c->snap_done[i], cudaEventDisableTiming) != cudaSuccess) return bail(LOWDIFF_E_CUDA);
  if (cfg->world > 1 && cfg->nccl_unique_id) {   // no id: recovery / merge-only context
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_unique_id, sizeof id);
    if (ncclCommInitRank(&c->comm, cfg->world, id, cfg->rank) != ncclSuccess) return bail(LOWDIFF_E_NCCL);
  }
  // pinned ring: R slots of (32-byte block header + 8K payload), 4 KiB aligned
  c->slot_bytes = ((32 + 8 * (size_t)c->K) + 4095) & ~(size_t)4095;
  if (cudaHostAlloc((void**)&c->ring, c->slot_bytes * c->R, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&c->err_pinned, sizeof(uint32_t) * 2 * c->R, cudaHostAllocDefault) != cudaSuccess)
    return bail(LOWDIFF_E_CUDA);
  std::memset(c->err_pinned, 0, sizeof(uint32_t) * 2 * c->R);
  c->slots.resize(c->R);
  for (int s = 0; s < c->R; ++s) {
    c->slots[s].host = c->ring + s * c->slot_bytes;
    c->slots[s].err_host = c->err_pinned + 2 * s;
    if (cudaEventCreateWithFlags(&c->slots[s].done, cudaEventDisableTiming) != cudaSuccess) return bail(LOWDIFF_E_CUDA);
    c->free_slots.push_back(s);
  }
  ld::build_prefix(c->cfg, c->numel, c->psi, c->K, c->prefix);
  if (c->cfg.ckpt_dir && c->cfg.write_files) ::mkdir(c->cfg.ckpt_dir, 0755);
  c->writer = std::thread(writer_loop, c);
  *out = c;
  return LOWDIFF_OK;
}

static void union_drain(lowdiff_ctx* c);
static void union_shutdown(lowdiff_ctx* c);

lowdiff_status lowdiff_sync(lowdiff_ctx* c) {
  lowdiff_status st = entry(c);
  if (st) return st;
  {
    std::unique_lock<std::mutex> lk(c->mu);
    c->flush_req = true;
    c->cv_work.notify_all();
    c->cv_idle.wait(lk, [&] { return c->queued.empty() && !c->flush_req && !c->writer_busy; });
  }
  if (c->full_writer.joinable()) c->full_writer.join();
  union_drain(c);
  CK(cudaStreamSynchronize(c->side));
  uint32_t err[2];
  CK(cudaMemcpy(err, c->plan.err, 8, cudaMemcpyDeviceToHost));
  lowdiff_status d = take_deferred(c);
  if (d) return d;
  if (c->peer_flags) {
    unsigned long long pe = 0;
    CK(cudaMemcpy(&pe, c->peer_flags + ld::peer_err_word(c->peer_slots), 8, cudaMemcpyDeviceToHost));
    if (pe) {
      CK(cudaMemset(c->peer_flags + ld::peer_err_word(c->peer_slots), 0, 8));
      return fail(c, LOWDIFF_E_STATE, "peer exchange: a wait for another rank timed out (protocol misuse)");
    }
  }
  if (err[0] > c->err_seen.load()) {
    // the device keeps a monotone counter of non-finite events; report only new ones
    c->err_seen = err[0];
    return fail(c, LOWDIFF_E_NUMERIC, "non-finite accumulated gradient (first layer " + std::to_string(err[1]) + ")");
  }
  return LOWDIFF_OK;
}

static void replica_drain(lowdiff_ctx* c);
static void replica_shutdown(lowdiff_ctx* c);

lowdiff_status lowdiff_destroy(lowdiff_ctx* c) {
  if (!c) return LOWDIFF_OK;
  lowdiff_status st = LOWDIFF_OK;
  if (c->writer.joinable()) {
    if (c->poisoned == LOWDIFF_OK) st = lowdiff_sync(c);
    {
      std::lock_guard<std::mutex> g(c->mu);
      c->stop = true;
      c->cv_work.notify_all();
    }
    c->writer.join();
  }
  if (c->full_writer.joinable()) c->full_writer.join();
  replica_drain(c);
  replica_shutdown(c);
  union_drain(c);
  union_shutdown(c);
  cudaSetDevice(c->device);
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->rep_host) cudaFreeHost(c->rep_host);
  if (c->rep_init_done) cudaEventDestroy(c->rep_init_done);
  if (c->comm) ncclCommDestroy(c->comm);
  for (auto& s : c->slots) if (s.done) cudaEventDestroy(s.done);
  for (auto e : c->prof_pool) cudaEventDestroy(e);
  if (c->ring) cudaFreeHost(c->ring);
  if (c->err_pinned) cudaFreeHost(c->err_pinned);
  if (c->full_host) cudaFreeHost(c->full_host);
  for (auto* p : c->snap_host) if (p) cudaFreeHost(p);
  for (auto* p : c->dev_allocs) cudaFree(p);
  if (c->replay_scratch) cudaFree(c->replay_scratch);
  if (c->merge_scratch) cudaFree(c->merge_scratch);
  if (c->full_stage) cudaFree(c->full_stage);
  for (void* q : c->peer_opened) cudaIpcCloseMemHandle(q);
  for (uint32_t* q : c->peer_own) cudaFree(q);
  if (c->peer_flags) cudaFree(c->peer_flags);
  for (auto e : {c->ev_tmp, c->ev_side_all, c->last_d2h, c->full_done, c->full_staged, c->snap_done[0], c->snap_done[1]})
    if (e) cudaEventDestroy(e);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  for (auto* b : c->stage.bufs) cudaFreeHost(b);
  for (auto st : c->stage.streams) cudaStreamDestroy(st);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
  return st;
}

lowdiff_status lowdiff_query(const lowdiff_ctx* c, int64_t* psi, int64_t* k_tot) {
  if (!c) return LOWDIFF_E_INVALID;
  if (psi) *psi = c->psi;
  if (k_tot) *k_tot = c->K;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_layer_k(const lowdiff_ctx* c, int32_t layer, int64_t* k, int64_t* koff) {
  if (!c || layer < 0 || layer >= c->cfg.n_layers) return LOWDIFF_E_INVALID;
  if (k) *k = c->k[layer];
  if (koff) *koff = (int64_t)c->koff[layer];
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_set_graphs(lowdiff_ctx* c, int32_t enable) {
  lowdiff_status st = entry(c);
  if (st) return st;
  c->use_graphs = enable != 0;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_compress(lowdiff_ctx* c, const float* grad, float* residual, uint32_t* send, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!grad || !send || (c->cfg.error_feedback && !residual)) return fail(c, LOWDIFF_E_INVALID, "compress: NULL buffer");
  // grad/residual are streamed with 128-bit accesses; the send block only needs 4-byte alignment
  if (!aligned16(grad) || (reinterpret_cast<uintptr_t>(send) & 3u) || (residual && !aligned16(residual)))
    return fail(c, LOWDIFF_E_INVALID, "compress: buffers must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (auto& ps : c->d2h_src)   // WAR: a persist of this buffer may still be copying it out
    if (ps.first == send) CK(cudaStreamWaitEvent(s, c->slots[ps.second].done, 0));
  int pslot = -1;                // a peer-exchange slot (NEXT-1)?
  for (int i = 0; i < c->peer_slots; ++i)
    if (c->peer_own[i] == send) pslot = i;
  if (pslot >= 0 && c->peer_set && c->peer_epoch[pslot] > 0)   // WAR: every rank has read the old block
    CK(ld::launch_peer_wait_done(c->peer_flags, c->peer_slots, pslot, c->cfg.world, c->peer_epoch[pslot], s));
  float* res = c->cfg.error_feedback ? residual : nullptr;
  if (c->use_graphs && !c->prof) {
    const int lazy = (res && c->lazy_residual == res) ? 1 : 0;   // the only host state the sequence reads
    // (measured: the refill levels as conditional IF nodes set by a flag kernel were slower than
    // replaying their empty grids -- ResNet-50 174 -> 188 us per step -- so the graph is a plain capture)
    if ((st = run_graphed(c, 0, grad, res, send, lazy, s,
                          [&](cudaStream_t cs) { return ld::launch_compress(c, grad, res, send, cs); })))
      return st;
    c->lazy_residual = res;   // what launch_compress records for a replayed call too
  } else {
    CK(ld::launch_compress(c, grad, res, send, s));
  }
  if (pslot >= 0) {              // publish: the block's merge tile starts, then its ready flag
    CK(ld::launch_tile_start(send, (uint64_t)c->K, c->psi, send + 2 * c->K, s));
    c->peer_epoch[pslot] += 1;
    CK(ld::launch_peer_ready(c->peer_flags, pslot, c->peer_epoch[pslot], s));
    c->launches += 2;
  }
  return LOWDIFF_OK;
}

// ---------------------------------------------------------------- peer-memory exchange (NEXT-1)
lowdiff_status lowdiff_peer_alloc(lowdiff_ctx* c, int32_t n_slots, uint32_t** slots_out, void** flags_out,
                                  void* handles_out) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (n_slots < 1 || n_slots > 4 || !slots_out || c->cfg.world > ld::kPeerMaxWorld)
    return fail(c, LOWDIFF_E_INVALID, "peer_alloc: bad argument (1..4 slots, world <= 8)");
  if (c->peer_slots) return fail(c, LOWDIFF_E_STATE, "peer_alloc: already allocated");
  const int64_t n_tiles = (c->psi + ld::kMergeTile - 1) / ld::kMergeTile;
  for (int i = 0; i < n_slots; ++i) {
    void* b = nullptr;
    CK(cudaMalloc(&b, (2 * (size_t)c->K + (size_t)n_tiles + 1) * 4));
    c->peer_own.push_back(static_cast<uint32_t*>(b));
  }
  const size_t fbytes = (size_t)(ld::peer_err_word(n_slots) + 1) * 8;
  CK(cudaMalloc((void**)&c->peer_flags, fbytes));
  CK(cudaMemset(c->peer_flags, 0, fbytes));
  c->peer_slots = n_slots;
  c->peer_epoch.assign(n_slots, 0);
  uint8_t* h = static_cast<uint8_t*>(handles_out);
  for (int i = 0; i < n_slots; ++i) {
    slots_out[i] = c->peer_own[i];
    if (h) CK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(h + 64 * i), c->peer_own[i]));
  }
  if (h) CK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(h + 64 * n_slots), c->peer_flags));
  if (flags_out) *flags_out = c->peer_flags;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_ipc_open(lowdiff_ctx* c, const void* handle64, void** ptr) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!handle64 || !ptr) return fail(c, LOWDIFF_E_INVALID, "ipc_open: NULL argument");
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, sizeof hd);
  CK(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess));
  c->peer_opened.push_back(*ptr);
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_peer_set(lowdiff_ctx* c, const void* const* ptrs) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->peer_slots || !ptrs) return fail(c, LOWDIFF_E_STATE, "peer_set: call lowdiff_peer_alloc first");
  const int n = c->peer_slots, W = c->cfg.world;
  for (int q = 0; q < W; ++q)
    for (int i = 0; i <= n; ++i)
      if (!ptrs[q * (n + 1) + i]) return fail(c, LOWDIFF_E_INVALID, "peer_set: NULL pointer");
  for (int i = 0; i < n; ++i)
    if (ptrs[c->cfg.rank * (n + 1) + i] != c->peer_own[i])
      return fail(c, LOWDIFF_E_INVALID, "peer_set: own entries must be this context's slots");
  if (ptrs[c->cfg.rank * (n + 1) + n] != c->peer_flags)
    return fail(c, LOWDIFF_E_INVALID, "peer_set: own flag entry must be this context's flags");
  c->peer_ptrs.assign(ptrs, ptrs + (size_t)W * (n + 1));
  c->peer_set = true;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_exchange_peer(lowdiff_ctx* c, int32_t slot, float* dense_out, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->peer_set) return fail(c, LOWDIFF_E_STATE, "exchange_peer: call lowdiff_peer_set first");
  if (slot < 0 || slot >= c->peer_slots || !dense_out || !aligned16(dense_out))
    return fail(c, LOWDIFF_E_INVALID, "exchange_peer: bad argument");
  if (!c->peer_epoch[slot]) return fail(c, LOWDIFF_E_STATE, "exchange_peer: nothing was compressed into the slot");
  const int n = c->peer_slots;
  ld::PeerTable T{};
  T.world = c->cfg.world;
  T.self = c->cfg.rank;
  T.slot = slot;
  T.n_slots = n;
  T.epoch = c->peer_epoch[slot];
  for (int q = 0; q < T.world; ++q) {
    T.send[q] = static_cast<const uint32_t*>(c->peer_ptrs[q * (n + 1) + slot]);
    T.start[q] = T.send[q] + 2 * c->K;
    T.flags[q] = const_cast<unsigned long long*>(static_cast<const unsigned long long*>(c->peer_ptrs[q * (n + 1) + n]));
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int h;
  ld::prof_begin(c, "peer_merge", s, &h);
  cudaError_t e = ld::launch_peer_merge(T, (uint64_t)c->K, c->psi, c->cfg.mean != 0, dense_out, s);
  ld::prof_end(c, h, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "peer_merge");
  c->launches += 2;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_residual_materialize(lowdiff_ctx* c, float* residual, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!residual || !aligned16(residual)) return fail(c, LOWDIFF_E_INVALID, "residual_materialize: bad buffer");
  CK(ld::launch_materialize(c, residual, static_cast<cudaStream_t>(stream)));
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_merge(lowdiff_ctx* c, int32_t world, const uint32_t* gathered, float* dense_out, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (world < 1 || !gathered || !dense_out) return fail(c, LOWDIFF_E_INVALID, "merge: bad argument");
  if ((reinterpret_cast<uintptr_t>(gathered) & 3u) || !aligned16(dense_out))
    return fail(c, LOWDIFF_E_INVALID, "merge: gathered must be 4-byte and dense_out 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->use_graphs && !c->prof) {
    // size the scratch outside the capture (its pointer is baked into the graph)
    if (c->merge_scratch_bytes < ld::merge_scratch_bytes(c->psi, world, world)) CK(ld::launch_merge(c, world, gathered, dense_out, s));
    else return run_graphed(c, 1, gathered, dense_out, nullptr, world, s,
                            [&](cudaStream_t cs) { return ld::launch_merge(c, world, gathered, dense_out, cs); });
    return LOWDIFF_OK;
  }
  CK(ld::launch_merge(c, world, gathered, dense_out, s));
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_exchange(lowdiff_ctx* c, const uint32_t* send, uint32_t* gathered, float* dense_out,
                                void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!send || !dense_out || (c->cfg.world > 1 && !gathered)) return fail(c, LOWDIFF_E_INVALID, "exchange: NULL buffer");
  const size_t blk = 2 * (size_t)c->K;
  if (c->cfg.world > 1) {
    if (!c->comm) return fail(c, LOWDIFF_E_STATE, "exchange: context was created without an NCCL id");
    int h;
    ld::prof_begin(c, "allgather", s, &h);
    ncclResult_t r = ncclAllGather(send, gathered, blk, ncclUint32, c->comm, s);
    ld::prof_end(c, h, s);
    if (r != ncclSuccess) return fail(c, LOWDIFF_E_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return lowdiff_merge(c, c->cfg.world, gathered, dense_out, stream);
  }
  if (gathered && gathered != send) CK(cudaMemcpyAsync(gathered, send, blk * 4, cudaMemcpyDeviceToDevice, s));
  return lowdiff_merge(c, 1, send, dense_out, stream);
}

// SURVEY NEXT-1 (second half): the live optimizer step straight from the gathered blocks -- the
// fused replay with n = 1 -- so the dense G is never materialised in HBM (24 B/param + 8 N K instead
// of 4 B/param for the merge plus 28 B/param for a dense Adam step).
lowdiff_status lowdiff_exchange_update(lowdiff_ctx* c, const uint32_t* send, uint32_t* gathered,
                                       const lowdiff_step_scalars* scalars, float* p, float* m, float* v,
                                       void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!send || !scalars || (c->cfg.world > 1 && !gathered)) return fail(c, LOWDIFF_E_INVALID, "exchange_update: NULL buffer");
  const size_t blk = 2 * (size_t)c->K;
  const uint32_t* blocks = send;
  if (c->cfg.world > 1) {
    if (!c->comm) return fail(c, LOWDIFF_E_STATE, "exchange_update: context was created without an NCCL id");
    int h;
    ld::prof_begin(c, "allgather", s, &h);
    ncclResult_t r = ncclAllGather(send, gathered, blk, ncclUint32, c->comm, s);
    ld::prof_end(c, h, s);
    if (r != ncclSuccess) return fail(c, LOWDIFF_E_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    blocks = gathered;
  }
  if (!p || (c->cfg.optim == LOWDIFF_ADAM && (!m || !v)) || !aligned16(p) || (m && !aligned16(m)) ||
      (v && !aligned16(v)))
    return fail(c, LOWDIFF_E_INVALID, "exchange_update: p, m, v must be 16-byte aligned device arrays");
  cudaError_t e = ld::launch_update(c, c->cfg.world, blocks, *scalars, p, m, v, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "launch_update");
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_batch_persist(lowdiff_ctx* c, int64_t iteration, const lowdiff_step_scalars* scalars,
                                     const uint32_t* send, void* producer) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!scalars || !send) return fail(c, LOWDIFF_E_INVALID, "batch_persist: NULL argument");
  if (c->next_iter >= 0 && iteration != c->next_iter)
    return fail(c, LOWDIFF_E_STATE, "batch_persist: iteration " + std::to_string(iteration) + " after " +
                                        std::to_string(c->next_iter - 1) + " (must be consecutive)");
  int slot;
  {
    std::unique_lock<std::mutex> lk(c->mu);
    if (c->free_slots.empty()) {
      const int64_t t0 = now_ns();
      c->cv_free.wait(lk, [&] { return !c->free_slots.empty(); });
      c->stall_ns += now_ns() - t0;
    }
    slot = c->free_slots.front();
    c->free_slots.pop_front();
  }
  c->next_iter = iteration + 1;
  ld::Slot& S = c->slots[slot];
  S.iteration = iteration;
  uint8_t* h = S.host;                          // 32-byte block header
  std::memset(h, 0, 32);
  const uint64_t it = (uint64_t)iteration;
  std::memcpy(h, &it, 8);
  std::memcpy(h + 8, &scalars->lr, 4);
  std::memcpy(h + 12, &scalars->bc1_inv, 4);
  std::memcpy(h + 16, &scalars->bc2_inv, 4);
  cudaStream_t p = static_cast<cudaStream_t>(producer);
  int hnd;
  CK(cudaEventRecord(c->ev_tmp, p));
  CK(cudaStreamWaitEvent(c->side, c->ev_tmp, 0));
  ld::prof_begin(c, "d2h", c->side, &hnd);
  CK(cudaMemcpyAsync(h + 32, send, 8 * (size_t)c->K, cudaMemcpyDeviceToHost, c->side));
  ld::prof_end(c, hnd, c->side);
  CK(cudaMemcpyAsync(S.err_host, c->plan.err, 8, cudaMemcpyDeviceToHost, c->side));
  CK(cudaEventRecord(S.done, c->side));
  // remember the latest slot copying `send` (its event orders after every earlier copy: one side stream)
  bool found = false;
  for (auto& ps : c->d2h_src)
    if (ps.first == send) { ps.second = slot; found = true; }
  if (!found) {
    if (c->d2h_src.size() >= 64) {   // many distinct send buffers: drain instead of tracking them all
      CK(cudaStreamSynchronize(c->side));
      c->d2h_src.clear();
    }
    c->d2h_src.push_back({send, slot});
  }
  {
    std::lock_guard<std::mutex> g(c->mu);
    c->queued.push_back(slot);
    c->cv_work.notify_all();
  }
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_wait_persist(lowdiff_ctx* c, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  CK(cudaEventRecord(c->ev_side_all, c->side));
  CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), c->ev_side_all, 0));
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_full_ckpt(lowdiff_ctx* c, int64_t iteration, const float* p, const float* m, const float* v,
                                 void* producer) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!p || iteration < 0) return fail(c, LOWDIFF_E_INVALID, "full_ckpt: bad argument");
  if (c->full_writer.joinable()) c->full_writer.join();   // one full checkpoint in flight
  const uint64_t sb = (uint64_t)c->psi * c->cfg.rank / c->cfg.world;
  const uint64_t se = (uint64_t)c->psi * (c->cfg.rank + 1) / c->cfg.world;
  const size_t S = se - sb;
  if (c->full_cap < 3 * S) {
    if (c->full_host) cudaFreeHost(c->full_host);
    c->full_host = nullptr;
    c->full_cap = 0;
    CK(cudaHostAlloc((void**)&c->full_host, std::max<size_t>(1, 3 * S) * 4, cudaHostAllocDefault));
    c->full_cap = 3 * S;
  }
  cudaStream_t pr = static_cast<cudaStream_t>(producer);
  CK(cudaEventRecord(c->ev_tmp, pr));
  CK(cudaStreamWaitEvent(c->side, c->ev_tmp, 0));
  const float* src[3] = {p, m, v};
  // D2D stage: the producer's next update waits only for an HBM->HBM copy of the
  // shard (12 S bytes at HBM speed) instead of the PCIe transfer; the D2H then runs from the stage.
  // Without the device memory for the stage, the snapshot goes straight D2H.
  if (c->full_stage_cap < 3 * S) {
    if (c->full_stage) cudaFree(c->full_stage);
  for (void* q : c->peer_opened) cudaIpcCloseMemHandle(q);
  for (uint32_t* q : c->peer_own) cudaFree(q);
  if (c->peer_flags) cudaFree(c->peer_flags);
    c->full_stage = nullptr;
    c->full_stage_cap = 0;
    if (cudaMalloc((void**)&c->full_stage, std::max<size_t>(1, 3 * S) * 4) == cudaSuccess) c->full_stage_cap = 3 * S;
    else { c->full_stage = nullptr; cudaGetLastError(); }
  }
  int h;
  ld::prof_begin(c, "full_snapshot", c->side, &h);
  if (c->full_stage) {
    for (int a = 0; a < 3; ++a) {
      if (src[a]) CK(cudaMemcpyAsync(c->full_stage + a * S, src[a] + sb, S * 4, cudaMemcpyDeviceToDevice, c->side));
      else CK(cudaMemsetAsync(c->full_stage + a * S, 0, S * 4, c->side));
    }
    CK(cudaEventRecord(c->full_staged, c->side));
    CK(cudaStreamWaitEvent(pr, c->full_staged, 0));   // the next update waits for the stage (WAR)
    ld::prof_end(c, h, c->side);
    CK(cudaMemcpyAsync(c->full_host, c->full_stage, 3 * S * 4, cudaMemcpyDeviceToHost, c->side));
    CK(cudaEventRecord(c->full_done, c->side));
  } else {
    for (int a = 0; a < 3; ++a) {
      if (src[a]) CK(cudaMemcpyAsync(c->full_host + a * S, src[a] + sb, S * 4, cudaMemcpyDeviceToHost, c->side));
      else std::memset(c->full_host + a * S, 0, S * 4);
    }
    CK(cudaEventRecord(c->full_done, c->side));
    CK(cudaStreamWaitEvent(pr, c->full_done, 0));   // the next update waits for the snapshot (WAR)
    ld::prof_end(c, h, c->side);
  }
  if (!c->cfg.ckpt_dir || !c->cfg.write_files) return LOWDIFF_OK;
  c->full_writer = std::thread([c, iteration, sb, se, S]() {
    cudaSetDevice(c->device);
    cudaError_t e = cudaEventSynchronize(c->full_done);
    if (e != cudaSuccess) { set_deferred(c, LOWDIFF_E_CUDA, cudaGetErrorString(e)); return; }
    const int64_t t0 = now_ns();
    std::string err;
    lowdiff_status s2 = write_ldf(c->cfg, c->ckpt_dir, iteration, (uint64_t)c->psi, sb, se, c->full_host, &err);
    if (s2) set_deferred(c, s2, err);
    else { c->files_written += 1; c->bytes_written += (int64_t)(100 + 12 * S); }
    c->writer_ns += now_ns() - t0;
  });
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_replay_range(lowdiff_ctx* c, int32_t optim, int32_t world, int64_t n_steps,
                                    const uint32_t* diffs, const lowdiff_step_scalars* scalars, int64_t begin,
                                    int64_t end, float* p, float* m, float* v, void* stream) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (begin >= 0 && begin == end && end <= c->psi && n_steps >= 0) return LOWDIFF_OK;   // empty range
  if (world < 1 || n_steps < 0 || (n_steps && (!diffs || !scalars)) || !p ||
      (optim == LOWDIFF_ADAM && (!m || !v)) || (optim != LOWDIFF_ADAM && optim != LOWDIFF_SGD) || begin < 0 ||
      end > c->psi || begin > end)
    return fail(c, LOWDIFF_E_INVALID, "replay: bad argument");
  if (!n_steps || begin == end) return LOWDIFF_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // per-step scalars to the device (tail of the replay scratch is not reused: own buffer)
  float* scal_dev = nullptr;
  CK(cudaMallocAsync((void**)&scal_dev, (size_t)n_steps * 12, s));
  CK(cudaMemcpyAsync(scal_dev, scalars, (size_t)n_steps * 12, cudaMemcpyHostToDevice, s));
  const float consts[5] = {c->cfg.adam.beta1, c->cfg.adam.one_minus_beta1, c->cfg.adam.beta2,
                           c->cfg.adam.one_minus_beta2, c->cfg.adam.eps};
  cudaError_t e = ld::launch_replay(c, optim, c->cfg.mean != 0, consts, world, n_steps, diffs, scal_dev,
                                    (uint64_t)begin, (uint64_t)end, nullptr, p, m, v, s);
  cudaFreeAsync(scal_dev, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "launch_replay");
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_replay(lowdiff_ctx* c, int32_t optim, int32_t world, int64_t n_steps, const uint32_t* diffs,
                              const lowdiff_step_scalars* scalars, float* p, float* m, float* v, void* stream) {
  if (!c) return LOWDIFF_E_INVALID;
  return lowdiff_replay_range(c, optim, world, n_steps, diffs, scalars, 0, c->psi, p, m, v, stream);
}

lowdiff_status lowdiff_chain_scan(const lowdiff_config* cfg, int64_t target, int64_t* full_iter, int64_t* last_iter) {
  if (validate_cfg(cfg) || !cfg->ckpt_dir) return LOWDIFF_E_INVALID;
  Chain ch;
  std::string err;
  lowdiff_status st = scan_chain(*cfg, target, &ch, &err);
  if (st) return st;
  if (full_iter) *full_iter = ch.F;
  if (last_iter) *last_iter = ch.last;
  return LOWDIFF_OK;
}

// Every rank's shard [floor(q Psi / N), floor((q+1) Psi / N)) of each non-NULL dst array, broadcast
// from its owner q (uneven shard sizes: one broadcast per owner, grouped).
static lowdiff_status bcast_shards(lowdiff_ctx* c, float* dst[3], cudaStream_t s) {
  ncclResult_t r = ncclGroupStart();
  const uint64_t psi = (uint64_t)c->psi, W = (uint64_t)c->cfg.world;
  for (int a = 0; a < 3 && r == ncclSuccess; ++a) {
    if (!dst[a]) continue;
    for (uint64_t q = 0; q < W && r == ncclSuccess; ++q) {
      const uint64_t qb = psi * q / W, qe = psi * (q + 1) / W;
      r = ncclBroadcast(dst[a] + qb, dst[a] + qb, qe - qb, ncclFloat, (int)q, c->comm, s);
    }
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return fail(c, LOWDIFF_E_NCCL, std::string("shard broadcast: ") + ncclGetErrorString(r));
  return LOWDIFF_OK;
}

// Full checkpoint F -> p, m, v (every shard, or only this rank's when sharded): size, magic, CRC and
// header fields verified (else E_CORRUPT); optim, Adam constants and flags from the file.
static lowdiff_status load_full_shards(lowdiff_ctx* c, const std::vector<std::string>& paths, int64_t F, bool sharded,
                                       float* p, float* m, float* v, uint32_t* optim, float* consts, uint16_t* flags) {
  const uint32_t world = (uint32_t)c->cfg.world;
  const uint64_t psi = (uint64_t)c->psi;
  for (uint32_t r = sharded ? (uint32_t)c->cfg.rank : 0; r < (sharded ? (uint32_t)c->cfg.rank + 1 : world); ++r) {
    const uint64_t sb = psi * r / world, se = psi * (r + 1) / world, S = se - sb;
    const std::string& path = paths[r];
    int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd < 0) return fail(c, LOWDIFF_E_IO, "cannot read " + path);
    struct stat stt;
    uint8_t h[96];
    uint32_t trailer = 0;
    const bool ok = fstat(fd, &stt) == 0 && (uint64_t)stt.st_size == 100 + 12 * S &&
                    ::pread(fd, h, 96, 0) == 96 && ::pread(fd, &trailer, 4, (off_t)(96 + 12 * S)) == 4 &&
                    std::memcmp(h, "LDF1", 4) == 0 && rd<uint32_t>(h + 8) == r && rd<uint32_t>(h + 12) == world &&
                    (int64_t)rd<uint64_t>(h + 16) == F && rd<uint64_t>(h + 24) == psi &&
                    rd<uint64_t>(h + 32) == sb && rd<uint64_t>(h + 40) == se;
    if (!ok) {
      ::close(fd);
      return fail(c, LOWDIFF_E_CORRUPT, "corrupt full checkpoint " + path);
    }
    *optim = rd<uint32_t>(h + 48);
    *flags = rd<uint16_t>(h + 6);
    std::memcpy(consts, h + 64, 20);
    // body p | m | v streamed to the device through pinned chunks (read, CRC and H2D overlapped)
    uint32_t crc_body = 0;
    std::string err;
    lowdiff_status st2 = ld::stream_to_device(fd, 96, {{p + sb, 4 * S}, {m ? m + sb : nullptr, 4 * S},
                                                       {v ? v + sb : nullptr, 4 * S}}, c->stage, &crc_body, &err);
    ::close(fd);
    if (st2) return fail(c, st2, err + " (" + path + ")");
    const uint32_t crc = ld::crc32c_combine(lowdiff_crc32c(h, 96), crc_body, 12 * S);
    if (crc != trailer) return fail(c, LOWDIFF_E_CORRUPT, "corrupt full checkpoint " + path + " (CRC)");
  }
  if (*optim == LOWDIFF_ADAM && (!m || !v)) return fail(c, LOWDIFF_E_INVALID, "recover: Adam needs m and v");
  return LOWDIFF_OK;
}

// Differential blocks of steps [t0, t1] of every rank into d_diffs (block of (t, r) at
// ((t - t0) world + r) 2K), file by file: header fields and block headers read with small preads
// (scalars kept, ranks must agree), then the whole file streamed through pinned chunks by parallel
// readers (payloads of the wanted blocks copied H2D, everything checksummed; ld::stream_to_device)
// and its CRC-32C checked against the trailer.
static lowdiff_status load_blocks_streamed(lowdiff_ctx* c, const Chain& ch, int64_t t0, int64_t t1, uint32_t optim,
                                           uint32_t* d_diffs, std::vector<lowdiff_step_scalars>& scal) {
  const uint32_t world = (uint32_t)c->cfg.world;
  const uint64_t psi = (uint64_t)c->psi, K = (uint64_t)c->K, L = (uint64_t)c->cfg.n_layers;
  const size_t pre = 96 + 16 * L, blk = 32 + 8 * K;
  std::vector<char> have((size_t)(t1 - t0 + 1) * world, 0);
  for (uint32_t r = 0; r < world; ++r) {
    std::map<std::string, bool> files;   // the files holding this rank's blocks of [t0, t1]
    for (int64_t t = t0; t <= t1; ++t) files[ch.where[r].at(t).first] = true;
    for (auto& fe : files) {
      const std::string& path = fe.first;
      int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
      if (fd < 0) return fail(c, LOWDIFF_E_IO, "cannot read " + path);
      struct stat stt;
      uint8_t h[64];
      bool ok = fstat(fd, &stt) == 0 && stt.st_size >= (off_t)(pre + 4) && ::pread(fd, h, 64, 0) == 64;
      const uint32_t nit = ok ? rd<uint32_t>(h + 24) : 0;
      ok = ok && (size_t)stt.st_size == pre + (size_t)nit * blk + 4 && std::memcmp(h, "LDB1", 4) == 0 &&
           rd<uint32_t>(h + 8) == r && rd<uint32_t>(h + 12) == world && rd<uint32_t>(h + 28) == (uint32_t)L &&
           rd<uint64_t>(h + 32) == psi && rd<uint64_t>(h + 40) == K && rd<uint32_t>(h + 48) == c->cfg.density_ppm &&
           rd<uint32_t>(h + 52) == optim;
      const int64_t first = ok ? (int64_t)rd<uint64_t>(h + 16) : 0;
      std::vector<std::pair<void*, uint64_t>> segs{{nullptr, (uint64_t)pre}};
      for (uint32_t i = 0; ok && i < nit; ++i) {
        uint8_t bh[32];
        ok = ::pread(fd, bh, 32, (off_t)(pre + i * blk)) == 32 && (int64_t)rd<uint64_t>(bh) == first + i;
        const int64_t t = first + i;
        void* dst = nullptr;
        if (ok && t >= t0 && t <= t1 && ch.where[r].at(t).first == path) {
          lowdiff_step_scalars sc;
          std::memcpy(&sc, bh + 8, 12);
          if (r == 0) scal[t - t0] = sc;
          else if (std::memcmp(&sc, &scal[t - t0], 12) != 0) {
            ::close(fd);
            return fail(c, LOWDIFF_E_CORRUPT, "ranks disagree on the scalars of iteration " + std::to_string(t));
          }
          dst = d_diffs + ((size_t)(t - t0) * world + r) * 2 * K;
          have[(size_t)(t - t0) * world + r] = 1;
        }
        segs.push_back({nullptr, 32});
        segs.push_back({dst, 8 * K});
      }
      uint32_t trailer = 0;
      ok = ok && ::pread(fd, &trailer, 4, stt.st_size - 4) == 4;
      if (!ok) {
        ::close(fd);
        return fail(c, LOWDIFF_E_CORRUPT, "corrupt batch file " + path);
      }
      uint32_t crc = 0;
      std::string err;
      lowdiff_status st = ld::stream_to_device(fd, 0, segs, c->stage, &crc, &err);
      ::close(fd);
      if (st) return fail(c, st, err + " (" + path + ")");
      if (crc != trailer) return fail(c, LOWDIFF_E_CORRUPT, "corrupt batch file " + path + " (CRC)");
    }
  }
  for (char x : have)
    if (!x) return fail(c, LOWDIFF_E_CORRUPT, "a block of the chain is missing from its file");
  return LOWDIFF_OK;
}

// Recovery of elements [lo, hi): lo = 0, hi = Psi loads every full shard and replays everything;
// the sharded form (NEXT-2) loads only this rank's .ldf shard and replays only its element range,
// uploading only the entries of each differential block that fall in it.
static lowdiff_status recover_impl(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int64_t* recovered,
                                   void* stream, bool sharded) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->cfg.ckpt_dir) return fail(c, LOWDIFF_E_INVALID, "recover: no ckpt_dir");
  if (!p) return fail(c, LOWDIFF_E_INVALID, "recover: NULL p");
  if ((st = lowdiff_sync(c))) return st;     // our own pending files first
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Chain ch;
  std::string err;
  if ((st = scan_chain(c->cfg, target, &ch, &err))) return fail(c, st, err);
  const uint32_t world = (uint32_t)c->cfg.world;
  const uint64_t psi = (uint64_t)c->psi, K = (uint64_t)c->K;
  const uint64_t lo = sharded ? psi * (uint64_t)c->cfg.rank / world : 0;
  const uint64_t hi = sharded ? psi * ((uint64_t)c->cfg.rank + 1) / world : psi;
  // 1. full checkpoint shards -> p, m, v
  uint32_t optim = 0;
  float consts[5] = {0, 0, 0, 0, 0};
  uint16_t flags = 0;
  if ((st = load_full_shards(c, ch.full_paths, ch.F, sharded, p, m, v, &optim, consts, &flags))) return st;
  const int64_t n = ch.last - ch.F;
  // 2. stream the differentials through the fused replay in chunks of steps that fit HBM
  const size_t step_bytes = (size_t)world * 8 * K;
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const size_t per_step = step_bytes + ld::replay_scratch_bytes(c->psi, (int)world, 1);
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)(free_b / 2 / std::max<size_t>(1, per_step))));
  uint32_t* d_diffs = nullptr;
  uint32_t* d_ranges = nullptr;
  std::vector<uint32_t> ranges;
  if (n > 0) CK(cudaMalloc(&d_diffs, (size_t)chunk * step_bytes));
  if (n > 0 && sharded) CK(cudaMalloc(&d_ranges, (size_t)chunk * world * 8));
  std::map<std::string, std::vector<uint8_t>> cache;   // verified batch files in use
  lowdiff_status result = LOWDIFF_OK;
  std::vector<lowdiff_step_scalars> scal;
  for (int64_t t0 = ch.F + 1; t0 <= ch.last && result == LOWDIFF_OK; t0 += chunk) {
    const int64_t t1 = std::min<int64_t>(ch.last, t0 + chunk - 1);
    scal.assign((size_t)(t1 - t0 + 1), {0, 0, 0});
    ranges.assign((size_t)(t1 - t0 + 1) * world * 2, 0);
    if (!sharded) result = load_blocks_streamed(c, ch, t0, t1, optim, d_diffs, scal);
    for (int64_t t = t0; sharded && t <= t1 && result == LOWDIFF_OK; ++t) {
      for (uint32_t r = 0; r < world; ++r) {
        const auto& w = ch.where[r][t];
        auto itc = cache.find(w.first);
        if (itc == cache.end()) {
          // drop files no longer needed by this rank (iterations are visited in order)
          for (auto jt = cache.begin(); jt != cache.end();) {
            bool used = false;
            for (uint32_t q = 0; q < world && !used; ++q) {
              auto f = ch.where[q].find(t);
              used = f != ch.where[q].end() && f->second.first == jt->first;
            }
            jt = used ? std::next(jt) : cache.erase(jt);
          }
          std::vector<uint8_t> buf;
          if (!read_all(w.first, buf)) { result = fail(c, LOWDIFF_E_IO, "cannot read " + w.first); break; }
          const uint32_t nit = buf.size() >= 100 ? rd<uint32_t>(buf.data() + 24) : 0;
          const size_t want = 100 + 16 * (size_t)c->cfg.n_layers + (size_t)nit * (32 + 8 * K);
          if (buf.size() != want || std::memcmp(buf.data(), "LDB1", 4) != 0 ||
              lowdiff_crc32c(buf.data(), buf.size() - 4) != rd<uint32_t>(buf.data() + buf.size() - 4) ||
              rd<uint32_t>(buf.data() + 8) != r || rd<uint32_t>(buf.data() + 12) != world ||
              rd<uint32_t>(buf.data() + 28) != (uint32_t)c->cfg.n_layers || rd<uint64_t>(buf.data() + 32) != psi ||
              rd<uint64_t>(buf.data() + 40) != K || rd<uint32_t>(buf.data() + 48) != c->cfg.density_ppm ||
              rd<uint32_t>(buf.data() + 52) != optim) {
            result = fail(c, LOWDIFF_E_CORRUPT, "corrupt batch file " + w.first);
            break;
          }
          itc = cache.emplace(w.first, std::move(buf)).first;
        }
        const uint8_t* blk = itc->second.data() + 96 + 16 * (size_t)c->cfg.n_layers + (size_t)w.second * (32 + 8 * K);
        if ((int64_t)rd<uint64_t>(blk) != t) { result = fail(c, LOWDIFF_E_CORRUPT, "block iteration mismatch"); break; }
        lowdiff_step_scalars sc;
        std::memcpy(&sc, blk + 8, 12);
        if (r == 0) scal[t - t0] = sc;
        else if (std::memcmp(&sc, &scal[t - t0], 12) != 0) {
          result = fail(c, LOWDIFF_E_CORRUPT, "ranks disagree on the scalars of iteration " + std::to_string(t));
          break;
        }
        uint32_t* dst = d_diffs + ((size_t)(t - t0) * world + r) * 2 * K;
        cudaError_t e;
        if (!sharded) {
          e = cudaMemcpy(dst, blk + 32, 8 * K, cudaMemcpyHostToDevice);
        } else {
          // the block's indices ascend: its entries inside [lo, hi) are one contiguous run [a, b)
          // (Psi < 2^32, so lo and hi fit the u32 index type)
          const uint32_t* idx = reinterpret_cast<const uint32_t*>(blk + 32);
          const uint32_t a = (uint32_t)(std::lower_bound(idx, idx + K, (uint32_t)lo) - idx);
          const uint32_t b = (uint32_t)(std::lower_bound(idx, idx + K, (uint32_t)hi) - idx);
          ranges[((size_t)(t - t0) * world + r) * 2] = a;
          ranges[((size_t)(t - t0) * world + r) * 2 + 1] = b;
          e = cudaSuccess;
          if (b > a) e = cudaMemcpy(dst + a, idx + a, (size_t)(b - a) * 4, cudaMemcpyHostToDevice);
          if (e == cudaSuccess && b > a)
            e = cudaMemcpy(dst + K + a, idx + K + a, (size_t)(b - a) * 4, cudaMemcpyHostToDevice);
        }
        if (e != cudaSuccess) { result = cuda_fail(c, e, "H2D differential"); break; }
      }
    }
    if (result) break;
    // per-step scalars to the device, then one fused replay launch for the chunk of steps
    float* scal_dev = nullptr;
    cudaError_t e2 = cudaMalloc((void**)&scal_dev, scal.size() * 12);
    if (e2 == cudaSuccess) e2 = cudaMemcpy(scal_dev, scal.data(), scal.size() * 12, cudaMemcpyHostToDevice);
    if (e2 == cudaSuccess && sharded)
      e2 = cudaMemcpy(d_ranges, ranges.data(), ranges.size() * 4, cudaMemcpyHostToDevice);
    if (e2 == cudaSuccess)
      e2 = ld::launch_replay(c, (int)optim, (flags & 2) != 0, consts, (int)world, t1 - t0 + 1, d_diffs, scal_dev, lo,
                             hi, sharded ? d_ranges : nullptr, p + lo, m ? m + lo : nullptr, v ? v + lo : nullptr, s);
    if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s);
    if (scal_dev) cudaFree(scal_dev);
    if (e2 != cudaSuccess) result = cuda_fail(c, e2, "replay");
  }
  if (d_diffs) cudaFree(d_diffs);
  if (d_ranges) cudaFree(d_ranges);
  if (result) return result;
  CK(cudaStreamSynchronize(s));
  if (recovered) *recovered = ch.last;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_recover(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int64_t* recovered,
                               void* stream) {
  return recover_impl(c, target, p, m, v, recovered, stream, false);
}

lowdiff_status lowdiff_recover_sharded(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int32_t gather,
                                       int64_t* recovered, void* stream) {
  lowdiff_status st = recover_impl(c, target, p, m, v, recovered, stream, true);
  if (st || !gather || c->cfg.world == 1) return st;
  if (!c->comm) return fail(c, LOWDIFF_E_STATE, "recover_sharded: gather needs an NCCL context");
  float* dst[3] = {p, m, v};
  if ((st = bcast_shards(c, dst, static_cast<cudaStream_t>(stream)))) return st;
  CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return LOWDIFF_OK;
}

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

// 80-byte header + hyper (32 B) + layer table (16 B per layer) of a .ldu file
static std::vector<uint8_t> ldu_prefix(const lowdiff_ctx* c, int64_t first, uint32_t n_iters) {
  std::vector<uint8_t> b(112 + 16 * (size_t)c->cfg.n_layers, 0);
  const uint16_t ver = 1, flags = (uint16_t)((c->cfg.error_feedback ? 1 : 0) | (c->cfg.mean ? 2 : 0));
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

static void union_write(lowdiff_ctx* c, std::vector<UBlock>& batch) {
  if (batch.empty()) return;
  if (c->cfg.ckpt_dir) {
    const int64_t t0 = now_ns();
    const std::vector<uint8_t> pre = ldu_prefix(c, batch[0].it, (uint32_t)batch.size());
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
    uint32_t crc = 0xFFFFFFFFu;
    size_t bytes = 4;
    for (auto& q : parts) {
      crc = ld::crc32c_update(crc, q.first, q.second);
      bytes += q.second;
    }
    crc ^= 0xFFFFFFFFu;
    parts.push_back({&crc, 4});
    std::string err;
    lowdiff_status st = ld::write_file_atomic(union_name(c->ckpt_dir, c->cfg.rank, batch[0].it), parts,
                                              c->cfg.fsync != 0, &err);
    if (st) set_deferred(c, st, err);
    else { c->u_files += 1; c->u_bytes += (int64_t)bytes; }
    c->writer_ns += now_ns() - t0;
  }
  batch.clear();
}

static void union_loop(lowdiff_ctx* c) {
  cudaSetDevice(c->device);
  std::vector<UBlock> batch;
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
        union_write(c, batch);   // the chain stops before this iteration
      } else {
        c->u_entries += (int64_t)B.n;
        batch.push_back(std::move(B));
        if ((int)batch.size() == c->b) union_write(c, batch);
      }
    } else if (flush) {
      union_write(c, batch);
      std::lock_guard<std::mutex> g(c->u_mu);
      c->u_flush = false;
    } else {
      union_write(c, batch);
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
static void union_drain(lowdiff_ctx* c) {
  if (!c->u_writer.joinable()) return;
  std::unique_lock<std::mutex> lk(c->u_mu);
  c->u_flush = true;
  c->u_cv.notify_all();
  c->u_cv_idle.wait(lk, [&] { return c->u_q.empty() && !c->u_flush && !c->u_busy; });
}

static void union_shutdown(lowdiff_ctx* c) {
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

lowdiff_status lowdiff_union_persist(lowdiff_ctx* c, int64_t iteration, const lowdiff_step_scalars* scalars,
                                     const uint32_t* gathered, void* producer) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!scalars || !gathered) return fail(c, LOWDIFF_E_INVALID, "union_persist: NULL argument");
  if (c->u_next_iter >= 0 && iteration != c->u_next_iter)
    return fail(c, LOWDIFF_E_STATE, "union_persist: iteration " + std::to_string(iteration) + " after " +
                                        std::to_string(c->u_next_iter - 1) + " (must be consecutive)");
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
    c->u_q.push_back(ld::UJob{iteration, *scalars, buf});
    c->u_cv.notify_all();
  }
  return LOWDIFF_OK;
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
  struct Where { std::string path; size_t off; uint64_t n; };
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
      size_t off = 112 + 16 * L;
      for (uint32_t i = 0; i < n_it; ++i) {
        if (off + 32 > buf.size() - 4 || (int64_t)rd<uint64_t>(buf.data() + off) != fe.first + i)
          return fail(c, LOWDIFF_E_CORRUPT, "corrupt union file " + fe.second);
        const uint64_t n = rd<uint32_t>(buf.data() + off + 20);
        where[r][fe.first + i] = Where{fe.second, off, n};
        off += 32 + 8 * n;
      }
      if (off != buf.size() - 4) return fail(c, LOWDIFF_E_CORRUPT, "corrupt union file " + fe.second);
    }
  }
  int64_t last = F;
  for (;;) {
    const int64_t t = last + 1;
    if (target >= 0 && t > target) break;
    bool all = true;
    for (uint32_t r = r0; r < r1 && all; ++r) all = where[r].count(t) > 0;
    if (!all) break;
    last = t;
  }
  if (target >= 0 && last < target) return fail(c, LOWDIFF_E_GAP, "union chain has a gap after " + std::to_string(last));
  const uint64_t lo = sharded ? psi * c->cfg.rank / world : 0, hi = sharded ? psi * (c->cfg.rank + 1) / world : psi;
  // replay in chunks of steps: block of step t = idx[Kc] | val[Kc], entries [0, U_t) valid
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  std::map<std::string, std::vector<uint8_t>> cache;
  lowdiff_status result = LOWDIFF_OK;
  for (int64_t t0 = F + 1; t0 <= last && result == LOWDIFF_OK;) {
    // grow the chunk while its padded size stays within a quarter of free memory
    uint64_t Kc = 1;
    int64_t t1 = t0;
    for (int64_t t = t0; t <= last; ++t) {
      uint64_t U = 0;
      for (uint32_t r = r0; r < r1; ++r) U += where[r][t].n;
      const uint64_t k2 = std::max<uint64_t>(Kc, U);
      if (t > t0 && (uint64_t)(t - t0 + 1) * 8 * k2 > free_b / 4) break;
      Kc = k2;
      t1 = t;
    }
    const int64_t ns = t1 - t0 + 1;
    std::vector<uint32_t> host((size_t)ns * 2 * Kc, 0u), ranges((size_t)ns * 2, 0u);
    std::vector<lowdiff_step_scalars> scal((size_t)ns);
    for (int64_t t = t0; t <= t1 && result == LOWDIFF_OK; ++t) {
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
        if (r == r0) scal[t - t0] = sc;
        else if (std::memcmp(&sc, &scal[t - t0], 12) != 0) {
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
        uint32_t* dst = host.data() + (size_t)(t - t0) * 2 * Kc;
        std::memcpy(dst + at, idx, 4 * w.n);
        std::memcpy(dst + Kc + at, idx + w.n, 4 * w.n);
        at += w.n;
      }
      ranges[2 * (size_t)(t - t0) + 1] = (uint32_t)at;
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
    t0 = t1 + 1;
  }
  if (result) return result;
  if (recovered) *recovered = last;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_recover_union(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int32_t sharded,
                                     int64_t* recovered, void* stream) {
  return union_recover_impl(c, target, p, m, v, sharded != 0, recovered, stream);
}

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
static void replica_drain(lowdiff_ctx* c) {
  if (!c->rep_active) return;
  {
    std::unique_lock<std::mutex> lk(c->rep_mu);
    c->rep_done_cv.wait(lk, [&] { return c->rep_q.empty() && !c->rep_busy; });
  }
  // the writer is only joined by the worker or here; the worker is idle now
  if (c->rep_writer.joinable()) c->rep_writer.join();
}

static void replica_shutdown(lowdiff_ctx* c) {
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
  if (c->cfg.world > 1 && (st = bcast_shards(c, dst, s))) return st;
  CK(cudaStreamSynchronize(s));
  if (iteration) *iteration = c->rep_iter.load();
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_get_stats(const lowdiff_ctx* c, lowdiff_stats* out) {
  if (!c || !out) return LOWDIFF_E_INVALID;
  out->files_written = c->files_written;
  out->bytes_written = c->bytes_written;
  out->ring_stall_ns = c->stall_ns;
  out->writer_busy_ns = c->writer_ns;
  uint32_t cnt[4] = {0, 0, 0, 0};
  if (cudaMemcpy(cnt, c->plan.counters, 16, cudaMemcpyDeviceToHost) == cudaSuccess) {
    out->spec_hits = cnt[1];
    out->spec_misses = cnt[2];
    out->spec_candidates = cnt[3];
  } else {
    out->spec_hits = out->spec_misses = out->spec_candidates = -1;
  }
  out->replica_busy_ns = c->rep_ns;
  out->replica_stall_ns = c->rep_stall_ns;
  out->union_files_written = c->u_files;
  out->union_bytes_written = c->u_bytes;
  out->union_entries = c->u_entries;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_prof_enable(lowdiff_ctx* c, int32_t enable) {
  if (!c) return LOWDIFF_E_INVALID;
  cudaDeviceSynchronize();
  c->prof_recs.clear();   // the events stay in prof_pool for reuse
  c->prof = enable != 0;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_prof_read(lowdiff_ctx* c, const char* name, double* total_ms, int64_t* launches) {
  lowdiff_status st = entry(c);
  if (st) return st;
  double ms = 0;
  int64_t n = 0;
  for (auto& r : c->prof_recs) {
    if (name && name[0] && std::strcmp(name, r.name) != 0) continue;
    CK(cudaEventSynchronize(r.b));
    float x = 0;
    CK(cudaEventElapsedTime(&x, r.a, r.b));
    ms += x;
    ++n;
  }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = n;
  return LOWDIFF_OK;
}

int64_t lowdiff_kernel_launches(const lowdiff_ctx* c) { return c ? c->launches.load() : 0; }

const char* lowdiff_last_error(const lowdiff_ctx* c) { return c ? c->last_error.c_str() : "null context"; }

// ---- host-only serialisers used by multi-rank host tests
lowdiff_status lowdiff_write_batch_host(const lowdiff_config* cfg, int64_t first_iter, int32_t n_iters,
                                        const lowdiff_step_scalars* scalars, const uint32_t* blocks) {
  if (validate_cfg(cfg) || !cfg->ckpt_dir || n_iters < 1 || !scalars || !blocks) return LOWDIFF_E_INVALID;
  std::vector<int64_t> numel(cfg->numel, cfg->numel + cfg->n_layers);
  int64_t psi = 0, K = 0;
  for (int l = 0; l < cfg->n_layers; ++l) { psi += numel[l]; K += (int64_t)k_rule((uint64_t)numel[l], cfg->density_ppm); }
  std::vector<uint8_t> pre;
  ld::build_prefix(*cfg, numel, psi, K, pre);
  const uint64_t first = (uint64_t)first_iter;
  const uint32_t n = (uint32_t)n_iters;
  std::memcpy(pre.data() + 16, &first, 8);
  std::memcpy(pre.data() + 24, &n, 4);
  std::vector<uint8_t> body((size_t)n * (32 + 8 * K), 0);
  for (uint32_t i = 0; i < n; ++i) {
    uint8_t* b = body.data() + (size_t)i * (32 + 8 * K);
    const uint64_t it = first + i;
    std::memcpy(b, &it, 8);
    std::memcpy(b + 8, &scalars[i], 12);
    std::memcpy(b + 32, blocks + (size_t)i * 2 * K, 8 * K);
  }
  uint32_t crc = ld::crc32c_update(0xFFFFFFFFu, pre.data(), pre.size());
  crc = ld::crc32c_update(crc, body.data(), body.size()) ^ 0xFFFFFFFFu;
  ::mkdir(cfg->ckpt_dir, 0755);
  std::string err;
  return ld::write_file_atomic(ld::batch_name(cfg->ckpt_dir, cfg->rank, first_iter),
                               {{pre.data(), pre.size()}, {body.data(), body.size()}, {&crc, 4}}, cfg->fsync != 0, &err);
}

lowdiff_status lowdiff_write_full_host(const lowdiff_config* cfg, int64_t iteration, const float* p, const float* m,
                                       const float* v) {
  if (validate_cfg(cfg) || !cfg->ckpt_dir || !p || iteration < 0) return LOWDIFF_E_INVALID;
  uint64_t psi = 0;
  for (int l = 0; l < cfg->n_layers; ++l) psi += (uint64_t)cfg->numel[l];
  const uint64_t sb = psi * cfg->rank / cfg->world, se = psi * (cfg->rank + 1) / cfg->world, S = se - sb;
  std::vector<float> body(3 * S, 0.f);
  const float* src[3] = {p, m, v};
  for (int a = 0; a < 3; ++a)
    if (src[a]) std::memcpy(body.data() + a * S, src[a] + sb, S * 4);
  ::mkdir(cfg->ckpt_dir, 0755);
  std::string err;
  return write_ldf(*cfg, cfg->ckpt_dir, iteration, psi, sb, se, body.data(), &err);
}

}  // extern "C"
