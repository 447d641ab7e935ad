// C-ABI implementation of liblowdiff (part 1): context, compress / exchange (NCCL, peer memory,
// CUDA graphs), reuse queue -> pinned ring -> writer thread, full checkpoints, stats, host writers,
// and the shared helpers of api_util.h.  Recovery: recover.cpp; union-compacted differentials:
// union_api.cpp; LowDiff+ snapshot and CPU replica: lowdiff_plus.cpp.  Kernels: *.cu.
// See include/lowdiff.h.
#include <dirent.h>
#include <cerrno>
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

using ld::DevPlan;

namespace ld {
namespace api {

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
  c->plan_bytes += bytes;
  if (!h.empty()) CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *d = static_cast<T*>(p);
  return LOWDIFF_OK;
}

lowdiff_status dalloc(lowdiff_ctx* c, size_t bytes, void** d) {
  CK(cudaMalloc(d, std::max<size_t>(bytes, 16)));
  c->dev_allocs.push_back(*d);
  c->plan_bytes += std::max<size_t>(bytes, 16);
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
  // bounded candidate scratch: cs slots per 1024-element segment, O(K) in total
  P.cs = ld::compress_seg_capacity(c->cfg.density_ppm, (uint64_t)P.n_chunks * ld::kSegsPerChunk);
  if (const char* v = std::getenv("LOWDIFF_SEG_SLOTS")) {   // tests / tuning: force the slot capacity
    const int f = std::atoi(v);
    if (f >= 8 && f <= ld::kSeg) P.cs = f & ~7;
  }
  if ((st = dalloc(c, nc * ld::kSegsPerChunk * (size_t)P.cs * sizeof(uint64_t), &p))) return st; P.cand = (uint64_t*)p;
  if ((st = dalloc(c, nc * ld::kSegsPerChunk * sizeof(uint32_t), &p))) return st; P.seg_count = (uint32_t*)p;
  if ((st = dalloc(c, nc * 4 * 3, &p))) return st;
  P.chunk_count = (uint32_t*)p; P.chunk_dm = P.chunk_count + nc; P.refill_list = P.chunk_dm + nc;
  if ((st = dalloc(c, ld::compress_hist_bytes((int)nl), &p))) return st; P.hist = (uint32_t*)p;
  if ((st = dalloc(c, nl * sizeof(ld::LayerSel), &p))) return st; P.sel = (ld::LayerSel*)p;
  CK(cudaMemset(P.sel, 0, nl * sizeof(ld::LayerSel)));   // band = 0: not yet adapted
  if ((st = dalloc(c, nl * 4 * 6, &p))) return st;
  P.thr = (uint32_t*)p; P.thr_used = P.thr + nl; P.sel_T = P.thr_used + nl; P.layer_total = P.sel_T + nl;
  P.sel_cut = P.layer_total + nl; P.trace = P.sel_cut + nl;
  CK(cudaMemset(P.layer_total, 0, nl * 4 * 3));   // layer_total, sel_cut, trace
  if ((st = dalloc(c, (size_t)nc * 8, &p))) return st; P.chunk_state = (unsigned long long*)p;
  CK(cudaMemset(P.thr, 0xFF, nl * 4));   // no speculative band before the first call
  CK(cudaMemset(P.sel_T, 0xFF, nl * 4));  // no previous k-th key (no drift estimate yet)
  CK(cudaMemset(P.thr_used, 0, nl * 4));
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

// Restart hygiene: when persisting (re)starts at iteration t -- the first
// batch_persist / union_persist of a context, or the first after a recovery -- every file of this
// rank that holds iterations >= t belongs to an abandoned run (blocks t.. of the previous
// trajectory, full checkpoints of states >= t).  Left in place, the chain rule "the file with the
// later first iteration wins" could splice its blocks into the new run's chain (an old
// ..._000000000008.ldb would override blocks 8.. of a new ..._000000000007.ldb), or extend the
// chain past the new run's last block.  So: files starting at >= t are removed; a batch file
// straddling t is rewritten (atomically) with only its blocks < t; .ldf files of iterations >= t
// are removed.  kinds: bit0 .ldb, bit1 .ldu, bit2 .ldf.
static bool rewrite_prefix_blocks(const std::string& path, size_t head, int64_t first, int64_t keep, bool ldu,
                                  bool do_fsync, std::string* err) {
  std::vector<uint8_t> buf;
  if (!read_all(path, buf) || buf.size() < head + 4) return false;
  if (lowdiff_crc32c(buf.data(), buf.size() - 4) != rd<uint32_t>(buf.data() + buf.size() - 4)) return false;
  const uint64_t K = rd<uint64_t>(buf.data() + 40);
  size_t off = head;
  for (int64_t i = 0; i < keep; ++i) {
    if (off + 32 > buf.size() - 4 || (int64_t)rd<uint64_t>(buf.data() + off) != first + i) return false;
    const uint64_t n = ldu ? rd<uint32_t>(buf.data() + off + 20) : K;
    off += 32 + 8 * n;
  }
  if (off > buf.size() - 4) return false;
  const uint32_t n_it = (uint32_t)keep;
  std::memcpy(buf.data() + 24, &n_it, 4);
  const uint32_t crc = lowdiff_crc32c(buf.data(), off);
  return ld::write_file_atomic(path, {{buf.data(), off}, {&crc, 4}}, do_fsync, err) == LOWDIFF_OK;
}

lowdiff_status retire_from(const lowdiff_config& cfg, int64_t t, int kinds, std::string* err) {
  if (!cfg.ckpt_dir) return LOWDIFF_OK;
  DIR* d = opendir(cfg.ckpt_dir);
  if (!d) return LOWDIFF_OK;   // nothing persisted yet
  std::vector<std::pair<std::string, int>> mine;   // (name, kind bit)
  while (dirent* de = readdir(d)) {
    unsigned r; long long it;
    if ((kinds & 1) && parse_name(de->d_name, "diff", "ldb", &r, &it) && r == (unsigned)cfg.rank) mine.push_back({de->d_name, 1});
    else if ((kinds & 2) && parse_name(de->d_name, "union", "ldu", &r, &it) && r == (unsigned)cfg.rank) mine.push_back({de->d_name, 2});
    else if ((kinds & 4) && parse_name(de->d_name, "full", "ldf", &r, &it) && r == (unsigned)cfg.rank) mine.push_back({de->d_name, 4});
  }
  closedir(d);
  for (auto& f : mine) {
    unsigned r; long long it;
    const char* kind = f.second == 1 ? "diff" : f.second == 2 ? "union" : "full";
    const char* ext = f.second == 1 ? "ldb" : f.second == 2 ? "ldu" : "ldf";
    parse_name(f.first.c_str(), kind, ext, &r, &it);
    const std::string path = std::string(cfg.ckpt_dir) + "/" + f.first;
    if (it >= t) {
      if (::unlink(path.c_str()) != 0 && errno != ENOENT) { *err = "cannot remove stale " + path; return LOWDIFF_E_IO; }
      continue;
    }
    if (f.second == 4) continue;
    uint8_t h[32];
    size_t fsz = 0;
    if (!read_head(path, h, 32, &fsz)) continue;     // unreadable: recovery reports it as before
    const int64_t n = rd<uint32_t>(h + 24);
    if (it + n <= t) continue;                       // entirely before the restart
    const size_t head = f.second == 1 ? 96 + 16 * (size_t)cfg.n_layers : 112 + 16 * (size_t)cfg.n_layers;
    if (!rewrite_prefix_blocks(path, head, it, t - it, f.second == 2, cfg.fsync != 0, err)) {
      if (err->empty()) *err = "cannot truncate stale blocks of " + path;
      return LOWDIFF_E_IO;
    }
  }
  return LOWDIFF_OK;
}

lowdiff_status validate_cfg(const lowdiff_config* cfg) {
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

}  // namespace api
}  // namespace ld
using namespace ld::api;

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
  if (!mismatches || !first_bad || which < 0 || which > 5) return LOWDIFF_E_INVALID;
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
  // An NCCL communicator whenever an id is given -- also at world 1 (a 1-rank communicator: the
  // allgather is then a device copy, but every NCCL call site runs).  No id: world 1 merges straight
  // from the send block; world > 1 without an id is a recovery / merge-only context.
  if (cfg->nccl_unique_id) {
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
  if (c->scal_dev) cudaFree(c->scal_dev);
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
  NvtxRange nvtx_("lowdiff_compress");
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
  NvtxRange nvtx_("lowdiff_exchange_peer");
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

// SURVEY NEXT-1, both halves fused: the allgather folded into the merge over peer memory AND the
// merge folded into the optimizer step -- the peers' entries of each tile are read over NVLink,
// merged in shared memory and applied to p, m, v in one pass (no gathered buffer, no dense G).
lowdiff_status lowdiff_exchange_peer_update(lowdiff_ctx* c, int32_t slot, const lowdiff_step_scalars* scalars,
                                            float* p, float* m, float* v, void* stream) {
  NvtxRange nvtx_("lowdiff_exchange_peer_update");
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!c->peer_set) return fail(c, LOWDIFF_E_STATE, "exchange_peer_update: call lowdiff_peer_set first");
  const bool adam = c->cfg.optim == LOWDIFF_ADAM;
  if (slot < 0 || slot >= c->peer_slots || !scalars || !p || !aligned16(p) || (adam && (!m || !v)) ||
      (m && !aligned16(m)) || (v && !aligned16(v)))
    return fail(c, LOWDIFF_E_INVALID, "exchange_peer_update: bad argument (p, m, v 16-byte aligned device arrays)");
  if (!c->peer_epoch[slot]) return fail(c, LOWDIFF_E_STATE, "exchange_peer_update: nothing was compressed into the slot");
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
  const ld::PeerOpt o{c->cfg.adam.beta1, c->cfg.adam.one_minus_beta1, c->cfg.adam.beta2, c->cfg.adam.one_minus_beta2,
                      c->cfg.adam.eps, scalars->lr, scalars->bc1_inv, scalars->bc2_inv};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int h;
  ld::prof_begin(c, "peer_update", s, &h);
  cudaError_t e = ld::launch_peer_update(T, (uint64_t)c->K, c->psi, c->cfg.mean != 0, adam, o, p, m, v, s);
  ld::prof_end(c, h, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "peer_update");
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
  NvtxRange nvtx_("lowdiff_merge");
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
  NvtxRange nvtx_("lowdiff_exchange");
  lowdiff_status st = entry(c);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!send || !dense_out || (c->cfg.world > 1 && !gathered)) return fail(c, LOWDIFF_E_INVALID, "exchange: NULL buffer");
  const size_t blk = 2 * (size_t)c->K;
  if (c->cfg.world > 1 || (c->comm && gathered)) {
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
  NvtxRange nvtx_("lowdiff_exchange_update");
  lowdiff_status st = entry(c);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!send || !scalars || (c->cfg.world > 1 && !gathered)) return fail(c, LOWDIFF_E_INVALID, "exchange_update: NULL buffer");
  const size_t blk = 2 * (size_t)c->K;
  const uint32_t* blocks = send;
  if (c->cfg.world > 1 || (c->comm && gathered)) {
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
  NvtxRange nvtx_("lowdiff_batch_persist");
  lowdiff_status st = entry(c);
  if (st) return st;
  if ((st = take_deferred(c))) return st;
  if (!scalars || !send) return fail(c, LOWDIFF_E_INVALID, "batch_persist: NULL argument");
  if (c->next_iter >= 0 && iteration != c->next_iter)
    return fail(c, LOWDIFF_E_STATE, "batch_persist: iteration " + std::to_string(iteration) + " after " +
                                        std::to_string(c->next_iter - 1) + " (must be consecutive)");
  if (c->next_iter < 0 && c->cfg.write_files) {   // persisting (re)starts here: retire the abandoned run
    if (c->full_writer.joinable()) c->full_writer.join();
    std::string err;
    if ((st = retire_from(c->cfg, iteration, 1 | 4, &err))) return fail(c, st, err);
  }
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
  NvtxRange nvtx_("lowdiff_full_ckpt");
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

lowdiff_status lowdiff_get_stats(const lowdiff_ctx* c, lowdiff_stats* out) {
  if (!c || !out) return LOWDIFF_E_INVALID;
  out->files_written = c->files_written;
  out->bytes_written = c->bytes_written;
  out->ring_stall_ns = c->stall_ns;
  out->writer_busy_ns = c->writer_ns;
  uint32_t cnt[4] = {0, 0, 0, 0};
  if (cudaMemcpy(cnt, c->plan.counters, 16, cudaMemcpyDeviceToHost) == cudaSuccess) {   // of the last call
    out->spec_hits = cnt[1];
    out->spec_misses = cnt[2];
    out->spec_candidates = cnt[3];
  } else {
    out->spec_hits = out->spec_misses = out->spec_candidates = -1;
  }
  uint32_t cnt2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  out->direct_segments = cudaMemcpy(cnt2, c->plan.counters, 32, cudaMemcpyDeviceToHost) == cudaSuccess ? cnt2[5] : -1;
  out->compress_scratch_bytes = (int64_t)c->plan_bytes;
  out->device_bytes = (int64_t)(c->plan_bytes + c->merge_scratch_bytes + c->replay_scratch_bytes +
                                c->full_stage_cap * 4 + c->union_scratch_bytes);
  out->replica_busy_ns = c->rep_ns;
  out->replica_stall_ns = c->rep_stall_ns;
  out->union_files_written = c->u_files;
  out->union_bytes_written = c->u_bytes;
  out->union_entries = c->u_entries;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_compress_trace(lowdiff_ctx* c, int32_t cap, int32_t* n_large, int32_t* layer, int32_t* level,
                                      uint32_t* candidates, uint32_t* threshold) {
  lowdiff_status st = entry(c);
  if (st) return st;
  if (!n_large) return fail(c, LOWDIFF_E_INVALID, "compress_trace: NULL n_large");
  const int nl = c->plan.n_large;
  *n_large = nl;
  if (!layer && !level && !candidates && !threshold) return LOWDIFF_OK;
  if (cap < nl) return fail(c, LOWDIFF_E_INVALID, "compress_trace: arrays shorter than n_large");
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> ids((size_t)nl);
  if (nl) CK(cudaMemcpy(ids.data(), c->plan.large_layers, (size_t)nl * 4, cudaMemcpyDeviceToHost));
  if (layer) std::copy(ids.begin(), ids.end(), layer);
  if (level && nl) CK(cudaMemcpy(level, c->plan.trace, (size_t)nl * 4, cudaMemcpyDeviceToHost));
  if (candidates && nl) CK(cudaMemcpy(candidates, c->plan.layer_total, (size_t)nl * 4, cudaMemcpyDeviceToHost));
  if (threshold && nl) CK(cudaMemcpy(threshold, c->plan.thr_used, (size_t)nl * 4, cudaMemcpyDeviceToHost));
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

lowdiff_status lowdiff_retire_from(const lowdiff_config* cfg, int64_t iteration, int32_t kinds) {
  if (validate_cfg(cfg) || !cfg->ckpt_dir || iteration < 0 || kinds < 0 || kinds > 7) return LOWDIFF_E_INVALID;
  std::string err;
  return retire_from(*cfg, iteration, kinds, &err);
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
