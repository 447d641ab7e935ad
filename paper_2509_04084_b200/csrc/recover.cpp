// C-ABI implementation of liblowdiff (part 2): chain scan and recovery -- full checkpoints and
// differential blocks streamed to the device (files.cpp), the fused replay (merge_replay.cu),
// sharded recovery (Alg. 1 recovery).
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

lowdiff_status bcast_shards(lowdiff_ctx* c, float* dst[3], cudaStream_t s) {
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

lowdiff_status load_full_shards(lowdiff_ctx* c, const std::vector<std::string>& paths, int64_t F, bool sharded,
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

}  // namespace api
}  // namespace ld

extern "C" {

lowdiff_status lowdiff_replay_range(lowdiff_ctx* c, int32_t optim, int32_t world, int64_t n_steps,
                                    const uint32_t* diffs, const lowdiff_step_scalars* scalars, int64_t begin,
                                    int64_t end, float* p, float* m, float* v, void* stream) {
  NvtxRange nvtx_("lowdiff_replay_range");
  lowdiff_status st = entry(c);
  if (st) return st;
  if (begin >= 0 && begin == end && end <= c->psi && n_steps >= 0) return LOWDIFF_OK;   // empty range
  if (world < 1 || n_steps < 0 || (n_steps && (!diffs || !scalars)) || !p ||
      (optim == LOWDIFF_ADAM && (!m || !v)) || (optim != LOWDIFF_ADAM && optim != LOWDIFF_SGD) || begin < 0 ||
      end > c->psi || begin > end)
    return fail(c, LOWDIFF_E_INVALID, "replay: bad argument");
  if (!n_steps || begin == end) return LOWDIFF_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // per-step scalars to the device: a context buffer that only grows (a cudaMallocAsync / free
  // pair per call returned the pool's memory at every synchronisation and re-mapped it: ~27 ms)
  const size_t sbytes = (size_t)n_steps * 12;
  if (c->scal_cap < sbytes) {
    if (c->scal_dev) cudaFree(c->scal_dev);
    c->scal_dev = nullptr;
    c->scal_cap = 0;
    CK(cudaMalloc((void**)&c->scal_dev, sbytes));
    c->scal_cap = sbytes;
  }
  CK(cudaMemcpyAsync(c->scal_dev, scalars, sbytes, cudaMemcpyHostToDevice, s));
  const float consts[5] = {c->cfg.adam.beta1, c->cfg.adam.one_minus_beta1, c->cfg.adam.beta2,
                           c->cfg.adam.one_minus_beta2, c->cfg.adam.eps};
  cudaError_t e = ld::launch_replay(c, optim, c->cfg.mean != 0, consts, world, n_steps, diffs, c->scal_dev,
                                    (uint64_t)begin, (uint64_t)end, nullptr, p, m, v, s);
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

// Full checkpoint F -> p, m, v (every shard, or only this rank's when sharded): size, magic, CRC and
// header fields verified (else E_CORRUPT); optim, Adam constants and flags from the file.

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
  NvtxRange nvtx_(sharded ? "lowdiff_recover_sharded" : "lowdiff_recover");
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
  c->next_iter = -1;     // persisting may resume at ch.last + 1; its first call retires the abandoned run
  c->u_next_iter = -1;
  return LOWDIFF_OK;
}

lowdiff_status lowdiff_recover(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int64_t* recovered,
                               void* stream) {
  return recover_impl(c, target, p, m, v, recovered, stream, false);
}

lowdiff_status lowdiff_recover_sharded(lowdiff_ctx* c, int64_t target, float* p, float* m, float* v, int32_t gather,
                                       int64_t* recovered, void* stream) {
  lowdiff_status st = recover_impl(c, target, p, m, v, recovered, stream, true);
  if (st || !gather || (c->cfg.world == 1 && !c->comm)) return st;   // world 1 without NCCL: nothing to gather
  if (!c->comm) return fail(c, LOWDIFF_E_STATE, "recover_sharded: gather needs an NCCL context");
  float* dst[3] = {p, m, v};
  if ((st = bcast_shards(c, dst, static_cast<cudaStream_t>(stream)))) return st;
  CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return LOWDIFF_OK;
}

}  // extern "C"
