// Checkpoint file formats, CRC-32C and atomic writes (host side of lowdiff_batch_persist /
// lowdiff_full_ckpt / lowdiff_recover).
//
// .ldb (batched differential checkpoint C^B; "groups the buffered
// differential checkpoints ... writes it to storage in a single I/O operation"):
//   header 64 B | hyper 32 B | layer table 16 B x L | n_iters x (32 B block header + 8K) | CRC32C
// .ldf (full checkpoint C^F, this rank's shard of p, m, v, 3*Psi PAPER.md:150):
//   header 64 B | hyper 32 B | p, m, v f32[shard] | CRC32C
// Written as <name>.tmp then rename() so a crash never exposes a partial file.
// Exact byte layout: DESIGN.md "File formats".
#include <fcntl.h>
#include <nmmintrin.h>
#include <sys/stat.h>
#include <sys/uio.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

#include "internal.h"

namespace ld {

uint32_t crc32c_update(uint32_t crc, const void* data, size_t len) {
  // hardware CRC32 (SSE4.2 crc32 instruction implements the Castagnoli polynomial)
  const uint8_t* p = static_cast<const uint8_t*>(data);
  uint64_t c = crc;
  while (len && (reinterpret_cast<uintptr_t>(p) & 7)) { c = _mm_crc32_u8((uint32_t)c, *p++); --len; }
  while (len >= 8) {
    uint64_t w;
    std::memcpy(&w, p, 8);
    c = _mm_crc32_u64(c, w);
    p += 8;
    len -= 8;
  }
  while (len) { c = _mm_crc32_u8((uint32_t)c, *p++); --len; }
  return (uint32_t)c;
}

static std::string pad(int64_t v, int w) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%0*lld", w, (long long)v);
  return buf;
}

std::string batch_name(const std::string& dir, int rank, int64_t first) {
  return dir + "/ld_diff_r" + pad(rank, 3) + "_" + pad(first, 12) + ".ldb";
}

std::string full_name(const std::string& dir, int rank, int64_t it) {
  return dir + "/ld_full_r" + pad(rank, 3) + "_" + pad(it, 12) + ".ldf";
}

namespace {
struct W {
  std::vector<uint8_t>& b;
  void u16(uint16_t v) { raw(&v, 2); }
  void u32(uint32_t v) { raw(&v, 4); }
  void u64(uint64_t v) { raw(&v, 8); }
  void f32(float v) { raw(&v, 4); }
  void raw(const void* p, size_t n) {   // x86-64 is little-endian: native order == file order
    const uint8_t* q = static_cast<const uint8_t*>(p);
    b.insert(b.end(), q, q + n);
  }
};
}  // namespace

// header + hyper + layer table; n_iters (offset 24) and first_iter (offset 16) patched per file
void build_prefix(const lowdiff_config& cfg, const std::vector<int64_t>& numel, int64_t psi, int64_t K,
                  std::vector<uint8_t>& out) {
  out.clear();
  W w{out};
  w.raw("LDB1", 4);
  w.u16(1);
  w.u16((uint16_t)((cfg.error_feedback ? 1 : 0) | (cfg.mean ? 2 : 0)));
  w.u32((uint32_t)cfg.rank);
  w.u32((uint32_t)cfg.world);
  w.u64(0);                        // first_iter (patched)
  w.u32(0);                        // n_iters (patched)
  w.u32((uint32_t)cfg.n_layers);
  w.u64((uint64_t)psi);
  w.u64((uint64_t)K);
  w.u32(cfg.density_ppm);
  w.u32((uint32_t)cfg.optim);
  w.u64(0);
  const float h[5] = {cfg.adam.beta1, cfg.adam.one_minus_beta1, cfg.adam.beta2, cfg.adam.one_minus_beta2,
                      cfg.adam.eps};
  for (float x : h) w.f32(x);
  w.u32(0); w.u32(0); w.u32(0);
  for (int l = 0; l < cfg.n_layers; ++l) {
    uint64_t n = (uint64_t)numel[l];
    uint64_t k = n * cfg.density_ppm / 1000000ull;
    if (k > n) k = n;
    if (k < 1) k = 1;
    w.u64(n);
    w.u32((uint32_t)k);
    w.u32(0);
  }
}

lowdiff_status write_file_atomic(const std::string& path, const std::vector<std::pair<const void*, size_t>>& parts,
                                 bool do_fsync, std::string* err) {
  const std::string tmp = path + ".tmp";
  int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) {
    *err = "open " + tmp + ": " + std::strerror(errno);
    return LOWDIFF_E_IO;
  }
  // one writev per <= 1024 segments / 1 GiB; restart on short writes
  std::vector<iovec> iov;
  for (auto& p : parts) {
    const uint8_t* q = static_cast<const uint8_t*>(p.first);
    size_t n = p.second;
    while (n) {
      size_t c = n > (1u << 30) ? (1u << 30) : n;
      iov.push_back({const_cast<uint8_t*>(q), c});
      q += c;
      n -= c;
    }
  }
  size_t i = 0;
  while (i < iov.size()) {
    int cnt = (int)std::min<size_t>(iov.size() - i, 1024);
    ssize_t wr = ::writev(fd, &iov[i], cnt);
    if (wr < 0) {
      if (errno == EINTR) continue;
      *err = "writev " + tmp + ": " + std::strerror(errno);
      ::close(fd);
      ::unlink(tmp.c_str());
      return LOWDIFF_E_IO;
    }
    size_t left = (size_t)wr;
    while (left && i < iov.size()) {
      if (left >= iov[i].iov_len) { left -= iov[i].iov_len; ++i; }
      else {
        iov[i].iov_base = static_cast<uint8_t*>(iov[i].iov_base) + left;
        iov[i].iov_len -= left;
        left = 0;
      }
    }
  }
  if (do_fsync && ::fsync(fd) != 0) {
    *err = "fsync " + tmp + ": " + std::strerror(errno);
    ::close(fd);
    ::unlink(tmp.c_str());
    return LOWDIFF_E_IO;
  }
  if (::close(fd) != 0) {
    *err = "close " + tmp + ": " + std::strerror(errno);
    ::unlink(tmp.c_str());
    return LOWDIFF_E_IO;
  }
  if (::rename(tmp.c_str(), path.c_str()) != 0) {
    *err = "rename " + tmp + ": " + std::strerror(errno);
    ::unlink(tmp.c_str());
    return LOWDIFF_E_IO;
  }
  if (do_fsync) {   // the rename itself is durable only once the directory entry is on storage
    const size_t slash = path.find_last_of('/');
    const std::string dir = slash == std::string::npos ? "." : (slash == 0 ? "/" : path.substr(0, slash));
    const int dfd = ::open(dir.c_str(), O_RDONLY | O_DIRECTORY | O_CLOEXEC);
    if (dfd < 0 || ::fsync(dfd) != 0) {
      *err = "fsync directory " + dir + ": " + std::strerror(errno);
      if (dfd >= 0) ::close(dfd);
      return LOWDIFF_E_IO;
    }
    ::close(dfd);
  }
  return LOWDIFF_OK;
}

// ---------------------------------------------------------------- CRC-32C combination
// crc(A || B) from crc(A), crc(B) and |B|: appending |B| zero bytes to A is a linear map over GF(2)
// on the 32-bit CRC register; it is applied by squaring the one-zero-bit operator (log |B| steps).
// Attribution: this is the standard zero-extension scheme of zlib's crc32_combine (Mark Adler,
// zlib license) -- same odd/even operator squaring -- with the reflected Castagnoli polynomial.
static uint32_t gf2_times(const uint32_t* mat, uint32_t vec) {
  uint32_t sum = 0;
  for (int i = 0; vec; ++i, vec >>= 1)
    if (vec & 1u) sum ^= mat[i];
  return sum;
}
static void gf2_square(uint32_t* sq, const uint32_t* mat) {
  for (int n = 0; n < 32; ++n) sq[n] = gf2_times(mat, mat[n]);
}
uint32_t crc32c_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b) {
  if (len_b == 0) return crc_a;
  uint32_t even[32], odd[32];
  odd[0] = 0x82F63B78u;   // one zero bit: the reflected Castagnoli polynomial
  for (int n = 1; n < 32; ++n) odd[n] = 1u << (n - 1);
  gf2_square(even, odd);   // two zero bits
  gf2_square(odd, even);   // four zero bits
  do {                     // one zero byte = eight zero bits, then doublings
    gf2_square(even, odd);
    if (len_b & 1u) crc_a = gf2_times(even, crc_a);
    len_b >>= 1;
    if (!len_b) break;
    gf2_square(odd, even);
    if (len_b & 1u) crc_a = gf2_times(odd, crc_a);
    len_b >>= 1;
  } while (len_b);
  return crc_a ^ crc_b;
}

// ---------------------------------------------------------------- streamed file -> device
// Bytes [off, off + total) of `fd` go to the device segments in order (a NULL segment is read and
// checksummed but not copied), through pinned chunks: `threads` readers each pread a chunk, take
// its CRC-32C and copy it H2D on their own stream, so storage, checksum and PCIe overlap.  *crc =
// CRC-32C of the bytes (standard init/xorout), combined in file order.
lowdiff_status stream_to_device(int fd, uint64_t off, const std::vector<std::pair<void*, uint64_t>>& segs,
                                Staging& stg, uint32_t* crc, std::string* err) {
  uint64_t total = 0;
  for (auto& sg : segs) total += sg.second;
  const uint64_t CH = Staging::kChunk;
  const uint64_t n_chunks = (total + CH - 1) / CH;
  if (n_chunks == 0) { *crc = 0; return LOWDIFF_OK; }
  std::vector<uint32_t> crcs(n_chunks, 0u);
  std::atomic<int> failed{0};
  std::string first_err;
  std::mutex emu;
  auto set_err = [&](const std::string& m) {
    std::lock_guard<std::mutex> g(emu);
    if (!failed.exchange(1)) first_err = m;
  };
  // pinned chunks and streams are allocated once per context and reused (cudaHostAlloc is slow)
  const int want = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  while ((int)stg.bufs.size() < want) {
    uint8_t* b = nullptr;
    cudaStream_t st = nullptr;
    if (cudaHostAlloc((void**)&b, CH, cudaHostAllocDefault) != cudaSuccess) break;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) { cudaFreeHost(b); break; }
    stg.bufs.push_back(b);
    stg.streams.push_back(st);
  }
  if (stg.bufs.empty()) {
    *err = "pinned staging for the checkpoint read";
    return LOWDIFF_E_CUDA;
  }
  const int threads = (int)std::min<uint64_t>(stg.bufs.size(), n_chunks);
  std::vector<uint8_t*>& bufs = stg.bufs;
  std::vector<cudaStream_t>& streams = stg.streams;
  int dev = 0;
  cudaGetDevice(&dev);
  auto worker = [&](int t) {
    cudaSetDevice(dev);
    for (uint64_t c = (uint64_t)t; c < n_chunks && !failed.load(); c += (uint64_t)threads) {
      const uint64_t b0 = c * CH, len = std::min(CH, total - b0);
      uint64_t got = 0;
      while (got < len) {
        const ssize_t r = ::pread(fd, bufs[t] + got, len - got, (off_t)(off + b0 + got));
        if (r <= 0) { set_err(std::string("read: ") + (r < 0 ? std::strerror(errno) : "unexpected end of file")); return; }
        got += (uint64_t)r;
      }
      crcs[c] = crc32c_update(0xFFFFFFFFu, bufs[t], len) ^ 0xFFFFFFFFu;
      // copy the chunk into the segments it overlaps
      uint64_t seg_start = 0;
      for (auto& sg : segs) {
        const uint64_t s0 = seg_start, s1 = seg_start + sg.second;
        seg_start = s1;
        const uint64_t a = std::max(s0, b0), z = std::min(s1, b0 + len);
        if (a >= z || !sg.first) continue;
        if (cudaMemcpyAsync(static_cast<uint8_t*>(sg.first) + (a - s0), bufs[t] + (a - b0), z - a,
                            cudaMemcpyHostToDevice, streams[t]) != cudaSuccess) {
          set_err("H2D of a checkpoint chunk");
          return;
        }
      }
      if (cudaStreamSynchronize(streams[t]) != cudaSuccess) { set_err("H2D of a checkpoint chunk"); return; }
    }
  };
  if (threads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
  }
  if (failed.load()) {
    *err = first_err;
    return LOWDIFF_E_IO;
  }
  uint32_t acc = crcs[0];
  for (uint64_t c = 1; c < n_chunks; ++c) acc = crc32c_combine(acc, crcs[c], std::min(CH, total - c * CH));
  *crc = acc;
  return LOWDIFF_OK;
}

}  // namespace ld
