// ============================================================================
// LowDiff ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the LowDiff
// (arXiv 2509.04084, SC'25) data-parallel hot path, written from the paper:
//   compress   -- Alg. 1 line 4 "Comp", sparsification with
//                 rho = 0.01, per-layer top-k with error feedback
//                 (BASELINE.json north_star; readings R-1..R-6)
//   exchange   -- Alg. 1 line 5 "Sync" ("Allgather or Allreduce"
//                 PAPER.md:213) and line 7 "Comp^-1"
//   serialize  -- batched gradient writing, Steps 1-3;
//                 full checkpoint Save(M_t), 3*Psi
//   optimizer  -- Eq. 1 M_{t+1} = M_t + Adam(G_t), Adam
//                 moments; SGD (north_star; not in the paper)
//   recover    -- Alg. 1 recovery process, Eq. 2
//   union      -- union-compacted differential C^U_t: the synchronised G~_t
//                 (Alg. 1 lines 5-6) kept as a dictionary
//                 (PAPER.md:452), its .ldu file and recovery from it (R-29)
//   accumulate -- Accumulated batch mode: the b dictionaries of a batch added
//                 into one ("tensor addition", PAPER.md:270/274/452), one
//                 optimizer step per batch at recovery -- INEXACT for b > 1
//                 by construction (R-30)
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this library.  It shares no code, header, table or constant generator
// with the CUDA path (paper_2509_04084_b200/csrc) and never includes a CUDA
// header.  Compiled -O2 -ffp-contract=off -fno-fast-math; FTZ/DAZ are checked
// off at every entry point.  Every float operation below is one IEEE-754
// binary32 operation, rounded to nearest even, in the order written.
//
// Parity pins: see tests/test_oracle_*.py (brute-force rank definition,
// worked examples of SPEC.md, invariants, density-1 SGD == dense DP, CRC-32C
// check value, Adam closed forms).  No function here is "parity unpinned".
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <dirent.h>
#include <map>
#include <string>
#include <vector>
#include <xmmintrin.h>

namespace {

enum Status {
  OK = 0, E_INVALID = 1, E_DIM = 2, E_NUMERIC = 3, E_IO = 6, E_CORRUPT = 7, E_GAP = 8,
  E_FPENV = 20
};

bool fp_env_ok() {
  // MXCSR bit 15 = FTZ, bit 6 = DAZ: denormals must be preserved (R-20).
  return (_mm_getcsr() & 0x8040u) == 0;
}

uint32_t float_bits(float x) { uint32_t u; std::memcpy(&u, &x, 4); return u; }
float bits_float(uint32_t u) { float x; std::memcpy(&x, &u, 4); return x; }

// k_l = max(1, min(n_l, floor(n_l * ppm / 1e6))) in integer arithmetic (R-3).
uint64_t k_of(uint64_t n, uint32_t ppm) {
  uint64_t k = (n * (uint64_t)ppm) / 1000000ull;
  if (k > n) k = n;
  if (k < 1) k = 1;
  return k;
}

// ---------------------------------------------------------------- little-endian put/get
void put_u16(std::vector<uint8_t>& b, uint16_t v) { for (int i = 0; i < 2; ++i) b.push_back((uint8_t)(v >> (8 * i))); }
void put_u32(std::vector<uint8_t>& b, uint32_t v) { for (int i = 0; i < 4; ++i) b.push_back((uint8_t)(v >> (8 * i))); }
void put_u64(std::vector<uint8_t>& b, uint64_t v) { for (int i = 0; i < 8; ++i) b.push_back((uint8_t)(v >> (8 * i))); }
void put_f32(std::vector<uint8_t>& b, float v) { put_u32(b, float_bits(v)); }
uint16_t get_u16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
uint32_t get_u32(const uint8_t* p) { uint32_t v = 0; for (int i = 3; i >= 0; --i) v = (v << 8) | p[i]; return v; }
uint64_t get_u64(const uint8_t* p) { uint64_t v = 0; for (int i = 7; i >= 0; --i) v = (v << 8) | p[i]; return v; }
float get_f32(const uint8_t* p) { return bits_float(get_u32(p)); }

// CRC-32C (Castagnoli), reflected polynomial 0x82F63B78, init and xorout
// 0xFFFFFFFF, one bit at a time (R-23; "32-bit CRC").
uint32_t crc32c_bitwise(const uint8_t* p, uint64_t n) {
  uint32_t crc = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) {
    crc ^= p[i];
    for (int b = 0; b < 8; ++b) crc = (crc & 1u) ? (crc >> 1) ^ 0x82F63B78u : (crc >> 1);
  }
  return crc ^ 0xFFFFFFFFu;
}

bool read_file(const std::string& path, std::vector<uint8_t>& out) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize((size_t)(sz < 0 ? 0 : sz));
  size_t got = out.empty() ? 0 : std::fread(out.data(), 1, out.size(), f);
  std::fclose(f);
  return got == out.size();
}

}  // namespace

extern "C" {

int lowdiff_ref_fp_env_ok() { return fp_env_ok() ? 1 : 0; }

uint64_t lowdiff_ref_k(uint64_t numel, uint32_t ppm) { return k_of(numel, ppm); }

uint32_t lowdiff_ref_crc32c(const void* buf, uint64_t len) {
  return crc32c_bitwise(static_cast<const uint8_t*>(buf), len);
}

// --------------------------------------------------------------------------
// compress: Alg. 1 line 4, G~_{i,t} <- Comp(G_{i,t})
//
// For each layer l in table order (R-2, per-layer top-k):
//  (1) acc[i] = residual[i] + grad[i]   (ef = 1; acc = grad when ef = 0)
//  (2) any non-finite acc -> E_NUMERIC  (R-5)
//  (3) key[i] = bits(acc[i]) & 0x7FFFFFFF  (R-4; monotone in |acc|)
//  (4) sort the layer's positions by (key descending, index ascending)
//  (5) keep the first k_l; sort them ascending
//  (6) emit idx = off_l + i and val = acc[i] at koff_l
//  (7) residual' = acc with the kept positions set to +0.0f (ef = 1 only, R-6)
// send = idx u32[K] followed by val f32-bits u32[K].
// --------------------------------------------------------------------------
int lowdiff_ref_compress(int n_layers, const int64_t* numel, uint32_t ppm, int ef,
                         const float* grad, float* residual, uint32_t* send) {
  if (!fp_env_ok()) return E_FPENV;
  if (n_layers <= 0 || !numel || !grad || !send || (ef && !residual)) return E_INVALID;
  if (ppm < 1 || ppm > 1000000) return E_INVALID;
  uint64_t K = 0;
  for (int l = 0; l < n_layers; ++l) {
    if (numel[l] <= 0) return E_DIM;
    K += k_of((uint64_t)numel[l], ppm);
  }
  uint32_t* out_idx = send;
  uint32_t* out_val = send + K;
  uint64_t off = 0, koff = 0;
  for (int l = 0; l < n_layers; ++l) {
    const uint64_t n = (uint64_t)numel[l];
    const uint64_t k = k_of(n, ppm);
    std::vector<float> acc(n);
    for (uint64_t i = 0; i < n; ++i) acc[i] = ef ? residual[off + i] + grad[off + i] : grad[off + i];
    for (uint64_t i = 0; i < n; ++i)
      if (!std::isfinite(acc[i])) return E_NUMERIC;
    std::vector<uint32_t> key(n);
    for (uint64_t i = 0; i < n; ++i) key[i] = float_bits(acc[i]) & 0x7FFFFFFFu;
    std::vector<uint64_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
      if (key[a] != key[b]) return key[a] > key[b];
      return a < b;
    });
    std::vector<uint64_t> sel(order.begin(), order.begin() + (long)k);
    std::sort(sel.begin(), sel.end());
    for (uint64_t e = 0; e < k; ++e) {
      out_idx[koff + e] = (uint32_t)(off + sel[e]);
      out_val[koff + e] = float_bits(acc[sel[e]]);
    }
    if (ef) {
      for (uint64_t i = 0; i < n; ++i) residual[off + i] = acc[i];
      for (uint64_t e = 0; e < k; ++e) residual[off + sel[e]] = 0.0f;
    }
    off += n;
    koff += k;
  }
  return OK;
}

// --------------------------------------------------------------------------
// exchange: Alg. 1 lines 5 and 7: the gathered blocks of
// all N ranks (rank r at offset r*2K) are decompressed into the dense
// aggregated gradient.  S = +0.0f everywhere; for r = 0..N-1 in order, for each
// entry: S[idx] = S[idx] + val.  Then G = S / N (mean = 1) or G = S (mean = 0).
// (R-8: rank-order sum from +0.0f, one IEEE divide.)
// --------------------------------------------------------------------------
int lowdiff_ref_exchange(int world, uint64_t K, uint64_t psi, const uint32_t* gathered,
                         int mean, float* dense_out) {
  if (!fp_env_ok()) return E_FPENV;
  if (world < 1 || !gathered || !dense_out) return E_INVALID;
  std::vector<float> S(psi, 0.0f);
  for (int r = 0; r < world; ++r) {
    const uint32_t* idx = gathered + (uint64_t)r * 2 * K;
    const uint32_t* val = idx + K;
    for (uint64_t e = 0; e < K; ++e) {
      if (idx[e] >= psi) return E_DIM;
      S[idx[e]] = S[idx[e]] + bits_float(val[e]);
    }
  }
  const float n = (float)world;
  for (uint64_t j = 0; j < psi; ++j) dense_out[j] = mean ? S[j] / n : S[j];
  return OK;
}

// --------------------------------------------------------------------------
// Adam constants and per-step scalars (R-11): derived in double and
// rounded to fp32 once.  consts = {beta1, 1-beta1, beta2, 1-beta2, eps};
// scalars(t) = {lr_t, 1/(1-beta1^t), 1/(1-beta2^t)} with beta^t formed by t
// repeated double multiplications.
// --------------------------------------------------------------------------
void lowdiff_ref_adam_consts(double beta1, double beta2, double eps, float* out5) {
  out5[0] = (float)beta1;
  out5[1] = (float)(1.0 - beta1);
  out5[2] = (float)beta2;
  out5[3] = (float)(1.0 - beta2);
  out5[4] = (float)eps;
}

void lowdiff_ref_step_scalars(int64_t t, double lr, double beta1, double beta2, float* out3) {
  double p1 = 1.0, p2 = 1.0;
  for (int64_t i = 0; i < t; ++i) { p1 *= beta1; p2 *= beta2; }
  out3[0] = (float)lr;
  out3[1] = (float)(1.0 / (1.0 - p1));
  out3[2] = (float)(1.0 / (1.0 - p2));
}

// Adam (Kingma-Ba with bias correction), Eq. 1, dense over
// all Psi (R-10), one element at a time, fp32, this exact op order (R-11):
//   m  = b1*m + c1*g ; v = b2*v + c2*(g*g) ; mh = m*r1 ; vh = v*r2
//   d  = sqrt(vh) + eps ; u = mh / d ; p = p - lr*u
int lowdiff_ref_adam_step(uint64_t psi, const float* G, const float* consts5, const float* scal3,
                          float* p, float* m, float* v) {
  if (!fp_env_ok()) return E_FPENV;
  const float b1 = consts5[0], c1 = consts5[1], b2 = consts5[2], c2 = consts5[3], eps = consts5[4];
  const float lr = scal3[0], r1 = scal3[1], r2 = scal3[2];
  for (uint64_t j = 0; j < psi; ++j) {
    const float g = G[j];
    const float t1 = b1 * m[j];
    const float t2 = c1 * g;
    m[j] = t1 + t2;
    const float gg = g * g;
    const float t3 = b2 * v[j];
    const float t4 = c2 * gg;
    v[j] = t3 + t4;
    const float mh = m[j] * r1;
    const float vh = v[j] * r2;
    const float d = std::sqrt(vh) + eps;
    const float u = mh / d;
    const float step = lr * u;
    p[j] = p[j] - step;
  }
  return OK;
}

// SGD: p = p - lr*G (north_star; not in the paper, R-12).
int lowdiff_ref_sgd_step(uint64_t psi, const float* G, float lr, float* p) {
  if (!fp_env_ok()) return E_FPENV;
  for (uint64_t j = 0; j < psi; ++j) {
    const float step = lr * G[j];
    p[j] = p[j] - step;
  }
  return OK;
}

// --------------------------------------------------------------------------
// .ldb batched differential checkpoint C^B (b differentials
// grouped and written in one I/O).  Layout:
//   header 64 B | hyper 32 B | layer table 16 B * L | n_iters blocks | CRC-32C
// block = {u64 iteration, f32 lr, f32 bc1_inv, f32 bc2_inv, 3 x u32 0} then the
// rank's own send block (idx u32[K], val u32[K]).
// --------------------------------------------------------------------------
int64_t lowdiff_ref_batch_bytes(int n_layers, uint64_t K, int n_iters) {
  return 64 + 32 + 16 * (int64_t)n_layers + (int64_t)n_iters * (32 + 8 * (int64_t)K) + 4;
}

int lowdiff_ref_batch_serialize(uint32_t rank, uint32_t world, uint64_t first_iter, uint32_t n_iters,
                                int n_layers, const int64_t* numel, uint32_t ppm, uint32_t optim,
                                uint32_t flags, const float* consts5, const float* scalars /* n x 3 */,
                                const uint32_t* blocks /* n x 2K */, uint8_t* out, uint64_t cap) {
  uint64_t psi = 0, K = 0;
  for (int l = 0; l < n_layers; ++l) { psi += (uint64_t)numel[l]; K += k_of((uint64_t)numel[l], ppm); }
  std::vector<uint8_t> b;
  b.push_back('L'); b.push_back('D'); b.push_back('B'); b.push_back('1');
  put_u16(b, 1); put_u16(b, (uint16_t)flags);
  put_u32(b, rank); put_u32(b, world);
  put_u64(b, first_iter);
  put_u32(b, n_iters); put_u32(b, (uint32_t)n_layers);
  put_u64(b, psi); put_u64(b, K);
  put_u32(b, ppm); put_u32(b, optim);
  put_u64(b, 0);
  for (int i = 0; i < 5; ++i) put_f32(b, consts5[i]);
  for (int i = 0; i < 3; ++i) put_u32(b, 0);
  for (int l = 0; l < n_layers; ++l) {
    put_u64(b, (uint64_t)numel[l]);
    put_u32(b, (uint32_t)k_of((uint64_t)numel[l], ppm));
    put_u32(b, 0);
  }
  for (uint32_t it = 0; it < n_iters; ++it) {
    put_u64(b, first_iter + it);
    for (int i = 0; i < 3; ++i) put_f32(b, scalars[3 * it + i]);
    for (int i = 0; i < 3; ++i) put_u32(b, 0);
    const uint32_t* blk = blocks + (uint64_t)it * 2 * K;
    for (uint64_t e = 0; e < 2 * K; ++e) put_u32(b, blk[e]);
  }
  put_u32(b, crc32c_bitwise(b.data(), b.size()));
  if (b.size() > cap) return E_INVALID;
  std::memcpy(out, b.data(), b.size());
  return OK;
}

// .ldf full checkpoint C^F (Alg. 1 line 15 Save(M_t)), rank r's
// shard [floor(r*Psi/N), floor((r+1)*Psi/N)) of p, m, v (3 Psi total).
int64_t lowdiff_ref_full_bytes(uint64_t psi, uint32_t rank, uint32_t world) {
  const uint64_t b = psi * rank / world, e = psi * (rank + 1) / world;
  return 64 + 32 + 12 * (int64_t)(e - b) + 4;
}

int lowdiff_ref_full_serialize(uint32_t rank, uint32_t world, uint64_t iteration, uint64_t psi,
                               uint32_t optim, uint32_t flags, const float* consts5,
                               const float* p, const float* m, const float* v,
                               uint8_t* out, uint64_t cap) {
  const uint64_t sb = psi * rank / world, se = psi * (rank + 1) / world;
  std::vector<uint8_t> b;
  b.push_back('L'); b.push_back('D'); b.push_back('F'); b.push_back('1');
  put_u16(b, 1); put_u16(b, (uint16_t)flags);
  put_u32(b, rank); put_u32(b, world);
  put_u64(b, iteration);
  put_u64(b, psi); put_u64(b, sb); put_u64(b, se);
  put_u32(b, optim); put_u32(b, 0);
  put_u64(b, 0);
  for (int i = 0; i < 5; ++i) put_f32(b, consts5[i]);
  for (int i = 0; i < 3; ++i) put_u32(b, 0);
  const float* arrs[3] = {p, m, v};
  for (int a = 0; a < 3; ++a)
    for (uint64_t j = sb; j < se; ++j) put_f32(b, arrs[a] ? arrs[a][j] : 0.0f);
  put_u32(b, crc32c_bitwise(b.data(), b.size()));
  if (b.size() > cap) return E_INVALID;
  std::memcpy(out, b.data(), b.size());
  return OK;
}

// --------------------------------------------------------------------------
// recover: Alg. 1 recovery process, Eq. 2,
// with the iteration reading of DESIGN.md R-14: block t turns S_{t-1} into
// S_t; Full@F stores S_F; recover(target) applies blocks F+1..target.
//  1. F = latest iteration <= target with all N .ldf shards present; every
//     shard's CRC and header must verify (else E_CORRUPT).  None -> E_GAP.
//  2. for t = F+1..target every rank must have block t in some .ldb file
//     (a file with a larger first_iter wins) else E_GAP; used files must
//     verify (else E_CORRUPT).  target = -1: the largest such t.
//  3. state = concatenated shards; for t in order: G_t = exchange of the N
//     rank blocks (rank order); apply SGD or Adam with block t's scalars.
// --------------------------------------------------------------------------
int lowdiff_ref_recover(const char* dir, uint32_t world, int n_layers, const int64_t* numel,
                        uint32_t ppm, int64_t target, float* p, float* m, float* v,
                        int64_t* recovered) {
  if (!fp_env_ok()) return E_FPENV;
  uint64_t psi = 0, K = 0;
  for (int l = 0; l < n_layers; ++l) { psi += (uint64_t)numel[l]; K += k_of((uint64_t)numel[l], ppm); }
  // scan the directory: ld_full_r{rank:03}_{iter:012}.ldf, ld_diff_r{rank:03}_{first:012}.ldb
  std::map<int64_t, std::map<uint32_t, std::string>> fulls;   // iter -> rank -> path
  std::vector<std::map<int64_t, std::string>> diffs(world);    // rank -> first -> path
  DIR* d = opendir(dir);
  if (!d) return E_IO;
  while (struct dirent* de = readdir(d)) {
    std::string name = de->d_name;
    unsigned r = 0; unsigned long long it = 0; char tail[16] = {0};
    if (name.size() == 29 && std::sscanf(name.c_str(), "ld_full_r%3u_%12llu.%3s", &r, &it, tail) == 3 &&
        std::string(tail) == "ldf" && r < world)
      fulls[(int64_t)it][r] = std::string(dir) + "/" + name;
    if (name.size() == 29 && std::sscanf(name.c_str(), "ld_diff_r%3u_%12llu.%3s", &r, &it, tail) == 3 &&
        std::string(tail) == "ldb" && r < world)
      diffs[r][(int64_t)it] = std::string(dir) + "/" + name;
  }
  closedir(d);

  // 1. the full checkpoint
  int64_t F = -1;
  for (auto it = fulls.rbegin(); it != fulls.rend(); ++it) {
    if (target >= 0 && it->first > target) continue;
    if (it->second.size() == world) { F = it->first; break; }
  }
  if (F < 0) return E_GAP;
  uint32_t optim = 0;
  for (uint32_t r = 0; r < world; ++r) {
    std::vector<uint8_t> buf;
    if (!read_file(fulls[F][r], buf)) return E_IO;
    const uint64_t sb = psi * r / world, se = psi * (r + 1) / world, S = se - sb;
    if (buf.size() != 64 + 32 + 12 * S + 4) return E_CORRUPT;
    if (std::memcmp(buf.data(), "LDF1", 4) != 0) return E_CORRUPT;
    if (crc32c_bitwise(buf.data(), buf.size() - 4) != get_u32(buf.data() + buf.size() - 4)) return E_CORRUPT;
    if (get_u32(buf.data() + 8) != r || get_u32(buf.data() + 12) != world ||
        (int64_t)get_u64(buf.data() + 16) != F || get_u64(buf.data() + 24) != psi ||
        get_u64(buf.data() + 32) != sb || get_u64(buf.data() + 40) != se)
      return E_CORRUPT;
    optim = get_u32(buf.data() + 48);
    const uint8_t* q = buf.data() + 96;
    for (uint64_t j = 0; j < S; ++j) p[sb + j] = get_f32(q + 4 * j);
    for (uint64_t j = 0; j < S; ++j) if (m) m[sb + j] = get_f32(q + 4 * (S + j));
    for (uint64_t j = 0; j < S; ++j) if (v) v[sb + j] = get_f32(q + 4 * (2 * S + j));
  }

  // 2. the differential chain: for each rank, iteration -> (path, block number)
  std::vector<std::map<int64_t, std::pair<std::string, uint32_t>>> where(world);
  std::map<std::string, std::vector<uint8_t>> loaded;
  for (uint32_t r = 0; r < world; ++r) {
    for (auto& fe : diffs[r]) {   // ascending first_iter: later files override earlier ones
      std::vector<uint8_t> hdr;
      if (!read_file(fe.second, hdr) || hdr.size() < 64) return E_CORRUPT;
      const uint32_t n_iters = get_u32(hdr.data() + 24);
      for (uint32_t i = 0; i < n_iters; ++i) where[r][fe.first + i] = {fe.second, i};
    }
  }
  int64_t last = F;
  while (true) {
    const int64_t t = last + 1;
    if (target >= 0 && t > target) break;
    bool all = true;
    for (uint32_t r = 0; r < world; ++r) all = all && where[r].count(t);
    if (!all) break;
    last = t;
  }
  if (target >= 0 && last < target) return E_GAP;

  // 3. replay blocks F+1..last
  std::vector<uint32_t> gathered((uint64_t)world * 2 * K);
  std::vector<float> G(psi);
  for (int64_t t = F + 1; t <= last; ++t) {
    float scal[3] = {0, 0, 0};
    float consts[5] = {0, 0, 0, 0, 0};
    uint32_t flags = 0;
    for (uint32_t r = 0; r < world; ++r) {
      const std::string& path = where[r][t].first;
      if (!loaded.count(path)) {
        std::vector<uint8_t> buf;
        if (!read_file(path, buf)) return E_IO;
        if (buf.size() < 100 || std::memcmp(buf.data(), "LDB1", 4) != 0) return E_CORRUPT;
        const uint32_t n_iters = get_u32(buf.data() + 24);
        if ((int64_t)buf.size() != lowdiff_ref_batch_bytes(n_layers, K, (int)n_iters)) return E_CORRUPT;
        if (crc32c_bitwise(buf.data(), buf.size() - 4) != get_u32(buf.data() + buf.size() - 4)) return E_CORRUPT;
        if (get_u32(buf.data() + 8) != r || get_u32(buf.data() + 12) != world ||
            get_u32(buf.data() + 28) != (uint32_t)n_layers || get_u64(buf.data() + 32) != psi ||
            get_u64(buf.data() + 40) != K || get_u32(buf.data() + 48) != ppm ||
            get_u32(buf.data() + 52) != optim)
          return E_CORRUPT;
        loaded[path] = std::move(buf);
      }
      const std::vector<uint8_t>& buf = loaded[path];
      const uint8_t* blk = buf.data() + 96 + 16 * (uint64_t)n_layers +
                           (uint64_t)where[r][t].second * (32 + 8 * K);
      if ((int64_t)get_u64(blk) != t) return E_CORRUPT;
      float s3[3] = {get_f32(blk + 8), get_f32(blk + 12), get_f32(blk + 16)};
      if (r == 0) {
        std::memcpy(scal, s3, sizeof scal);
        for (int i = 0; i < 5; ++i) consts[i] = get_f32(buf.data() + 64 + 4 * i);
        flags = get_u16(buf.data() + 6);
      } else if (std::memcmp(scal, s3, sizeof scal) != 0) {
        return E_CORRUPT;
      }
      for (uint64_t e = 0; e < 2 * K; ++e) gathered[(uint64_t)r * 2 * K + e] = get_u32(blk + 32 + 4 * e);
    }
    int st = lowdiff_ref_exchange((int)world, K, psi, gathered.data(), (flags >> 1) & 1, G.data());
    if (st) return st;
    if (optim == 1) st = lowdiff_ref_adam_step(psi, G.data(), consts, scal, p, m, v);
    else st = lowdiff_ref_sgd_step(psi, G.data(), scal[0], p);
    if (st) return st;
  }
  *recovered = last;
  return OK;
}

// --------------------------------------------------------------------------
// Union-compacted differential C^U_t (R-29).  After
// Sync (Alg. 1 line 5) the checkpointing process receives the
// synchronised compressed gradient G~_t (Q.put, line 6) and may
// keep it as a dictionary ("dictionary accumulation"):
//   U_t = { j : j is an index of some rank's block of iteration t }
//   C^U_t = [(j, G_t[j]) for j in U_t, ascending],  G_t = Comp^-1(G~_t)
// written here exactly in that order: (1) the dense G_t of the exchange above,
// (2) a membership flag per index from every rank's index list, (3) the
// members inside [lo, hi) in ascending order with their G_t value.  Rank r
// stores the members in its parameter shard [floor(r Psi/N), floor((r+1) Psi/N)).
// --------------------------------------------------------------------------
int lowdiff_ref_union_compact(int world, uint64_t K, uint64_t psi, const uint32_t* gathered, int mean,
                              uint64_t lo, uint64_t hi, uint32_t* out_idx, uint32_t* out_val, uint64_t cap,
                              uint64_t* count) {
  if (!fp_env_ok()) return E_FPENV;
  if (world < 1 || !gathered || !count || lo > hi || hi > psi) return E_INVALID;
  std::vector<float> G(psi);
  int st = lowdiff_ref_exchange(world, K, psi, gathered, mean, G.data());   // (1)
  if (st) return st;
  std::vector<char> member(psi, 0);                                         // (2)
  for (int r = 0; r < world; ++r)
    for (uint64_t e = 0; e < K; ++e) member[gathered[(uint64_t)r * 2 * K + e]] = 1;
  uint64_t n = 0;                                                           // (3)
  for (uint64_t j = lo; j < hi; ++j) {
    if (!member[j]) continue;
    if (n < cap) {
      out_idx[n] = (uint32_t)j;
      out_val[n] = float_bits(G[j]);
    }
    ++n;
  }
  *count = n;
  return n <= cap ? OK : E_DIM;
}

// .ldu file: b consecutive union-compacted differentials of rank r's shard
//   header 80 B: "LDU1" | u16 version=1 | u16 flags (bit0 EF, bit1 mean) | u32 rank |
//     u32 world | u64 first_iter (16) | u32 n_iters | u32 n_layers | u64 Psi (32) | u64 K |
//     u32 ppm (48) | u32 optim | u64 shard_begin (56) | u64 shard_end (64) | u64 0 (72)
//   hyper 32 B | layer table L x {u64 numel, u32 k, u32 0} |
//   n_iters x ({u64 iteration, f32 lr, f32 bc1_inv, f32 bc2_inv, u32 count, u64 0} +
//              idx u32[count] + val u32[count]) | u32 CRC-32C of all preceding bytes
int64_t lowdiff_ref_union_bytes(int n_layers, int n_iters, const uint64_t* counts) {
  int64_t b = 80 + 32 + 16 * (int64_t)n_layers + 4;
  for (int i = 0; i < n_iters; ++i) b += 32 + 8 * (int64_t)counts[i];
  return b;
}

int lowdiff_ref_union_serialize(uint32_t rank, uint32_t world, uint64_t first_iter, uint32_t n_iters,
                                int n_layers, const int64_t* numel, uint32_t ppm, uint32_t optim,
                                uint32_t flags, const float* consts5, const float* scalars /* n x 3 */,
                                const uint64_t* counts /* n */, const uint32_t* entries /* per iteration:
                                idx[count] then val[count], concatenated */, uint8_t* out, uint64_t cap) {
  uint64_t psi = 0, K = 0;
  for (int l = 0; l < n_layers; ++l) { psi += (uint64_t)numel[l]; K += k_of((uint64_t)numel[l], ppm); }
  std::vector<uint8_t> b;
  b.push_back('L'); b.push_back('D'); b.push_back('U'); b.push_back('1');
  put_u16(b, 1); put_u16(b, (uint16_t)flags);
  put_u32(b, rank); put_u32(b, world);
  put_u64(b, first_iter);
  put_u32(b, n_iters); put_u32(b, (uint32_t)n_layers);
  put_u64(b, psi); put_u64(b, K);
  put_u32(b, ppm); put_u32(b, optim);
  put_u64(b, psi * rank / world);
  put_u64(b, psi * (rank + 1) / world);
  put_u64(b, 0);
  for (int i = 0; i < 5; ++i) put_f32(b, consts5[i]);
  for (int i = 0; i < 3; ++i) put_u32(b, 0);
  for (int l = 0; l < n_layers; ++l) {
    put_u64(b, (uint64_t)numel[l]);
    put_u32(b, (uint32_t)k_of((uint64_t)numel[l], ppm));
    put_u32(b, 0);
  }
  const uint32_t* q = entries;
  for (uint32_t it = 0; it < n_iters; ++it) {
    put_u64(b, first_iter + it);
    for (int i = 0; i < 3; ++i) put_f32(b, scalars[3 * it + i]);
    put_u32(b, (uint32_t)counts[it]);
    put_u64(b, 0);
    for (uint64_t e = 0; e < 2 * counts[it]; ++e) put_u32(b, q[e]);
    q += 2 * counts[it];
  }
  put_u32(b, crc32c_bitwise(b.data(), b.size()));
  if (b.size() > cap) return E_INVALID;
  std::memcpy(out, b.data(), b.size());
  return OK;
}

// --------------------------------------------------------------------------
// Accumulated batch mode (R-30).  PAPER.md:270: writes of compressed
// gradients are batched "with the help of the widely-used gradient accumulation
// technique ... where the gradients of the same shape and size can be
// accumulated"; the CPU batching operation "mainly involves the
// addition of compressed gradients"; "checkpoints are aggregated
// (tensor addition or dictionary accumulation)".  Tensor addition of the b
// dictionaries C^U_t of one batch, written out as a dictionary in iteration
// order:
//   A = {}
//   for t in batch (ascending), for (j, x) in C^U_t:  A[j] = (j in A ? A[j] : +0) + x
// The accumulated file holds A and the scalars of the batch's last iteration;
// recovery applies it as ONE optimizer step (gradient-accumulation semantics).
// In exact arithmetic this equals the b steps only for SGD at a constant lr.
// --------------------------------------------------------------------------
int lowdiff_ref_accumulate(uint32_t n_iters, const uint64_t* counts, const uint32_t* entries /* per iteration
                           idx[count] then val[count], concatenated */, uint32_t* out_idx, uint32_t* out_val,
                           uint64_t cap, uint64_t* count) {
  if (!fp_env_ok()) return E_FPENV;
  if (!count || (n_iters && (!counts || !entries))) return E_INVALID;
  std::map<uint32_t, float> A;
  const uint32_t* q = entries;
  for (uint32_t it = 0; it < n_iters; ++it) {
    const uint64_t n = counts[it];
    for (uint64_t e = 0; e < n; ++e) {
      const uint32_t j = q[e];
      const float x = bits_float(q[n + e]);
      auto f = A.find(j);
      const float before = f == A.end() ? 0.0f : f->second;
      A[j] = before + x;
    }
    q += 2 * n;
  }
  uint64_t n = 0;
  for (const auto& kv : A) {
    if (n < cap) {
      out_idx[n] = kv.first;
      out_val[n] = float_bits(kv.second);
    }
    ++n;
  }
  *count = n;
  return n <= cap ? OK : E_DIM;
}

// Accumulated .ldu: the .ldu header with flags bit 2 (ACCUMULATED) and n_iters = b (the iterations
// the batch covers, first_iter .. first_iter + b - 1), then ONE block {u64 first_iter + b - 1, the
// scalars of that last iteration, u32 count, u64 0} + idx u32[count] + val u32[count], then CRC-32C.
int lowdiff_ref_accum_serialize(uint32_t rank, uint32_t world, uint64_t first_iter, uint32_t n_iters,
                                int n_layers, const int64_t* numel, uint32_t ppm, uint32_t optim, uint32_t flags,
                                const float* consts5, const float* last_scalars3, uint64_t count,
                                const uint32_t* idx_val /* idx[count] then val[count] */, uint8_t* out,
                                uint64_t cap) {
  if (n_iters < 1) return E_INVALID;
  uint64_t psi = 0, K = 0;
  for (int l = 0; l < n_layers; ++l) { psi += (uint64_t)numel[l]; K += k_of((uint64_t)numel[l], ppm); }
  std::vector<uint8_t> b;
  b.push_back('L'); b.push_back('D'); b.push_back('U'); b.push_back('1');
  put_u16(b, 1); put_u16(b, (uint16_t)(flags | 4u));
  put_u32(b, rank); put_u32(b, world);
  put_u64(b, first_iter);
  put_u32(b, n_iters); put_u32(b, (uint32_t)n_layers);
  put_u64(b, psi); put_u64(b, K);
  put_u32(b, ppm); put_u32(b, optim);
  put_u64(b, psi * rank / world);
  put_u64(b, psi * (rank + 1) / world);
  put_u64(b, 0);
  for (int i = 0; i < 5; ++i) put_f32(b, consts5[i]);
  for (int i = 0; i < 3; ++i) put_u32(b, 0);
  for (int l = 0; l < n_layers; ++l) {
    put_u64(b, (uint64_t)numel[l]);
    put_u32(b, (uint32_t)k_of((uint64_t)numel[l], ppm));
    put_u32(b, 0);
  }
  put_u64(b, first_iter + n_iters - 1);
  for (int i = 0; i < 3; ++i) put_f32(b, last_scalars3[i]);
  put_u32(b, (uint32_t)count);
  put_u64(b, 0);
  for (uint64_t e = 0; e < 2 * count; ++e) put_u32(b, idx_val[e]);
  put_u32(b, crc32c_bitwise(b.data(), b.size()));
  if (b.size() > cap) return E_INVALID;
  std::memcpy(out, b.data(), b.size());
  return OK;
}

// Recovery from union-compacted differentials (Alg. 1 recovery, with C^U_t in
// place of the gathered blocks): the same chain rules as lowdiff_ref_recover (.ldf shards of the
// latest complete full F <= target; for t = F+1..target every rank's .ldu must hold iteration t,
// later files winning), then per iteration G_t[j] = the stored value for every stored j (the ranks'
// shards are disjoint), +0.0f elsewhere, and the optimizer step with the block's scalars.  An
// accumulated file (flags bit 2, R-30) is one replay unit covering its n_iters iterations: one
// optimizer step with G[j] = the accumulated value and the stored scalars of its last iteration; a
// target inside such a batch is not reachable (E_GAP).
int lowdiff_ref_recover_union(const char* dir, uint32_t world, int n_layers, const int64_t* numel,
                              uint32_t ppm, int64_t target, float* p, float* m, float* v,
                              int64_t* recovered) {
  if (!fp_env_ok()) return E_FPENV;
  uint64_t psi = 0, K = 0;
  for (int l = 0; l < n_layers; ++l) { psi += (uint64_t)numel[l]; K += k_of((uint64_t)numel[l], ppm); }
  std::map<int64_t, std::map<uint32_t, std::string>> fulls;
  std::vector<std::map<int64_t, std::string>> diffs(world);
  DIR* d = opendir(dir);
  if (!d) return E_IO;
  while (struct dirent* de = readdir(d)) {
    std::string name = de->d_name;
    unsigned r = 0; unsigned long long it = 0; char tail[16] = {0};
    if (name.size() == 29 && std::sscanf(name.c_str(), "ld_full_r%3u_%12llu.%3s", &r, &it, tail) == 3 &&
        std::string(tail) == "ldf" && r < world)
      fulls[(int64_t)it][r] = std::string(dir) + "/" + name;
    if (name.size() == 30 && std::sscanf(name.c_str(), "ld_union_r%3u_%12llu.%3s", &r, &it, tail) == 3 &&
        std::string(tail) == "ldu" && r < world)
      diffs[r][(int64_t)it] = std::string(dir) + "/" + name;
  }
  closedir(d);
  int64_t F = -1;
  for (auto it = fulls.rbegin(); it != fulls.rend(); ++it) {
    if (target >= 0 && it->first > target) continue;
    if (it->second.size() == world) { F = it->first; break; }
  }
  if (F < 0) return E_GAP;
  uint32_t optim = 0;
  for (uint32_t r = 0; r < world; ++r) {
    std::vector<uint8_t> buf;
    if (!read_file(fulls[F][r], buf)) return E_IO;
    const uint64_t sb = psi * r / world, se = psi * (r + 1) / world, S = se - sb;
    if (buf.size() != 64 + 32 + 12 * S + 4) return E_CORRUPT;
    if (std::memcmp(buf.data(), "LDF1", 4) != 0) return E_CORRUPT;
    if (crc32c_bitwise(buf.data(), buf.size() - 4) != get_u32(buf.data() + buf.size() - 4)) return E_CORRUPT;
    if (get_u32(buf.data() + 8) != r || get_u32(buf.data() + 12) != world ||
        (int64_t)get_u64(buf.data() + 16) != F || get_u64(buf.data() + 24) != psi ||
        get_u64(buf.data() + 32) != sb || get_u64(buf.data() + 40) != se)
      return E_CORRUPT;
    optim = get_u32(buf.data() + 48);
    const uint8_t* q = buf.data() + 96;
    for (uint64_t j = 0; j < S; ++j) p[sb + j] = get_f32(q + 4 * j);
    for (uint64_t j = 0; j < S; ++j) if (m) m[sb + j] = get_f32(q + 4 * (S + j));
    for (uint64_t j = 0; j < S; ++j) if (v) v[sb + j] = get_f32(q + 4 * (2 * S + j));
  }
  // which file (and byte offset) holds the replay unit starting at iteration t of rank r, and how
  // many iterations it covers (1; b for an accumulated batch); every used file is verified
  struct Unit { std::string path; uint64_t off; int64_t span; };
  std::vector<std::map<int64_t, Unit>> where(world);
  std::map<std::string, std::vector<uint8_t>> loaded;
  for (uint32_t r = 0; r < world; ++r) {
    for (auto& fe : diffs[r]) {   // ascending first_iter: later files override earlier ones
      std::vector<uint8_t> buf;
      if (!read_file(fe.second, buf) || buf.size() < 116) return E_CORRUPT;
      if (std::memcmp(buf.data(), "LDU1", 4) != 0) return E_CORRUPT;
      if (crc32c_bitwise(buf.data(), buf.size() - 4) != get_u32(buf.data() + buf.size() - 4)) return E_CORRUPT;
      if (get_u32(buf.data() + 8) != r || get_u32(buf.data() + 12) != world ||
          get_u32(buf.data() + 28) != (uint32_t)n_layers || get_u64(buf.data() + 32) != psi ||
          get_u64(buf.data() + 40) != K || get_u32(buf.data() + 48) != ppm || get_u32(buf.data() + 52) != optim ||
          get_u64(buf.data() + 56) != psi * r / world || get_u64(buf.data() + 64) != psi * (r + 1) / world)
        return E_CORRUPT;
      const uint32_t n_iters = get_u32(buf.data() + 24);
      const bool accumulated = (get_u16(buf.data() + 6) & 4u) != 0;
      uint64_t off = 112 + 16 * (uint64_t)n_layers;
      if (accumulated) {   // one block for iterations fe.first .. fe.first + n_iters - 1
        if (n_iters < 1 || off + 32 > buf.size() - 4) return E_CORRUPT;
        const uint64_t cnt = get_u32(buf.data() + off + 20);
        if ((int64_t)get_u64(buf.data() + off) != fe.first + n_iters - 1) return E_CORRUPT;
        where[r][fe.first] = {fe.second, off, (int64_t)n_iters};
        off += 32 + 8 * cnt;
      }
      for (uint32_t i = 0; i < n_iters && !accumulated; ++i) {
        if (off + 32 > buf.size() - 4) return E_CORRUPT;
        const uint64_t cnt = get_u32(buf.data() + off + 20);
        if ((int64_t)get_u64(buf.data() + off) != fe.first + i) return E_CORRUPT;
        where[r][fe.first + i] = {fe.second, off, 1};
        off += 32 + 8 * cnt;
      }
      if (off != buf.size() - 4) return E_CORRUPT;
      loaded[fe.second] = std::move(buf);
    }
  }
  // the chain: units F+1 .., every rank holding a unit that starts there and covers the same
  // iterations; an accumulated batch is recovered whole or not at all
  int64_t last = F;
  std::vector<int64_t> starts;
  while (true) {
    const int64_t t = last + 1;
    bool all = true;
    int64_t span = 0;
    for (uint32_t r = 0; r < world && all; ++r) {
      all = where[r].count(t) > 0;
      if (all && r == 0) span = where[r][t].span;
      else if (all && where[r][t].span != span) return E_CORRUPT;
    }
    if (!all || (target >= 0 && t + span - 1 > target)) break;
    starts.push_back(t);
    last = t + span - 1;
  }
  if (target >= 0 && last < target) return E_GAP;
  std::vector<float> G(psi);
  for (int64_t t : starts) {
    float scal[3] = {0, 0, 0};
    float consts[5] = {0, 0, 0, 0, 0};
    std::fill(G.begin(), G.end(), 0.0f);
    for (uint32_t r = 0; r < world; ++r) {
      const std::vector<uint8_t>& buf = loaded[where[r][t].path];
      const uint8_t* blk = buf.data() + where[r][t].off;
      float s3[3] = {get_f32(blk + 8), get_f32(blk + 12), get_f32(blk + 16)};
      if (r == 0) {
        std::memcpy(scal, s3, sizeof scal);
        for (int i = 0; i < 5; ++i) consts[i] = get_f32(buf.data() + 80 + 4 * i);
      } else if (std::memcmp(scal, s3, sizeof scal) != 0) {
        return E_CORRUPT;
      }
      const uint64_t cnt = get_u32(blk + 20);
      const uint64_t sb = psi * r / world, se = psi * (r + 1) / world;
      for (uint64_t e = 0; e < cnt; ++e) {
        const uint32_t j = get_u32(blk + 32 + 4 * e);
        if (j < sb || j >= se) return E_CORRUPT;
        G[j] = get_f32(blk + 32 + 4 * (cnt + e));
      }
    }
    int st = optim == 1 ? lowdiff_ref_adam_step(psi, G.data(), consts, scal, p, m, v)
                        : lowdiff_ref_sgd_step(psi, G.data(), scal[0], p);
    if (st) return st;
  }
  *recovered = last;
  return OK;
}

// --------------------------------------------------------------------------
// Checkpointing configuration, §4.3 "Configuration Modeling", written
// term by term from the itemised list PAPER.md:322-330 (one time unit throughout, R-27):
//   failures            = T / M
//   full-ckpt write     = S / W
//   full checkpoints    = f x T
//   lost work           = N x T/M x b/2
//   merges on average   = 1/2 (1/f x 1/b - 1)
//   recovery time       = N x T/M x (R_F + R_D x merges)
//   steady-state cost   = N x S/W x f x T
//   T_wasted            = recovery time + lost work + steady-state cost        (Eq. 3)
// and the optimum stated by Eq. 5.
// --------------------------------------------------------------------------
double lowdiff_ref_wasted_time(double N, double M, double W, double S, double T, double R_F, double R_D,
                               double f, double b) {
  const double failures = T / M;
  const double full_ckpt_write = S / W;
  const double full_ckpts = f * T;
  const double lost_work = N * failures * (b / 2.0);
  const double merges = 0.5 * (1.0 / f * 1.0 / b - 1.0);
  const double recovery = N * failures * (R_F + R_D * merges);
  const double steady = N * full_ckpt_write * full_ckpts;
  return recovery + lost_work + steady;
}

void lowdiff_ref_optimal_config(double M, double W, double S, double R_D, double* f_star, double* b_star) {
  *f_star = std::cbrt(R_D * W * W / (4.0 * S * S * M * M));
  *b_star = std::cbrt(2.0 * S * R_D * M / W);
}

// --------------------------------------------------------------------------
// Failure-injection simulator (SPEC.md failure-sim module), written as a trace
// followed by a ledger so each step can be read against Eq. 3's itemised model:
//   trace: failures of the N GPUs form a Poisson process of rate N / M over the productive time
//          [0, T) (exponential inter-arrival times of mean M / N, inverse-CDF -log(1 - u)); each
//          failure is "software" with probability sw_fraction.  u comes from splitmix64 over a
//          counter (u_i = top 53 bits of splitmix64(seed + (i+1) * 0x9E3779B97F4A7C15) / 2^53),
//          draws in the order: inter-arrival, kind, inter-arrival, kind, ...
//   ledger per hardware failure at time t: x = t mod (1/f) (time since the last full checkpoint),
//          lost work = x mod b (since the last persisted batch), merges = floor(x / b) persisted
//          batches to replay, recovery = R_F + R_D x merges.
//   ledger per software failure (LowDiff+): recovery = R_S (replica restore), no
//          lost work (the replica is current).
//   steady = N x S/W x floor(f T) full checkpoints; wasted = lost + recovery + steady.
// --------------------------------------------------------------------------
static uint64_t ref_splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double ref_uniform(uint64_t seed, uint64_t i) {
  return (double)(ref_splitmix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull) >> 11) * (1.0 / 9007199254740992.0);
}

void lowdiff_ref_simulate(double N, double M, double W, double S, double T, double R_F, double R_D, double f,
                          double b, double sw_fraction, double R_S, uint64_t seed, int64_t* counts /*[2]*/,
                          double* ledger /*[4]: lost, recovery, steady, wasted*/) {
  // 1. the failure trace
  std::vector<double> times;
  std::vector<int> software;
  uint64_t draw = 0;
  double t = 0.0;
  for (;;) {
    const double u = ref_uniform(seed, draw++);
    t = t + (-std::log1p(-u)) * (M / N);
    const double k = ref_uniform(seed, draw++);
    if (t >= T) break;
    times.push_back(t);
    software.push_back(k < sw_fraction ? 1 : 0);
  }
  // 2. the ledger
  double lost = 0.0, recovery = 0.0;
  int64_t hw = 0;
  for (size_t i = 0; i < times.size(); ++i) {
    if (software[i]) {
      recovery = recovery + R_S;
      continue;
    }
    ++hw;
    const double x = std::fmod(times[i], 1.0 / f);
    lost = lost + std::fmod(x, b);
    recovery = recovery + (R_F + R_D * std::floor(x / b));
  }
  const double steady = N * (S / W) * std::floor(f * T);
  counts[0] = (int64_t)times.size();
  counts[1] = hw;
  ledger[0] = lost;
  ledger[1] = recovery;
  ledger[2] = steady;
  ledger[3] = lost + recovery + steady;
}

}  // extern "C"
