// Helpers shared by the C-ABI implementation files (api.cpp, recover.cpp, union_api.cpp,
// lowdiff_plus.cpp).  Internal to liblowdiff.
#pragma once
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

// NVTX range over a C-ABI call (host timeline: nsys / ncu --nvtx); header-only NVTX v3, a no-op
// unless a tool is attached (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// return a CUDA failure as LOWDIFF_E_CUDA (the context is poisoned); needs `c` in scope
#define CK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
  } while (0)

namespace ld {
namespace api {

int64_t now_ns();
bool aligned16(const void* p);
lowdiff_status fail(lowdiff_ctx* c, lowdiff_status st, const std::string& msg);
lowdiff_status cuda_fail(lowdiff_ctx* c, cudaError_t e, const char* what);
lowdiff_status entry(lowdiff_ctx* c);          // argument/poison check + cudaSetDevice
lowdiff_status take_deferred(lowdiff_ctx* c);
void set_deferred(lowdiff_ctx* c, lowdiff_status st, const std::string& msg);
lowdiff_status validate_cfg(const lowdiff_config* cfg);
lowdiff_status write_ldf(const lowdiff_config& cfg, const std::string& dir, int64_t iteration, uint64_t psi,
                         uint64_t sb, uint64_t se, const float* body, std::string* err);

// the differential chain of a checkpoint directory (recovery)
struct Chain {
  int64_t F = -1, last = -1;
  std::vector<std::string> full_paths;                                      // [world]
  std::vector<std::map<int64_t, std::pair<std::string, uint32_t>>> where;   // rank -> t -> (file, block)
};
bool parse_name(const char* name, const char* kind, const char* ext, unsigned* rank, long long* it);
bool read_all(const std::string& path, std::vector<uint8_t>& out);
bool read_head(const std::string& path, uint8_t* buf, size_t n, size_t* fsize);
template <class T> T rd(const uint8_t* p) { T v; std::memcpy(&v, p, sizeof v); return v; }
lowdiff_status scan_chain(const lowdiff_config& cfg, int64_t target, Chain* ch, std::string* err);
// remove / truncate this rank's files holding iterations >= t (kinds: bit0 .ldb, bit1 .ldu, bit2 .ldf)
lowdiff_status retire_from(const lowdiff_config& cfg, int64_t t, int kinds, std::string* err);

// recover.cpp
lowdiff_status bcast_shards(lowdiff_ctx* c, float* dst[3], cudaStream_t s);
lowdiff_status load_full_shards(lowdiff_ctx* c, const std::vector<std::string>& paths, int64_t F, bool sharded,
                                float* p, float* m, float* v, uint32_t* optim, float* consts, uint16_t* flags);
// union_api.cpp / lowdiff_plus.cpp: drain and stop the worker threads (lowdiff_sync / destroy)
void union_drain(lowdiff_ctx* c);
void union_shutdown(lowdiff_ctx* c);
void replica_drain(lowdiff_ctx* c);
void replica_shutdown(lowdiff_ctx* c);

}  // namespace api
}  // namespace ld
