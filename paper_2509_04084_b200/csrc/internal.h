// Internal declarations of liblowdiff (B200 / sm_100a).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lowdiff.h"

namespace ld {

// ---------------------------------------------------------------- compress plan
// Layers with n <= kSmallMax are selected by one CTA entirely in shared memory.
// Larger layers are cut into chunks of kChunk elements whose boundaries are
// 4-element aligned in the flat buffer (so every 16-byte slot lies in one chunk).
constexpr int kChunk = 16384;          // elements per chunk (64 KB of fp32)
constexpr int kSeg = 1024;             // candidate segment: the elements one scan warp streams
constexpr int kSegsPerChunk = kChunk / kSeg;   // 16
constexpr int kScanThreads = 512;      // threads per chunk CTA: 8 float4 slots each
constexpr int kSmallMax = 4096;        // small-layer bound: one CTA selects it in shared memory
                                       // (larger layers go through the parallel chunk path)
constexpr int kSmallThreads = 512;
constexpr int kMergeTileShift = 13;
constexpr int kMergeTile = 1 << kMergeTileShift;     // merge tile (elements per CTA)
constexpr int kReplayTileShift = 11;
constexpr int kReplayTile = 1 << kReplayTileShift;   // replay tile (elements per CTA)
#ifndef LD_REPLAY_THREADS
#define LD_REPLAY_THREADS 128   // x 4 float4 slots = 16 elements per thread (measured best, B200)
#endif
constexpr int kReplayThreads = LD_REPLAY_THREADS;
constexpr int kReplaySlots = kReplayTile / (4 * kReplayThreads);   // float4 slots per thread
constexpr uint32_t kNoThreshold = 0xFFFFFFFFu;

// per-large-layer selection state (device)
struct LayerSel {
  uint32_t prefix;   // key bits fixed by the digits done so far
  uint32_t kleft;    // entries still to take among those matching prefix
  uint32_t total;    // candidate count
  uint32_t refill;   // 1: speculative band too narrow, the layer was refilled (histogram + rescan)
  uint32_t next_thr; // speculative band for the next call (drift-led)
  float band;        // band width as a multiple of k_l in this call's distribution (adaptive; 0 = unset)
  uint32_t next_safe;// the same band without the drift lead
  float alpha;       // share of the last drift of T the next band leads by (adaptive)
  uint32_t drift;    // this layer's last upward drift of T (key units; 0 = none or downward)
};

struct DevPlan {
  // layers
  int32_t n_layers;
  int32_t n_large, n_small;
  const uint64_t* layer_off;     // [L+1]
  const uint32_t* layer_k;       // [L]
  const uint64_t* layer_koff;    // [L]
  const int32_t* small_layers;   // [n_small] layer ids
  const int32_t* large_layers;   // [n_large] layer ids
  const int32_t* large_chunk0;   // [n_large+1] first chunk of each large layer
  // chunks (large layers only)
  int32_t n_chunks;
  const int32_t* chunk_slot;     // [n_chunks] index into large_layers
  const uint64_t* chunk_base;    // [n_chunks] first element (4-aligned) of the chunk's slot grid
  const uint64_t* chunk_lo;      // [n_chunks] first element that belongs to the chunk
  const uint64_t* chunk_hi;      // [n_chunks] one past the last element
  // scratch
  int32_t cs;                    // candidate capacity of a segment (compress_seg_capacity)
  uint64_t* cand;                // [n_chunks * 16] segment slots of cs candidates (acc bits << 32 | index);
                                 //   chunk prep compacts each chunk's stored lists in place (chunk list)
  uint32_t* seg_count;           // [n_chunks * 16] candidates of the segment (| kDirect: not stored)
  uint32_t* chunk_count;         // [n_chunks] length of the chunk's compacted (stored) list
  uint32_t* chunk_dm;            // [n_chunks] its DIRECT segments (bit mask)
  uint32_t* layer_total;         // [n_large] candidates admitted per large layer (this call)
  uint32_t* hist;                // [n_large * (2048 + 2048 + 512)]
  LayerSel* sel;                 // [n_large]
  uint32_t* thr;                 // [n_large] speculative threshold key (persistent across calls)
  uint32_t* thr_used;            // [n_large] threshold this call's candidates were taken with
  // lazy residual zeroing: the previous call's selection of a large layer is
  // {key(r) > sel_T} U {key(r) == sel_T and index < sel_cut}; the next scan zeroes it on the fly
  uint32_t* sel_T;               // [n_large] previous call's exact k-th key
  uint32_t* sel_cut;             // [n_large] one past the global index of the last tie it took
  uint32_t* refill_list;         // [n_chunks] chunks of the missed layers (histogram pass + rescan)
  uint32_t* trace;               // [n_large] this call's path per layer: 0 hit, 1 refill
  unsigned long long* chunk_state;  // [n_chunks] count_emit look-back: status | eq_incl | gt_incl
  uint32_t* counters;            // [0] chunks queued for a refill, [1] spec hits, [2] spec misses,
                                 // [3] candidates of hit layers, [4] unused,
                                 // [5] DIRECT segments of the scan and the rescan (more than cs candidates),
                                 // [6] grid-barrier counter of the refill kernel
  uint32_t* err;                 // [0] non-finite flag, [1] first bad layer
};

// ---------------------------------------------------------------- context
struct ProfRec { const char* name; cudaEvent_t a, b; };

struct Slot {
  uint8_t* host;        // 32-byte block header + 8K payload
  uint32_t* err_host;   // device error flags copied next to the payload
  cudaEvent_t done;
  int64_t iteration;
};

// work item of the LowDiff+ replica worker: 0 = initial copy landed, 1 = apply the snapshotted
// gradient of `iteration`, 2 = persist the replica as it stands after the preceding items
struct RepJob { int kind; int64_t iteration; lowdiff_step_scalars sc; };
struct UJob { int64_t iteration; lowdiff_step_scalars sc; int buf; bool accumulate; };
// pinned chunks + streams of the recovery loader (files.cpp stream_to_device), kept per context
struct Staging {
  static constexpr uint64_t kChunk = 64ull << 20;
  std::vector<uint8_t*> bufs;
  std::vector<cudaStream_t> streams;
};
// a captured CUDA graph of one call's kernels, keyed by the call kind and its buffers
struct GraphEntry {
  int kind; const void *a, *b, *c; int flag; uint64_t gen;
  cudaGraphExec_t exec; int64_t launches; uint64_t last_use;
};

// peer-memory exchange (peer.cu): flag words per rank = ready[n_slots] | done[n_slots][kPeerMaxWorld]
// | error counter
constexpr int kPeerMaxWorld = 8;
__host__ __device__ constexpr int peer_err_word(int n_slots) { return n_slots + n_slots * kPeerMaxWorld; }
struct PeerTable {
  int world, self, slot, n_slots;
  unsigned long long epoch;
  const uint32_t* send[kPeerMaxWorld];     // rank q's send block in `slot` (u32[2K])
  const uint32_t* start[kPeerMaxWorld];    // rank q's merge tile-start table for that block
  unsigned long long* flags[kPeerMaxWorld];
};
cudaError_t launch_peer_ready(unsigned long long* own_flags, int slot, unsigned long long epoch, cudaStream_t s);
cudaError_t launch_peer_wait_done(unsigned long long* own_flags, int n_slots, int slot, int world,
                                  unsigned long long epoch, cudaStream_t s);
cudaError_t launch_peer_merge(const PeerTable& T, uint64_t K, int64_t psi, bool mean, float* dense, cudaStream_t s);
// the optimizer constants and one step's scalars of lowdiff_exchange_peer_update
struct PeerOpt { float b1, c1, b2, c2, eps, lr, r1, r2; };
cudaError_t launch_peer_update(const PeerTable& T, uint64_t K, int64_t psi, bool mean, bool adam, const PeerOpt& o,
                               float* p, float* m, float* v, cudaStream_t s);
// merge_replay.cu: the merge's tile-start table of one block (n_tiles + 1 entries)
cudaError_t launch_tile_start(const uint32_t* block, uint64_t K, int64_t psi, uint32_t* start, cudaStream_t s);

// replica.cpp: host optimizer steps over [0, n) split over `threads` (bitwise = the device replay)
void host_adam(int64_t n, const float* G, const lowdiff_adam_consts& a, const lowdiff_step_scalars& s, float* p,
               float* m, float* v, int threads);
void host_sgd(int64_t n, const float* G, float lr, float* p, int threads);

}  // namespace ld

struct lowdiff_ctx {
  // configuration
  lowdiff_config cfg;
  std::vector<int64_t> numel;
  std::string ckpt_dir;
  int64_t psi = 0, K = 0;
  std::vector<uint64_t> off, koff;
  std::vector<uint32_t> k;
  int device = 0;
  // device plan + buffers
  ld::DevPlan plan{};
  std::vector<void*> dev_allocs;
  size_t plan_bytes = 0;              // device memory of the plan + compress scratch (dev_allocs)
  // streams / events
  cudaStream_t side = nullptr;       // D2H copies
  cudaStream_t aux = nullptr;        // small-layer compress, forked from the caller's stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_tmp = nullptr;
  cudaEvent_t ev_side_all = nullptr; // lowdiff_wait_persist
  cudaEvent_t last_d2h = nullptr;    // unused (kept for ABI-stable layout of the struct)
  std::vector<std::pair<const void*, int>> d2h_src;   // send buffer -> ring slot of its latest D2H (WAR)
  std::atomic<uint32_t> err_seen{0};  // non-finite events already reported
  const float* lazy_residual = nullptr;   // residual whose last selection is not yet zeroed (large layers)
  // NCCL
  ncclComm_t comm = nullptr;
  // status
  lowdiff_status poisoned = LOWDIFF_OK;
  lowdiff_status deferred = LOWDIFF_OK;
  std::string last_error;
  std::mutex err_mu;
  // persistence ring + writer
  int R = 0, b = 1;
  size_t slot_bytes = 0;
  uint8_t* ring = nullptr;            // pinned
  uint32_t* err_pinned = nullptr;     // pinned [R*2]
  std::vector<ld::Slot> slots;
  std::deque<int> free_slots;
  std::deque<int> queued;             // FIFO to the writer
  std::mutex mu;
  std::condition_variable cv_free, cv_work, cv_idle;
  bool stop = false, flush_req = false;
  int writer_busy = 0;
  std::thread writer;
  int64_t next_iter = -1;
  std::vector<uint8_t> prefix;        // header + hyper + layer table (n_iters patched per file)
  // stats
  std::atomic<int64_t> files_written{0}, bytes_written{0}, stall_ns{0}, writer_ns{0};
  int64_t spec_hits = 0, spec_misses = 0;
  // full checkpoint staging
  float* full_host = nullptr;         // pinned 3 * shard
  size_t full_cap = 0;
  cudaEvent_t full_done = nullptr;
  float* full_stage = nullptr;        // device 3 * shard: D2D stage so the producer waits for HBM only
  size_t full_stage_cap = 0;
  cudaEvent_t full_staged = nullptr;
  bool full_pending = false;
  int64_t full_iter = -1;
  std::thread full_writer;
  // LowDiff+ snapshot
  float* snap_host[2] = {nullptr, nullptr};
  int64_t snap_iter[2] = {-1, -1};
  std::vector<uint8_t> snap_seen[2];
  cudaEvent_t snap_done[2] = {nullptr, nullptr};
  bool snap_sharded = false;
  ld::Staging stage;                  // recovery loader's pinned chunks          // lowdiff_snapshot_shard: copy only this rank's 1/N of each bucket
  // peer-memory exchange (NEXT-1; peer.cu): own slots = send u32[2K] | merge tile starts
  int peer_slots = 0;
  std::vector<uint32_t*> peer_own;
  unsigned long long* peer_flags = nullptr;
  std::vector<const void*> peer_ptrs;             // world x (n_slots + 1): slot buffers..., flags
  bool peer_set = false;
  std::vector<unsigned long long> peer_epoch;     // per slot: epoch of the block now in it
  std::vector<void*> peer_opened;                 // IPC mappings opened through this context
  // LowDiff+ CPU replica of this rank's shard [rep_sb, rep_se) (replica.cpp, api.cpp)
  bool rep_active = false;
  uint64_t rep_sb = 0, rep_se = 0;
  float* rep_host = nullptr;          // pinned 3 * shard: p | m | v
  int rep_threads = 1;
  std::atomic<int64_t> rep_iter{-1};  // optimizer steps applied to the replica (worker-visible)
  int64_t rep_tail = -1;              // iteration the replica reaches once the queue drains
  std::deque<ld::RepJob> rep_q;
  std::mutex rep_mu;
  std::condition_variable rep_cv, rep_done_cv;
  bool rep_stop = false;
  int rep_busy = 0;
  std::thread rep_thread, rep_writer;
  std::vector<float> rep_stage;       // persisted copy (the worker keeps updating the replica)
  cudaEvent_t rep_init_done = nullptr;
  std::atomic<int64_t> rep_ns{0}, rep_stall_ns{0};
  // profiling
  bool prof = false;
  std::vector<ld::ProfRec> prof_recs;
  std::vector<cudaEvent_t> prof_pool;
  std::atomic<int64_t> launches{0};
  // replay scratch
  void* replay_scratch = nullptr;
  size_t replay_scratch_bytes = 0;
  void* merge_scratch = nullptr;
  size_t merge_scratch_bytes = 0;
  void* union_scratch = nullptr;
  size_t union_scratch_bytes = 0;
  float* scal_dev = nullptr;          // lowdiff_replay(_range): per-step scalars on the device
  size_t scal_cap = 0;
  uint64_t scratch_gen = 0;          // bumped when a scratch buffer a graph may bake in is reallocated
  // CUDA graphs of lowdiff_compress / merge (lowdiff_set_graphs)
  bool use_graphs = false;
  cudaStream_t cap_stream = nullptr;
  std::vector<ld::GraphEntry> graphs;
  uint64_t graph_tick = 0;
  // union-compacted persistence (NEXT-4): two library-owned device buffers idx | val of u_cap
  // entries each (this rank's shard), their counts, a writer thread that copies exactly the
  // count out and writes .ldu batches
  uint32_t* u_buf[2] = {nullptr, nullptr};
  unsigned long long* u_cnt_dev = nullptr;      // [2]
  unsigned long long* u_cnt_host = nullptr;     // pinned [2]
  cudaEvent_t u_ready[2] = {nullptr, nullptr};
  bool u_inuse[2] = {false, false};
  uint64_t u_cap = 0;
  int64_t u_next_iter = -1;
  uint32_t u_err_seen = 0;
  std::deque<ld::UJob> u_q;
  std::mutex u_mu;
  std::condition_variable u_cv, u_cv_free, u_cv_idle;
  bool u_stop = false, u_flush = false;
  int u_busy = 0;
  std::thread u_writer;
  cudaStream_t u_stream = nullptr;
  std::atomic<int64_t> u_files{0}, u_bytes{0}, u_entries{0};
  // Accumulated batch mode (R-30): the writer adds each iteration's dictionary into u_acc_* (host
  // memory) and writes one accumulated .ldu per batch
  int u_accumulate = 0;
};

namespace ld {
// kernels.cu
cudaError_t launch_compress(lowdiff_ctx* c, const float* grad, float* residual, uint32_t* send,
                            cudaStream_t s);
cudaError_t launch_materialize(lowdiff_ctx* c, float* residual, cudaStream_t s);
int compress_seg_capacity(uint32_t ppm, uint64_t n_segments);   // candidate slots per 1024-element segment
size_t compress_hist_bytes(int n_large);   // the select chain's per-layer radix histograms
cudaError_t launch_merge(lowdiff_ctx* c, int world, const uint32_t* gathered, float* dense,
                         cudaStream_t s);
// replays elements [lo, hi); p, m, v point at element lo.  ranges: NULL (every entry of every block
// is valid) or device u32[2 * n_steps * world] = the valid entry range of each block.
// k_stride: blocks are u32[2 * k_stride] (idx | val); 0 = the context's K (fixed-K blocks)
cudaError_t launch_replay(lowdiff_ctx* c, int optim, bool mean, const float* consts5, int world,
                          int64_t n_steps, const uint32_t* diffs, const float* scal_dev, uint64_t lo,
                          uint64_t hi, const uint32_t* ranges, float* p, float* m, float* v, cudaStream_t s,
                          uint64_t k_stride = 0);
// start[b * (T1 - T0 + 1) + t - T0] = first entry of block b (stride 2K, indices ascending) in tile t;
// ranges: device scratch u32[2 * n_blocks] (the window's entry range of each block)
cudaError_t launch_tile_window(const uint32_t* blocks, int n_blocks, uint64_t K, int shift, uint32_t T0, uint32_t T1,
                               uint32_t* start, uint32_t* ranges, cudaStream_t s);
// union.cu: union-compacted differential of [lo, hi): out = idx u32[cap] | val u32[cap]
cudaError_t launch_union(lowdiff_ctx* c, int world, bool mean, const uint32_t* gathered, uint64_t lo, uint64_t hi,
                         uint32_t* out, uint64_t cap, unsigned long long* count_dev, cudaStream_t s);
size_t union_scratch_bytes(int world, uint64_t lo, uint64_t hi);
cudaError_t launch_update(lowdiff_ctx* c, int world, const uint32_t* gathered, const lowdiff_step_scalars& sc,
                          float* p, float* m, float* v, cudaStream_t s);
cudaError_t run_selftest(int which, uint64_t n, uint64_t seed, uint64_t* mismatches, uint64_t* first);
size_t merge_scratch_bytes(int64_t psi, int world, int64_t n_blocks);
size_t replay_scratch_bytes(int64_t psi, int world, int64_t n_steps);

// profiling helpers (api.cpp)
void prof_begin(lowdiff_ctx* c, const char* name, cudaStream_t s, int* handle);
void prof_end(lowdiff_ctx* c, int handle, cudaStream_t s);

// files.cpp
uint32_t crc32c_update(uint32_t crc, const void* data, size_t len);
std::string batch_name(const std::string& dir, int rank, int64_t first);
std::string full_name(const std::string& dir, int rank, int64_t it);
void build_prefix(const lowdiff_config& cfg, const std::vector<int64_t>& numel, int64_t psi,
                  int64_t K, std::vector<uint8_t>& out);
lowdiff_status write_file_atomic(const std::string& path, const std::vector<std::pair<const void*, size_t>>& parts,
                                 bool do_fsync, std::string* err);
uint32_t crc32c_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b);
lowdiff_status stream_to_device(int fd, uint64_t off, const std::vector<std::pair<void*, uint64_t>>& segs,
                                Staging& stg, uint32_t* crc, std::string* err);
}  // namespace ld
