/*
 * lowdiff.h -- C ABI of the B200-native LowDiff hot path (arXiv 2509.04084, SC'25).
 *
 * LowDiff reuses the compressed gradients of data-parallel training as differential
 * checkpoints (Finding 1; Alg. 1).  This library is the
 * data-parallel hot path of that method on sm_100a:
 *   lowdiff_compress       per-layer top-k with error feedback       Alg. 1 l.4
 *   lowdiff_exchange       allgather of fixed-K blocks + merge       Alg. 1 l.5,7 PAPER.md:231,235
 *   lowdiff_batch_persist  reuse queue -> pinned ring -> batched file Alg. 1 l.6,12-14
 *   lowdiff_full_ckpt      sharded full checkpoint C^F               Alg. 1 l.15
 *   lowdiff_recover        chain scan + fused replay onto C^F        Alg. 1 l.16-24 PAPER.md:248-259
 * plus the LowDiff+ layer-wise dense snapshot (Alg. 2 l.19), the LowDiff+ CPU
 * replica (Sec. 5.2), union-compacted differentials (the synchronised G~_t as a
 * per-shard dictionary), the peer-memory exchange and the live update
 * (allgather fused into the merge / the optimizer), the checkpointing-configuration model
 * (Eq. 3-5), CUDA-graph replay of compress / merge, and device-resident replay
 * entry points used by recover and the benchmark.
 *
 * Conventions (all calls):
 *  - Every call returns lowdiff_status; none throws, aborts or exits.  A CUDA or NCCL
 *    failure poisons the context: every later call returns the same code.
 *  - Device pointers are plain CUDA device addresses (e.g. torch tensor data_ptr()),
 *    contiguous; fp32 arrays of Psi elements 16-byte aligned, u32 send/gathered blocks 4-byte
 *    aligned (else LOWDIFF_E_INVALID).  The CALLER owns every
 *    device buffer; the library never frees or reallocates caller memory.
 *  - `stream` arguments are cudaStream_t handles passed as void*.  Calls that take a
 *    stream enqueue work on it and return without a host synchronisation unless
 *    stated otherwise.
 *  - The LIBRARY owns the context, its NCCL communicator, side streams and events,
 *    pinned host ring, device scratch (sized at create; no allocation on the
 *    compress/exchange hot path), the writer thread, and the files it writes.
 *  - One context per (process, GPU); one host thread drives a context.
 * File formats and the numerical readings are specified in DESIGN.md.
 */
#ifndef LOWDIFF_H_
#define LOWDIFF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LOWDIFF_OK = 0,
  LOWDIFF_E_INVALID = 1,  /* bad argument: NULL, misaligned, out of range            */
  LOWDIFF_E_DIM = 2,      /* size mismatch ("dimension error")        */
  LOWDIFF_E_NUMERIC = 3,  /* non-finite accumulated gradient           */
  LOWDIFF_E_CUDA = 4,     /* CUDA runtime failure (context poisoned)                */
  LOWDIFF_E_NCCL = 5,     /* NCCL failure (context poisoned)                        */
  LOWDIFF_E_IO = 6,       /* storage failure                          */
  LOWDIFF_E_CORRUPT = 7,  /* CRC / format / header mismatch       */
  LOWDIFF_E_GAP = 8,      /* missing full checkpoint or diff in the chain */
  LOWDIFF_E_STATE = 9     /* call out of order (iteration not consecutive, FIFO S:249) */
} lowdiff_status;

typedef enum { LOWDIFF_SGD = 0, LOWDIFF_ADAM = 1 } lowdiff_optim;

/* Per-iteration optimizer scalars, derived on the host in double and rounded once
 * (R-11); stored in every differential block so replay never re-derives them. */
typedef struct { float lr, bc1_inv, bc2_inv; } lowdiff_step_scalars;

/* Adam constants {beta1, 1-beta1, beta2, 1-beta2, eps}, each rounded once from double. */
typedef struct { float beta1, one_minus_beta1, beta2, one_minus_beta2, eps; } lowdiff_adam_consts;

typedef struct {
  int32_t n_layers;            /* entries of the layer table (one per parameter tensor)        */
  const int64_t *numel;        /* [n_layers] sizes, forward order; Psi = sum < 2^32            */
  uint32_t density_ppm;        /* 1..1e6; k_l = max(1, min(n_l, floor(n_l*ppm/1e6)))  (R-3)    */
  int32_t error_feedback;      /* 1: acc = residual + grad, residual' = unsent part (default)  */
  int32_t mean;                /* 1: merged G = sum / world (default); 0: sum                  */
  int32_t rank, world;         /* data-parallel rank and world size                            */
  const void *nccl_unique_id;  /* 128-byte ncclUniqueId from rank 0 (lowdiff_nccl_unique_id,
                                  broadcast by the caller).  Given: an NCCL communicator of
                                  `world` ranks -- also at world 1 (a 1-rank communicator, so
                                  the allgather / broadcasts run through NCCL).  NULL: no
                                  communicator -- world 1 merges straight from the send block;
                                  world > 1 is a recovery/merge-only context (exchange then
                                  returns LOWDIFF_E_STATE)                                     */
  int32_t device;              /* CUDA device ordinal this context drives                      */
  const char *ckpt_dir;        /* directory for .ldb/.ldf files; NULL disables persistence     */
  int32_t batch_size;          /* b >= 1 differentials per .ldb file            */
  int32_t ring_slots;          /* pinned ring slots R >= b (0 -> 2b)                           */
  int32_t write_files;         /* 1: writer thread writes files; 0: D2H only (ring recycled)   */
  int32_t fsync;               /* 1: fsync each file before rename                             */
  int32_t optim;               /* lowdiff_optim recorded in the files and used by recover      */
  lowdiff_adam_consts adam;    /* recorded in the files and used by recover                    */
} lowdiff_config;

typedef struct lowdiff_ctx lowdiff_ctx;

/* Create a context: validates the layer table, builds the chunk plan, allocates device
 * scratch and the pinned ring, initialises NCCL (when an id is given) and starts the writer thread.
 * Synchronous.  *out is NULL on failure. */
lowdiff_status lowdiff_create(const lowdiff_config *cfg, lowdiff_ctx **out);

/* Drain all pending work (implies lowdiff_sync), stop the writer, free library resources.
 * Returns the first deferred error, if any.  ctx may be NULL. */
lowdiff_status lowdiff_destroy(lowdiff_ctx *ctx);

/* Psi and K = sum_l k_l. */
lowdiff_status lowdiff_query(const lowdiff_ctx *ctx, int64_t *psi, int64_t *k_tot);

/* k_l and koff_l (offset of layer l's entries inside a send block). */
lowdiff_status lowdiff_layer_k(const lowdiff_ctx *ctx, int32_t layer, int64_t *k, int64_t *koff);

/* 1. Compress (Alg. 1 line 4).  For every layer l:
 *      acc = residual + grad (error_feedback = 1) or grad;
 *      select the k_l entries with the largest key = bits(acc) & 0x7FFFFFFF, ties to the
 *      LOWER index; write them index-ascending into `send` at koff_l:
 *      send = idx u32[K] (global flat index) || val f32-bits u32[K];
 *      residual' = acc with the selected entries set to +0.0f.
 *    For layers larger than 4096 elements the +0.0f at the selected positions are DEFERRED:
 *    the residual buffer keeps acc there and the next lowdiff_compress on the same buffer
 *    zeroes them on the fly (the selection is {key > T_l} U {key == T_l, index < cut_l}, kept in
 *    the context), saving a scattered write pass.  Call lowdiff_residual_materialize before
 *    reading or modifying the buffer outside lowdiff_compress.
 *    grad: device f32[Psi] (read).  residual: device f32[Psi] (read/write; ignored and may
 *    be NULL when error_feedback = 0).  send: device u32[2K] (written).
 *    A non-finite acc sets a device flag; the next persist/sync returns LOWDIFF_E_NUMERIC.
 *    If `send` is still being copied out by a previous lowdiff_batch_persist, the stream
 *    waits for that copy (write-after-read). */
lowdiff_status lowdiff_compress(lowdiff_ctx *ctx, const float *grad, float *residual,
                                uint32_t *send, void *stream);

/* Write the deferred +0.0f of the last lowdiff_compress into `residual` (device f32[Psi]), so
 *    that it equals residual' exactly; afterwards the buffer may be read or changed freely.
 *    A no-op when nothing is pending.  Asynchronous on `stream`. */
lowdiff_status lowdiff_residual_materialize(lowdiff_ctx *ctx, float *residual, void *stream);

/* 2. Exchange (Alg. 1 lines 5 and 7): ncclAllGather of the fixed-size
 *    blocks (rank r's block lands at gathered + r*2K; with a communicator this also runs at
 *    world 1 when `gathered` is given), then the merge
 *      G[j] = ((((+0 + v_0[j]) + v_1[j]) + ... ) + v_{N-1}[j]) / N   (rank order, IEEE divide)
 *    where v_r[j] is rank r's value when j is among its indices.  No atomics: deterministic.
 *    send: device u32[2K].  gathered: device u32[world*2K] (may be NULL when world == 1).
 *    dense_out: device f32[Psi] (written entirely). */
lowdiff_status lowdiff_exchange(lowdiff_ctx *ctx, const uint32_t *send, uint32_t *gathered,
                                float *dense_out, void *stream);

/* Merge only (the second half of lowdiff_exchange) for a gathered buffer of `world`
 *    blocks that the caller assembled itself.  world >= 1; same arithmetic as above. */
lowdiff_status lowdiff_merge(lowdiff_ctx *ctx, int32_t world, const uint32_t *gathered,
                             float *dense_out, void *stream);

/* ---- Peer-memory exchange: allgather fused into the merge over NVLink ----
 * Each rank's send blocks live in library-owned device "slots" that the other ranks map (CUDA
 * IPC); lowdiff_exchange_peer's merge kernel reads every rank's entries of its output tile
 * straight from the owner's HBM, so no gathered buffer is written or re-read locally.
 * Same arithmetic as lowdiff_exchange (bitwise equal).  Protocol (all ranks in lockstep):
 *   1. lowdiff_peer_alloc(ctx, n, slots, flags, handles): n in 1..4 slots of u32[2K] (+ a tile
 *      table) and a flag buffer (*flags, may be NULL); handles (may be NULL) = (n + 1) x 64-byte cudaIpcMemHandle_t (slots,
 *      then flags) to share with the other ranks (e.g. torch.distributed.all_gather_object).
 *   2. lowdiff_ipc_open(ctx, handle, &ptr) for every peer handle (mappings are closed by
 *      lowdiff_destroy), then lowdiff_peer_set(ctx, ptrs): ptrs = world x (n + 1) device
 *      pointers in rank order (rank q: its n slots, then its flags; own entries = own buffers).
 *      Ranks that share one device (tests) pass each other's pointers directly.
 *   3. every iteration: lowdiff_compress(ctx, g, r, slots[i], s) -- it first waits (device-side)
 *      until every rank has read the previous block of slot i, and afterwards publishes the new
 *      block with its per-slot epoch -- then lowdiff_exchange_peer(ctx, i, dense_out, s), which
 *      waits (device-side) for every rank's block of this epoch, merges, and tells every owner
 *      it is done.  Alternate slots so that one rank's compress overlaps the peers' reads.
 *   Every device-side wait is bounded (20 s): a protocol misuse (a rank that never compresses or
 *   exchanges) then surfaces as LOWDIFF_E_STATE from lowdiff_sync rather than a hang. */
lowdiff_status lowdiff_peer_alloc(lowdiff_ctx *ctx, int32_t n_slots, uint32_t **slots_out, void **flags_out,
                                  void *handles_out);
lowdiff_status lowdiff_ipc_open(lowdiff_ctx *ctx, const void *handle64, void **ptr);
lowdiff_status lowdiff_peer_set(lowdiff_ctx *ctx, const void *const *ptrs);
lowdiff_status lowdiff_exchange_peer(lowdiff_ctx *ctx, int32_t slot, float *dense_out, void *stream);
/* Both halves of NEXT-1 fused (Alg. 1 lines 5-8): like lowdiff_exchange_peer, the
 *    merge reads every rank's entries of its tile from their slots (peer memory), but instead of
 *    writing G it applies the optimizer of cfg->optim (R-11 Adam / R-12 SGD, the scalars of this
 *    step) to the tile's p, m, v in the same pass -- bitwise what lowdiff_exchange followed by the
 *    oracle's step gives, with neither a gathered buffer nor a dense G in HBM.  p, m, v: device
 *    f32[Psi] (m, v unused for SGD), 16-byte aligned.  Same ordering protocol as
 *    lowdiff_exchange_peer (call it instead of exchange_peer for the slot).  Asynchronous. */
lowdiff_status lowdiff_exchange_peer_update(lowdiff_ctx *ctx, int32_t slot, const lowdiff_step_scalars *scalars,
                                            float *p, float *m, float *v, void *stream);

/* Exchange + optimizer step without a dense gradient (Alg. 1 lines 5, 7, 8,
 *    PAPER.md:231-237): the allgather of lowdiff_exchange, then p, m, v <- Opt(G, scalars) with
 *    G the merge of the gathered blocks computed tile by tile in shared memory and never written
 *    to HBM (the fused replay kernel with n = 1; optimizer = cfg.optim).  Bitwise equal to
 *    lowdiff_exchange followed by the R-11 Adam / R-12 SGD step on dense_out.  p, m, v: device
 *    f32[Psi] (m, v unused for SGD); gathered as in lowdiff_exchange.  Asynchronous. */
lowdiff_status lowdiff_exchange_update(lowdiff_ctx *ctx, const uint32_t *send, uint32_t *gathered,
                                       const lowdiff_step_scalars *scalars, float *p, float *m, float *v,
                                       void *stream);

/* 3. Batch persist (Alg. 1 line 6 Q.put, lines 12-14; Steps 1-3).
 *    Records an event on `producer`; a library side stream waits on it and copies this
 *    rank's own send block (8K bytes) into a pinned-host ring slot.  The writer thread
 *    groups b consecutive iterations into one .ldb file written with one writev
 *    (`*.tmp`, then rename).  `iteration` must be the previous call's + 1 (else
 *    LOWDIFF_E_STATE), except for the first call of a context and the first after a recovery /
 *    replica restore, which (re)start the sequence at `iteration` and first retire this rank's
 *    files holding iterations >= `iteration` (lowdiff_retire_from kinds .ldb|.ldf; E_IO if that
 *    fails).  Blocks on the host only while the ring is full (backpressure);
 *    the blocked time is reported by lowdiff_stats.  scalars: host pointer. */
lowdiff_status lowdiff_batch_persist(lowdiff_ctx *ctx, int64_t iteration,
                                     const lowdiff_step_scalars *scalars, const uint32_t *send,
                                     void *producer);

/* Make `stream` wait (device-side, no host block) until every D2H copy issued so far by
 *    lowdiff_batch_persist / lowdiff_full_ckpt / lowdiff_snapshot_layer has landed in host memory. */
lowdiff_status lowdiff_wait_persist(lowdiff_ctx *ctx, void *stream);

/* 4. Full checkpoint (Alg. 1 line 15): this rank's shard
 *    [floor(rank*Psi/world), floor((rank+1)*Psi/world)) of p, m, v (m, v may be NULL ->
 *    zeros), copied on a side stream after an event on `producer`: first D2D into a library-
 *    owned device stage (12 * shard bytes of HBM, allocated at the first call), and `producer`
 *    waits (device-side) only for that copy, so the caller's next update cannot overwrite the
 *    snapshot (write-after-read) yet is not held behind PCIe; then D2H from the
 *    stage.  If the stage cannot be allocated the shard is copied D2H directly and `producer`
 *    waits for that.  Persisted asynchronously as .ldf.
 *    `iteration` = optimizer steps applied to (p, m, v). */
lowdiff_status lowdiff_full_ckpt(lowdiff_ctx *ctx, int64_t iteration, const float *p,
                                 const float *m, const float *v, void *producer);

/* 5. Recover (Alg. 1 recovery process; Eq. 2):
 *    F = latest iteration <= target (-1: no bound) with all `world` .ldf shards present;
 *    then blocks F+1..target of every rank must exist (LOWDIFF_E_GAP) and verify
 *    (LOWDIFF_E_CORRUPT); target = -1 replays the longest gap-free chain.  Loads C^F into
 *    p, m, v (device f32[Psi]; m, v may be NULL for SGD), replays the blocks through the
 *    optimizer recorded in the files with the fused replay kernel, and stores the
 *    iteration reached in *recovered.  Synchronous (returns after the replay finished).
 *    Afterwards persisting may resume at *recovered + 1: the next lowdiff_batch_persist /
 *    lowdiff_union_persist accepts any iteration t and first retires this rank's files holding
 *    iterations >= t (lowdiff_retire_from), so blocks of the abandoned run never enter a chain. */
lowdiff_status lowdiff_recover(lowdiff_ctx *ctx, int64_t target, float *p, float *m, float *v,
                               int64_t *recovered, void *stream);

/* Fused replay of n_steps differentials that are already in device memory:
 *    diffs: device u32[n_steps][world][2K] (the gathered blocks of each step, rank order);
 *    scalars: host [n_steps]; optim: lowdiff_optim.  For each step t in order,
 *    G_t = merge(diffs[t]) then p, m, v <- SGD/Adam(G_t, scalars[t]).  Every element's
 *    result equals applying the steps one at a time.  Asynchronous on `stream`. */
lowdiff_status lowdiff_replay(lowdiff_ctx *ctx, int32_t optim, int32_t world, int64_t n_steps,
                              const uint32_t *diffs, const lowdiff_step_scalars *scalars,
                              float *p, float *m, float *v, void *stream);

/* Sharded recovery (NEXT-2; the per-element replay of R-16 split by parameter range).
 * replay_range: lowdiff_replay restricted to elements [begin, end) of Psi; p, m, v are device
 *    f32[end - begin] holding exactly that range (p[0] = element begin).  The result equals the
 *    same elements of a full lowdiff_replay bit for bit.
 * recover_sharded: lowdiff_recover for this rank's shard [floor(rank*Psi/world),
 *    floor((rank+1)*Psi/world)) only: reads only this rank's .ldf shard, uploads only the entries
 *    of each differential block that fall in the shard (the indices ascend, so they are one
 *    contiguous run per block), and replays only the shard into p, m, v (device f32[Psi];
 *    elements outside the shard are not touched).  gather != 0 (NCCL context needed if world > 1;
 *    with a 1-rank communicator the broadcast runs too):
 *    then fills the other shards from their owners by NCCL broadcasts, so every rank ends with
 *    the full state.  Chain selection (F, last) is exactly that of lowdiff_recover (all ranks
 *    agree).  Synchronous. */
lowdiff_status lowdiff_replay_range(lowdiff_ctx *ctx, int32_t optim, int32_t world, int64_t n_steps,
                                    const uint32_t *diffs, const lowdiff_step_scalars *scalars,
                                    int64_t begin, int64_t end, float *p, float *m, float *v,
                                    void *stream);
lowdiff_status lowdiff_recover_sharded(lowdiff_ctx *ctx, int64_t target, float *p, float *m, float *v,
                                       int32_t gather, int64_t *recovered, void *stream);

/* ---- Union-compacted differentials (R-29) ----
 * C^U_t = the synchronised compressed gradient G~_t of Alg. 1 line 5, put in the
 * reusing queue after Sync (line 6), kept as an index -> value dictionary
 * ("dictionary accumulation"): every index j that appears in some rank's block of the
 * iteration, ascending, with the merged value G_t[j] exactly as lowdiff_exchange writes it (rank-
 * order sum from +0, then / N when the context's mean flag is set).  Smaller than the N fixed-K
 * blocks whenever the ranks' supports overlap; replays to the same state bit for bit.
 *
 * union_compact: the members in [begin, end) of the union of the `world` blocks in `gathered`
 *    (device u32[world * 2K], rank r's block at r * 2K, each index-ascending) ->
 *    out = idx u32[cap] | val u32[cap] (device, entries [0, *count_dev) valid, ascending),
 *    *count_dev = device u64.  cap must be >= min(world * K, end - begin) (the worst case; else
 *    E_INVALID), so the result always fits.  Enqueued on `stream`, no host synchronisation.
 *    E_DIM if [begin, end) is not inside [0, Psi). */
lowdiff_status lowdiff_union_compact(lowdiff_ctx *ctx, int32_t world, const uint32_t *gathered, int64_t begin,
                                     int64_t end, uint32_t *out, int64_t cap, uint64_t *count_dev, void *stream);
/* union_persist: compact this rank's shard [floor(rank*Psi/world), floor((rank+1)*Psi/world)) of
 *    the gathered blocks of `iteration` (as union_compact with world = the context's) into a
 *    library-owned device buffer on `producer`, then a writer thread copies exactly the union out
 *    (a count read first) and writes batches of batch_size iterations as
 *    <ckpt_dir>/ld_union_r{rank:03}_{first:012}.ldu (layout: DESIGN.md §3; *.tmp then rename;
 *    no files without a ckpt_dir).  `gathered` may be reused once `producer` has passed this call.
 *    Two buffers alternate: the call blocks on the host only while the buffer of iteration - 2 is
 *    still being copied out.  `iteration` must be the previous call's + 1 (else E_STATE).  A non-
 *    finite accumulated gradient before the iteration stops the chain (E_NUMERIC deferred to the
 *    next call / lowdiff_sync).  lowdiff_sync flushes the final partial batch. */
lowdiff_status lowdiff_union_persist(lowdiff_ctx *ctx, int64_t iteration, const lowdiff_step_scalars *scalars,
                                     const uint32_t *gathered, void *producer);
/* Batch mode of union_persist (R-30).
 *    LOWDIFF_BATCH_RECORD (default): a .ldu holds its b dictionaries verbatim; recovery is exact.
 *    LOWDIFF_BATCH_ACCUMULATED: the paper's "gradient accumulation" batching, done by
 *    the CPU as "the addition of compressed gradients" ("tensor addition or dictionary
 *    accumulation"): the writer thread adds the b dictionaries of a batch into ONE,
 *    in iteration order (A[j] = (j in A ? A[j] : +0.0f) + x, fp32), and writes it as a .ldu with
 *    flags bit 2 set, n_iters = b and a single block tagged with the batch's last iteration and
 *    its scalars.  recover_union replays such a batch as ONE optimizer step with G = A and those
 *    scalars: the state after the batch is NOT the live state for b > 1 (exact in real arithmetic
 *    only for SGD at a constant lr), and targets inside the batch are unreachable (E_GAP).
 *    Switching modes first writes the batch in flight (partial) in the old mode; setting the
 *    current mode is a no-op.  E_INVALID for another value. */
enum { LOWDIFF_BATCH_RECORD = 0, LOWDIFF_BATCH_ACCUMULATED = 1 };
lowdiff_status lowdiff_set_batch_mode(lowdiff_ctx *ctx, int32_t mode);
/* recover_union: Alg. 1 recovery from full checkpoints and .ldu files with the
 *    chain rules of lowdiff_recover (latest complete Full F <= target; every needed rank's .ldu
 *    must hold each of F+1..target, later files winning; E_GAP / E_CORRUPT / E_IO as there).
 *    sharded = 0: every shard and every rank's union files, all of p, m, v (f32[Psi]) restored;
 *    sharded = 1: only this rank's .ldf shard and .ldu files, only its element range of p, m, v
 *    written (the arrays are still indexed by global element).  The replay is the fused kernel
 *    of lowdiff_replay; the result is bitwise the state lowdiff_recover reaches from the .ldb
 *    chain of the same run (record mode).  An accumulated .ldu (see lowdiff_set_batch_mode) is one
 *    replay step covering its b iterations; every rank must hold a batch covering the same
 *    iterations (else E_CORRUPT).  Synchronous on `stream`. */
lowdiff_status lowdiff_recover_union(lowdiff_ctx *ctx, int64_t target, float *p, float *m, float *v, int32_t sharded,
                                     int64_t *recovered, void *stream);

/* LowDiff+ layer-wise snapshot (Sec. 5.1; Alg. 2 l.19):
 *    after the caller's gradient sync of layers [first_layer, first_layer+n_layers)
 *    (contiguous in the flat gradient; grad_bucket points at layer first_layer), copy
 *    them D2H on a side stream into the pinned buffer of `iteration` (double-buffered:
 *    iterations t and t+1 may be in flight).  grad_bucket must not be rewritten before the
 *    copy has read it: lowdiff_wait_persist(ctx, s) orders stream s after it.  While a CPU
 *    replica is active (lowdiff_replica_init) only the replica's shard of the bucket is copied;
 *    the rest of the host buffer is then not updated. */
lowdiff_status lowdiff_snapshot_layer(lowdiff_ctx *ctx, int64_t iteration, int32_t first_layer,
                                      int32_t n_layers, const float *grad_bucket, void *producer);

/* Sharded snapshots (enable != 0): lowdiff_snapshot_layer copies only this rank's shard
 *    [floor(rank*Psi/world), floor((rank+1)*Psi/world)) of each bucket -- the part of the synced
 *    gradient a data-parallel rank has to keep (PCIe bytes per rank / world); the rest of the host
 *    buffer is not updated.  Always the case while a CPU replica is active. */
lowdiff_status lowdiff_snapshot_shard(lowdiff_ctx *ctx, int32_t enable);

/* Wait until every layer of `iteration` has been snapshotted; *host_grad = pinned
 *    f32[Psi] valid until iteration + 2 is first snapshotted.  LOWDIFF_E_STATE if some
 *    layer of that iteration was never submitted. */
lowdiff_status lowdiff_snapshot_wait(lowdiff_ctx *ctx, int64_t iteration, const float **host_grad);

/* Snapshot bucket plan (no context, host only): cut the layer table into runs of contiguous
 *    layers of at least min_bytes of fp32 gradient each, in BACKWARD order (the order a
 *    backward pass finalises them: the last layer first; PAPER.md:366-369 snapshots layer by
 *    layer as gradients become ready, and SURVEY §8(a) a9 asks for >= 4 MB runs so the many
 *    6.4 KB LayerNorm/bias tensors are never copied one by one).  Bucket i covers layers
 *    [first[i], first[i] + count[i]); first[0] + count[0] == n_layers, first[n-1] == 0.  The
 *    last bucket formed (the one holding layer 0) absorbs any remainder below min_bytes.
 *    cap = capacity of first/count; *n_buckets = buckets written.  E_INVALID on bad arguments
 *    (n_layers < 1, a numel < 1, min_bytes < 0), E_DIM if cap is too small. */
lowdiff_status lowdiff_bucket_plan(int32_t n_layers, const int64_t *numel, int64_t min_bytes,
                                   int32_t *first, int32_t *count, int32_t cap, int32_t *n_buckets);

/* ---- LowDiff+ CPU replica (Sec. 5.2; Alg. 2 l.11-13) ----
 * A host-resident copy of this rank's shard [floor(rank*Psi/world), floor((rank+1)*Psi/world))
 * of (p, m, v), advanced on a worker thread by the snapshotted synced gradients with the host
 * optimizer (bitwise equal to the device replay), persisted as a regular .ldf shard, and
 * restored to the GPU after a software failure.
 *
 * replica_init: (re)start the replica from the device state (p, m, v; m, v may be NULL -> zeros)
 *    after `iteration` optimizer steps; the D2H copy is ordered after `producer`'s prior work and
 *    `producer` waits for it (write-after-read).  threads = host threads of the optimizer (>= 1).
 *    Pinned host memory: 12 * shard bytes.  Pending work of a previous replica is drained first. */
lowdiff_status lowdiff_replica_init(lowdiff_ctx *ctx, int64_t iteration, const float *p, const float *m,
                                    const float *v, int32_t threads, void *producer);
/* replica_step: queue M^C_t = M^C_{t-1} + Opt(G_t) for t = `iteration` = (replica iteration after
 *    the queued steps) + 1, G_t = the gradient snapshotted for `iteration` (every layer must have
 *    been submitted with lowdiff_snapshot_layer: else LOWDIFF_E_STATE), scalars = that step's
 *    scalars.  Returns at once; while the step is pending, lowdiff_snapshot_layer for
 *    iteration + 2 blocks (the snapshot buffer is still being read; counted in replica_stall_ns). */
lowdiff_status lowdiff_replica_step(lowdiff_ctx *ctx, int64_t iteration, const lowdiff_step_scalars *scalars);
/* replica_persist: queue a persist of the replica as it stands after the queued steps, as
 *    ld_full_r{rank}_{iteration}.ldf (same format and sharding as lowdiff_full_ckpt, so
 *    lowdiff_recover uses it as a full checkpoint).  The worker copies the shard to a staging
 *    buffer and a writer thread writes it while the replica keeps advancing. */
lowdiff_status lowdiff_replica_persist(lowdiff_ctx *ctx);
/* replica_wait: drain the queue (and the persist writer); *iteration = replica iteration.
 *    *p, *m, *v (any may be NULL) = host pointers to the shard (valid until the next call that
 *    queues work or destroys the context); *shard_begin / *shard_end = the shard range. */
lowdiff_status lowdiff_replica_wait(lowdiff_ctx *ctx, int64_t *iteration, const float **p, const float **m,
                                    const float **v, int64_t *shard_begin, int64_t *shard_end);
/* replica_restore: drain, then copy the replica into device p, m, v (f32[Psi]; m, v may be NULL
 *    for SGD): this rank's shard H2D, the other shards by an NCCL broadcast from their owners
 *    (world > 1: every rank must call it; needs an NCCL context; a 1-rank communicator also
 *    broadcasts).  Synchronous on `stream`; *iteration = the restored iteration.  Persisting may
 *    then resume at *iteration + 1 (its first lowdiff_batch_persist retires the abandoned run's
 *    files, see lowdiff_retire_from). */
lowdiff_status lowdiff_replica_restore(lowdiff_ctx *ctx, float *p, float *m, float *v, int64_t *iteration,
                                       void *stream);
/* Host optimizer used by the replica (no context; element-wise over n, split over `threads`
 *    host threads): Adam in the op order of DESIGN.md R-11 / SGD p -= lr * G, IEEE single
 *    precision, no contraction.  Arrays are host memory, p/m/v updated in place. */
lowdiff_status lowdiff_host_adam_step(int64_t n, const float *G, const lowdiff_adam_consts *consts,
                                      const lowdiff_step_scalars *scalars, float *p, float *m, float *v,
                                      int32_t threads);
lowdiff_status lowdiff_host_sgd_step(int64_t n, const float *G, float lr, float *p, int32_t threads);

/* Drain D2H copies and the writer (flushing a final partial batch) and
 * surface deferred errors. */
lowdiff_status lowdiff_sync(lowdiff_ctx *ctx);

typedef struct {
  int64_t files_written, bytes_written;
  int64_t ring_stall_ns;       /* host time lowdiff_batch_persist spent blocked on a full ring */
  int64_t writer_busy_ns;      /* writer thread time spent building + writing files            */
  int64_t spec_hits, spec_misses;   /* large layers selected from the speculative band / refilled */
  int64_t spec_candidates;          /* candidates the band admitted in those hit layers (last call) */
  int64_t replica_busy_ns;          /* replica worker time spent in the host optimizer            */
  int64_t replica_stall_ns;         /* host time lowdiff_snapshot_layer waited for the replica    */
  int64_t union_files_written;      /* .ldu files written (lowdiff_union_persist)                 */
  int64_t union_bytes_written;
  int64_t union_entries;            /* union entries persisted (sum over iterations)              */
  int64_t direct_segments;          /* last call: 1024-element segments with more candidates than
                                       their bounded slot (re-read from acc instead)              */
  int64_t compress_scratch_bytes;   /* device memory of the plan + compress scratch (O(K))        */
  int64_t device_bytes;             /* all library-owned device memory now allocated              */
} lowdiff_stats;
lowdiff_status lowdiff_get_stats(const lowdiff_ctx *ctx, lowdiff_stats *out);

/* Per-layer trace of the last lowdiff_compress (synchronises the device): for each of the
 * n_large layers above 4096 elements (in layer-table order; *n_large receives the count, arrays
 * may be NULL to query it): layer[i] = its layer id, level[i] = 0 selected from the speculative
 * band, 1 refilled (a histogram pass over the layer, then a rescan at the lower edge of the
 * digit-0 bin (key bits [30:20]) holding the k-th key: at least k candidates by construction),
 * candidates[i] = keys admitted at the threshold finally used, threshold[i] = that threshold key. */
lowdiff_status lowdiff_compress_trace(lowdiff_ctx *ctx, int32_t cap, int32_t *n_large, int32_t *layer,
                                      int32_t *level, uint32_t *candidates, uint32_t *threshold);

/* Per-kernel device timing (CUDA events recorded on the launching stream).  enable != 0
 * starts recording; lowdiff_prof_read synchronises and returns the summed milliseconds
 * and launch count of kernel `name` since enabling ("" = all). */
lowdiff_status lowdiff_prof_enable(lowdiff_ctx *ctx, int32_t enable);
lowdiff_status lowdiff_prof_read(lowdiff_ctx *ctx, const char *name, double *total_ms,
                                 int64_t *launches);

/* CUDA graphs (enable != 0): lowdiff_compress and the merge of lowdiff_exchange / lowdiff_merge
 *    capture their kernel sequence into a CUDA graph per (call, buffer addresses, deferred-zero
 *    state) on first use and replay it afterwards -- the same kernels with the same arguments, so
 *    the same bits, with fewer launch gaps (what bounds small models).  Up to 8 graphs are cached;
 *    a graph is rebuilt when a library scratch buffer it uses is reallocated.  Ignored while
 *    profiling is enabled (lowdiff_prof_enable).  Off by default. */
lowdiff_status lowdiff_set_graphs(lowdiff_ctx *ctx, int32_t enable);

/* Number of kernels this library launched on behalf of ctx since creation. */
int64_t lowdiff_kernel_launches(const lowdiff_ctx *ctx);

const char *lowdiff_last_error(const lowdiff_ctx *ctx);

/* ---- host helpers (no context, no GPU needed) ---- */
/* Write a fresh 128-byte ncclUniqueId into out (rank 0 calls this, then broadcasts). */
lowdiff_status lowdiff_nccl_unique_id(void *out128);
/* {lr, 1/(1-beta1^t), 1/(1-beta2^t)} in double with beta^t by t repeated products, rounded once. */
lowdiff_status lowdiff_derive_step_scalars(int64_t t, double lr, double beta1, double beta2,
                                           lowdiff_step_scalars *out);
lowdiff_status lowdiff_derive_adam_consts(double beta1, double beta2, double eps,
                                          lowdiff_adam_consts *out);
/* CRC-32C (Castagnoli) of len bytes, as stored in the file trailers. */
uint32_t lowdiff_crc32c(const void *data, size_t len);
/* Locate the recoverable chain in cfg->ckpt_dir without loading it (host only):
 *    *full_iter = F, *last_iter = last replayable iteration (target rules as recover). */
lowdiff_status lowdiff_chain_scan(const lowdiff_config *cfg, int64_t target, int64_t *full_iter,
                                  int64_t *last_iter);
/* Serialise a batch file from host blocks exactly as the writer thread does (host only;
 *    used by multi-rank host tests): blocks = n_iters x 2K u32, scalars = n_iters. */
lowdiff_status lowdiff_write_batch_host(const lowdiff_config *cfg, int64_t first_iter,
                                        int32_t n_iters, const lowdiff_step_scalars *scalars,
                                        const uint32_t *blocks);
/* Restart hygiene (host only): remove / truncate this rank's (cfg->rank) files in cfg->ckpt_dir that
 * hold iterations >= `iteration` -- they belong to an abandoned run.  kinds: bit0 .ldb (files
 * starting at >= iteration removed, a file straddling it rewritten atomically with its blocks <
 * iteration), bit1 .ldu (same), bit2 .ldf (iterations >= iteration removed).  lowdiff_batch_persist
 * (kinds .ldb|.ldf) and lowdiff_union_persist (.ldu|.ldf) call it on their first call of a context
 * and on their first call after lowdiff_recover* / lowdiff_replica_restore, which re-open the
 * iteration sequence (the next persisted iteration may then be any value).  E_IO if a file cannot
 * be removed or rewritten. */
lowdiff_status lowdiff_retire_from(const lowdiff_config *cfg, int64_t iteration, int32_t kinds);
/* Serialise this rank's full-checkpoint shard from host arrays of length Psi (host only). */
lowdiff_status lowdiff_write_full_host(const lowdiff_config *cfg, int64_t iteration, const float *p,
                                       const float *m, const float *v);
/* ---- checkpointing configuration (§4.3, Eq. 3-5; module PAPER.md:454-455)
 * System parameters of the wasted-time model, all times in ONE unit (R-27 uses
 * iterations): N GPUs, M mean time between failures, W write bandwidth (bytes per time unit),
 * S full-checkpoint bytes, T total run time, R_F time to load a full checkpoint, R_D time to
 * merge one differential. */
typedef struct { double N, M, W, S, T, R_F, R_D; } lowdiff_sys_params;
/* Eq. 3: T_wasted(f, b) for f full checkpoints per time unit and b differentials per batch.
 * The model's domain is f b <= 1 (a batch inside one full-checkpoint interval): f b > 1 -> E_INVALID
 * (also for lowdiff_simulate_failures). */
lowdiff_status lowdiff_wasted_time(const lowdiff_sys_params *p, double f, double b, double *out);
/* Eq. 5: the stationary point f* = cbrt(R_D W^2/(4 S^2 M^2)), b* = cbrt(2 S R_D M / W). */
lowdiff_status lowdiff_optimal_config(const lowdiff_sys_params *p, double *f_star, double *b_star);
/* Eq. 5 clamped to f b <= 1: (f*, b*) when f* b* <= 1 (*clamped = 0); else the minimum of Eq. 3 on
 * the boundary f b = 1, f = sqrt(W / (2 M S)), b = 1/f (*clamped = 1).  f_unc / b_unc (optional)
 * receive the unconstrained Eq. 5 point. */
lowdiff_status lowdiff_optimal_config_feasible(const lowdiff_sys_params *p, double *f_opt, double *b_opt,
                                               double *f_unc, double *b_unc, int32_t *clamped);
/* One stepwise adaptation of the integer configuration (full-checkpoint interval *fcf in time
 * units, batch size *batch <= *fcf) toward the rounded feasible optimum, applied only if it lowers
 * Eq. 3; the step never leaves batch <= fcf. */
lowdiff_status lowdiff_config_step(const lowdiff_sys_params *p, int64_t *fcf, int32_t *batch);
/* Failure-injection simulator: failures of the N GPUs as a Poisson process of rate
 * N / M over the productive time [0, T) (inter-arrival -log(1 - u) M / N; u from splitmix64 over a
 * counter starting at `seed`), each "software" with probability sw_fraction.
 * Hardware failure at t: x = t mod (1/f); lost work x mod b; recovery R_F + R_D floor(x / b).
 * Software failure (LowDiff+ replica restore): recovery R_S, no lost work.
 * steady = N (S / W) floor(f T); wasted = lost + recovery + steady (the ledger of Eq. 3, whose
 * expectation it equals when 1/f is a multiple of b); effective_ratio = T / (T + wasted). */
typedef struct {
  int64_t failures, hw_failures;
  double lost_work, recovery, steady, wasted, effective_ratio;
} lowdiff_sim_report;
lowdiff_status lowdiff_simulate_failures(const lowdiff_sys_params *p, double f, double b, double sw_fraction,
                                         double R_S, uint64_t seed, lowdiff_sim_report *out);

int32_t lowdiff_abi_version(void);
/* Device self-test of the branch-free IEEE sqrt/division used by the replay kernel against
 * __fsqrt_rn/__fdiv_rn (which = 0: all 2^31+1 non-negative floats; which = 1: n pseudo-random
 * operand pairs from `seed`; which = 2: Adam's fused u = mh / (sqrt(vh) + eps) on n random
 * triples; which = 3: the paired (f32x2) Adam step of the replay / update kernels on n random
 * element pairs against the scalar R-11 sequence; which = 4: the division on every exponent pair
 * of [2^-70, 2^67]^2 (the fast window and ten binades around each edge: extreme mantissas and
 * n / 138^2 - 4 random ones per pair, all signs); which = 5: the paired Adam direction
 * mh / (sqrt(vh) + eps) with its window test on every exponent pair of mh in [2^-90, 2^87] and vh
 * over the whole float range).  Needs a GPU (current device); synchronous. */
lowdiff_status lowdiff_selftest(int32_t which, uint64_t n, uint64_t seed, uint64_t *mismatches,
                                uint64_t *first_bad);

#ifdef __cplusplus
}
#endif
#endif /* LOWDIFF_H_ */
