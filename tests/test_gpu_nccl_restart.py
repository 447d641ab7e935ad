"""GPU tests of the NCCL call sites (Alg. 1 l.5 Sync; "Allgather or Allreduce",
PAPER.md:213), the restart rules of persistence, and the peer-slot / full-checkpoint
lifetime.  Everything goes through the C ABI and is compared with the oracle.

* NCCL on one GPU: a context created with an NCCL id at world 1 owns a 1-rank communicator, so
  lowdiff_exchange (ncclAllGather), lowdiff_exchange_update (ncclAllGather), lowdiff_recover_sharded
  (gather: grouped ncclBroadcast) and lowdiff_replica_restore (ncclBroadcast) all execute NCCL.
* NCCL on >= 2 GPUs (skipped on a 1-GPU box): one process per GPU, real allgather over NVLink,
  every rank's dense G, live Adam state and sharded+gathered recovery against the oracle.
"""
import os

import numpy as np
import pytest
import torch

import paper_2509_04084_b200 as ld
from inputs import gradient

pytestmark = pytest.mark.gpu

DEV = "cuda"


def npf32(t):
    return t.cpu().numpy().astype(np.float32, copy=False)


def npu32(t):
    return t.cpu().numpy().view(np.uint32)


SIZES = [30000, 1600, 50000, 7, 4096, 20001]
PPM = 10000


def test_nccl_one_rank_every_call_site(ref, tmp_path):
    psi = sum(SIZES)
    nid = ld.nccl_unique_id()
    ctx = ld.Context(SIZES, density_ppm=PPM, world=1, rank=0, nccl_id=nid, ckpt_dir=str(tmp_path), batch_size=2,
                     optim=ld.ADAM)
    K = ctx.K
    rng = np.random.default_rng(7)
    p0 = rng.standard_normal(psi).astype(np.float32)
    p, m, v = torch.from_numpy(p0.copy()).to(DEV), torch.zeros(psi, device=DEV), torch.zeros(psi, device=DEV)
    P, M, V = p0.copy(), np.zeros(psi, np.float32), np.zeros(psi, np.float32)
    R = np.zeros(psi, np.float32)
    r = torch.zeros(psi, device=DEV)
    send = torch.empty(2 * K, dtype=torch.int32, device=DEV)
    gathered = torch.full((2 * K,), -1, dtype=torch.int32, device=DEV)
    dense = torch.empty(psi, device=DEV)
    ctx.full_ckpt(0, p, m, v)
    for t in range(1, 5):
        g = gradient(SIZES, 0, t, dist="D4", device=DEV)
        ctx.compress(g, r, send)
        gathered.fill_(-1)
        ctx.exchange(send, gathered, dense)                     # ncclAllGather (1 rank) + merge
        sc = ld.derive_step_scalars(t, 1e-2)
        ctx.exchange_update(send, gathered, sc, p, m, v)        # ncclAllGather + fused merge/Adam
        ctx.batch_persist(t, sc, send)
        torch.cuda.synchronize()
        want, R = ref.compress(SIZES, PPM, npf32(g), R, ef=True)
        assert np.array_equal(npu32(send), want) and np.array_equal(npu32(gathered), want)
        G = ref.exchange(want, 1, K, psi)
        assert np.array_equal(npf32(dense), G)
        ref.adam_step(G, ref.adam_consts(), ref.step_scalars(t, 1e-2), P, M, V)
        assert np.array_equal(npf32(p), P) and np.array_equal(npf32(m), M) and np.array_equal(npf32(v), V)
    ctx.sync()
    # sharded recovery with the gather leg (grouped ncclBroadcast over the 1-rank communicator)
    q, mq, vq = (torch.full((psi,), float("nan"), device=DEV) for _ in range(3))
    assert ctx.recover_sharded(q, mq, vq, gather=True) == 4
    assert np.array_equal(npf32(q), P) and np.array_equal(npf32(mq), M) and np.array_equal(npf32(vq), V)
    # replica restore (ncclBroadcast): the replica of the state at 4, restored into fresh buffers
    ctx.replica_init(4, p, m, v, threads=2)
    ctx.replica_wait()
    q2, m2, v2 = (torch.zeros(psi, device=DEV) for _ in range(3))
    assert ctx.replica_restore(q2, m2, v2) == 4
    assert np.array_equal(npf32(q2), P) and np.array_equal(npf32(m2), M) and np.array_equal(npf32(v2), V)
    ctx.close()


def _grads(seed, ts, psi):
    return {t: (np.random.default_rng([seed, t]).standard_normal(psi) * 1e-2).astype(np.float32) for t in ts}


@pytest.mark.parametrize("new_ctx_b", [None, 3])
def test_restart_after_recovery_misaligned_batches(ref, tmp_path, new_ctx_b):
    """run 1..10 with b = 4 (files …01 1-4, …05 5-8, …09 9-10), recover to 6, continue
    7..12 with other gradients (same context, b = 4: files …07 7-10, …11 11-12; or a new context
    with b = 3).  Without retiring the abandoned run, …09 (later first iteration) would override
    blocks 9-10 of …07.  Recovery of the latest state must equal the oracle's trajectory
    Full@0 + old 1..6 + new 7..12 (residual zeroed at the restart, R-7)."""
    psi = sum(SIZES)
    K = sum(ref.k_table(SIZES, PPM))
    old, new = _grads(1, range(1, 11), psi), _grads(2, range(7, 13), psi)
    p0 = np.random.default_rng(3).standard_normal(psi).astype(np.float32)
    ctx = ld.Context(SIZES, density_ppm=PPM, ckpt_dir=str(tmp_path), batch_size=4, optim=ld.ADAM)
    p, m, v = torch.from_numpy(p0.copy()).to(DEV), torch.zeros(psi, device=DEV), torch.zeros(psi, device=DEV)
    r = torch.zeros(psi, device=DEV)
    send = torch.empty(2 * K, dtype=torch.int32, device=DEV)
    ctx.full_ckpt(0, p, m, v)

    def run(c, grads, ts):
        for t in ts:
            c.compress(torch.from_numpy(grads[t]).to(DEV), r, send)
            sc = ld.derive_step_scalars(t, 1e-2)
            c.replay(ld.ADAM, 1, 1, send, [sc], p, m, v)
            c.batch_persist(t, sc, send)
        c.sync()

    run(ctx, old, range(1, 11))
    assert ctx.recover(p, m, v, target=6) == 6
    r.zero_()
    c2 = ctx
    if new_ctx_b is not None:
        ctx.close()
        c2 = ld.Context(SIZES, density_ppm=PPM, ckpt_dir=str(tmp_path), batch_size=new_ctx_b, optim=ld.ADAM)
    run(c2, new, range(7, 13))
    names = sorted(os.listdir(tmp_path))
    assert ref.batch_name(0, 9) not in names
    q, mq, vq = (torch.empty(psi, device=DEV) for _ in range(3))
    assert c2.recover(q, mq, vq) == 12
    # the oracle's trajectory
    P, M, V = p0.copy(), np.zeros(psi, np.float32), np.zeros(psi, np.float32)
    R = np.zeros(psi, np.float32)
    for t in range(1, 13):
        if t == 7:
            R = np.zeros(psi, np.float32)
        blk, R = ref.compress(SIZES, PPM, (old if t < 7 else new)[t], R, ef=True)
        ref.adam_step(ref.exchange(blk, 1, K, psi), ref.adam_consts(), ref.step_scalars(t, 1e-2), P, M, V)
    assert np.array_equal(npf32(q), P) and np.array_equal(npf32(mq), M) and np.array_equal(npf32(vq), V)
    # and the live state the context holds equals it too
    assert np.array_equal(npf32(p), P)
    c2.close()


def test_peer_slots_survive_full_checkpoint(ref, tmp_path):
    """a full checkpoint that allocates its stage must not free the peer slots.
    peer_alloc / peer_set, full_ckpt, then compress into a slot + exchange_peer, equal to the oracle."""
    psi = sum(SIZES)
    ctx = ld.Context(SIZES, density_ppm=PPM, ckpt_dir=str(tmp_path), batch_size=1)
    K = ctx.K
    slots, _ = ctx.peer_alloc(2, handles=False)
    ctx.peer_set([ctx.peer_ptrs + [ctx.peer_flags_ptr]])
    p = torch.randn(psi, device=DEV)
    r = torch.zeros(psi, device=DEV)
    R = np.zeros(psi, np.float32)
    dense = torch.empty(psi, device=DEV)
    for t in range(1, 5):
        ctx.full_ckpt(t - 1, p, None, None)      # the first call allocates the stage
        g = gradient(SIZES, 0, t, dist="D1", device=DEV)
        ctx.compress(g, r, slots[t % 2])
        ctx.exchange_peer(t % 2, dense)
        torch.cuda.synchronize()
        want, R = ref.compress(SIZES, PPM, npf32(g), R, ef=True)
        assert np.array_equal(npu32(slots[t % 2]), want)
        assert np.array_equal(npf32(dense), ref.exchange(want, 1, K, psi))
    ctx.sync()
    ctx.close()


# ---------------------------------------------------------------- real multi-GPU NCCL (>= 2 GPUs)
def _mgpu_worker(rank, world, port, tmp, q):
    try:
        import torch.distributed as dist
        import oracle as ref2
        import paper_2509_04084_b200 as ld2
        from inputs import gradient as grad2
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt = torch.frombuffer(bytearray(ld2.nccl_unique_id()), dtype=torch.uint8).clone()
        dist.broadcast(idt, 0)
        nid = bytes(idt.tolist())
        psi = sum(SIZES)
        ctx = ld2.Context(SIZES, density_ppm=PPM, world=world, rank=rank, nccl_id=nid, device=rank, ckpt_dir=tmp,
                          batch_size=2, optim=ld2.ADAM)
        K = ctx.K
        dev = torch.device("cuda", rank)
        p0 = np.random.default_rng(11).standard_normal(psi).astype(np.float32)
        p = torch.from_numpy(p0.copy()).to(dev)
        m, v, r = (torch.zeros(psi, device=dev) for _ in range(3))
        send = torch.empty(2 * K, dtype=torch.int32, device=dev)
        gathered = torch.empty(world * 2 * K, dtype=torch.int32, device=dev)
        dense = torch.empty(psi, device=dev)
        ctx.full_ckpt(0, p, m, v)
        P, M, V = p0.copy(), np.zeros(psi, np.float32), np.zeros(psi, np.float32)
        Rs = [np.zeros(psi, np.float32) for _ in range(world)]
        ok = True
        for t in range(1, 4):
            g = grad2(SIZES, rank, t, dist="D5", alpha=0.5, device=dev)
            ctx.compress(g, r, send)
            ctx.exchange(send, gathered, dense)
            sc = ld2.derive_step_scalars(t, 1e-2)
            ctx.exchange_update(send, gathered, sc, p, m, v)
            ctx.batch_persist(t, sc, send)
            torch.cuda.synchronize()
            blocks = []
            for q_ in range(world):
                gq = grad2(SIZES, q_, t, dist="D5", alpha=0.5, device=dev).cpu().numpy()
                b_, Rs[q_] = ref2.compress(SIZES, PPM, gq, Rs[q_], ef=True)
                blocks.append(b_)
            want = np.concatenate(blocks)
            G = ref2.exchange(want, world, K, psi)
            ok &= np.array_equal(gathered.cpu().numpy().view(np.uint32), want)
            ok &= np.array_equal(dense.cpu().numpy(), G)
            ref2.adam_step(G, ref2.adam_consts(), ref2.step_scalars(t, 1e-2), P, M, V)
            ok &= np.array_equal(p.cpu().numpy(), P) and np.array_equal(v.cpu().numpy(), V)
        ctx.full_ckpt(3, p, m, v)
        ctx.sync()
        dist.barrier()
        qq, mq, vq = (torch.zeros(psi, device=dev) for _ in range(3))
        rec = ctx.recover_sharded(qq, mq, vq, gather=True)
        ok &= rec == 3 and np.array_equal(qq.cpu().numpy(), P) and np.array_equal(mq.cpu().numpy(), M)
        ctx.close()
        q.put((rank, bool(ok), None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, False, repr(e)))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one rank per GPU)")
def test_nccl_multi_gpu_exchange_update_recovery(tmp_path):
    import multiprocessing as mp
    import socket
    world = min(torch.cuda.device_count(), 8)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_mgpu_worker, args=(r, world, port, str(tmp_path), q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
    assert all(ok for _, ok, _ in res), res


def test_ring_backpressure_blocks_after_exactly_ring_slots(tmp_path):
    """Backpressure: with the consumer stalled, the producer's
    lowdiff_batch_persist returns for the first R = ring_slots iterations and blocks on the next one
    until the consumer frees a slot.  The writer is stalled without a test hook: the first file's
    *.tmp name is a FIFO, so the writer's open() blocks until a reader opens the other end."""
    import threading
    import time

    sizes = [5000, 300]
    ctx = ld.Context(sizes, density_ppm=10000, ckpt_dir=str(tmp_path), batch_size=1, ring_slots=2,
                     write_files=True, fsync=False, optim=ld.ADAM)
    K = ctx.K
    fifo = tmp_path / "ld_diff_r000_000000000001.ldb.tmp"
    os.mkfifo(fifo)
    g = torch.randn(sum(sizes), device=DEV)
    r = torch.zeros(sum(sizes), device=DEV)
    sends = [torch.empty(2 * K, dtype=torch.int32, device=DEV) for _ in range(3)]
    rd = None
    try:
        for t in (1, 2):                          # iteration 1 -> the (stalled) writer, 2 -> the second slot
            ctx.compress(g, r, sends[t - 1])
            ctx.batch_persist(t, ld.derive_step_scalars(t, 1e-3), sends[t - 1])
        ctx.compress(g, r, sends[2])
        torch.cuda.synchronize()
        done = threading.Event()
        th = threading.Thread(target=lambda: (ctx.batch_persist(3, ld.derive_step_scalars(3, 1e-3), sends[2]),
                                              done.set()), daemon=True)
        th.start()
        time.sleep(1.0)
        assert not done.is_set(), "the third persist should block: both ring slots are held"
        rd = os.open(fifo, os.O_RDONLY | os.O_NONBLOCK)   # release the writer
        th.join(timeout=30)
        assert done.is_set(), "the blocked persist never resumed after the writer was released"
        assert ctx.stats()["ring_stall_ns"] >= 0.5e9
    finally:
        if rd is None:
            rd = os.open(fifo, os.O_RDONLY | os.O_NONBLOCK)
        os.close(rd)
    try:
        ctx.close()
    except ld.LowDiffError:
        pass   # the first file went into the pipe; later files are regular
