"""NEXT-1 across processes: two ranks in two processes on the one GPU of the test box (CUDA IPC
works between processes that share a device; the time-sliced contexts make the cross-process
waits real).  Each process maps the other's send slots and flag words through the IPC handles
exchanged over torch.distributed (gloo), runs compress -> exchange_peer for several iterations
with alternating slots, and returns its merged G and its send blocks; the parent checks that both
ranks' G equal the oracle's exchange (R-8) of the oracle's own compressed blocks bit for bit, and
that both ranks' p, m, v after the fused peer update (lowdiff_exchange_peer_update) equal the
oracle's Adam step on that G."""
import multiprocessing as mp
import socket

import numpy as np
import pytest
import torch

import paper_2509_04084_b200 as ld
from inputs import gradient, table

pytestmark = pytest.mark.gpu
T = 4


def _worker(rank, world, port, q):
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        sizes = table("resnet50")
        psi = sum(sizes)
        ctx = ld.Context(sizes, density_ppm=10000, world=world, rank=rank)   # no NCCL: peer exchange only
        slots = ctx.peer_setup(2)
        r = torch.zeros(psi, device="cuda")
        dense = torch.empty(psi, device="cuda")
        p = torch.full((psi,), 0.5, device="cuda")
        m = torch.zeros(psi, device="cuda")
        v = torch.zeros(psi, device="cuda")
        out = []
        for t in range(T):
            g = gradient(sizes, rank, t, dist="D5", alpha=0.5, model="resnet50", device="cuda")
            ctx.compress(g, r, slots[t % 2])
            ctx.exchange_peer(t % 2, dense)
            ctx.exchange_peer_update(t % 2, ld.derive_step_scalars(t + 1, 1e-3), p, m, v)
            torch.cuda.synchronize()
            out.append((slots[t % 2].cpu().numpy().copy(), dense.cpu().numpy().copy(), p.cpu().numpy().copy(),
                        v.cpu().numpy().copy()))
            dist.barrier()     # the peer's slot is re-used two iterations later; keep the copies consistent
        ctx.sync()
        dist.barrier()
        ctx.close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_two_process_ipc_peer_exchange(ref):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=240) for _ in procs)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for rank in (0, 1):
        assert not isinstance(res[rank], str), res[rank]
    sizes = table("resnet50")
    psi = sum(sizes)
    K = sum(ref.k_table(sizes, 10000))
    R = [np.zeros(psi, np.float32) for _ in range(2)]
    P, M, V = np.full(psi, 0.5, np.float32), np.zeros(psi, np.float32), np.zeros(psi, np.float32)
    for t in range(T):
        blocks = []
        for rank in (0, 1):
            g = gradient(sizes, rank, t, dist="D5", alpha=0.5, model="resnet50", device="cuda").cpu().numpy()
            b, R[rank] = ref.compress(sizes, 10000, g, R[rank], ef=True)
            blocks.append(b)
            assert np.array_equal(res[rank][t][0].view(np.uint32), b), (t, rank)   # the slot = the oracle block
        G = ref.exchange(np.concatenate(blocks), 2, K, psi)
        ref.adam_step(G, ref.adam_consts(), ref.step_scalars(t + 1, 1e-3), P, M, V)
        for rank in (0, 1):
            assert np.array_equal(res[rank][t][1].view(np.uint32), G.view(np.uint32)), (t, rank)
            assert np.array_equal(res[rank][t][2].view(np.uint32), P.view(np.uint32)), (t, rank)
            assert np.array_equal(res[rank][t][3].view(np.uint32), V.view(np.uint32)), (t, rank)
