"""NEXT-1 across processes: two ranks in two processes on the one GPU of the test box (CUDA IPC
works between processes that share a device; the time-sliced contexts make the cross-process
waits real).  Each process maps the other's send slots and flag words through the IPC handles
exchanged over torch.distributed (gloo), runs compress -> exchange_peer for several iterations
with alternating slots, and returns its merged G and its send blocks; the parent checks that both
ranks' G equal lowdiff_merge of the two blocks bit for bit."""
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
        out = []
        for t in range(T):
            g = gradient(sizes, rank, t, dist="D5", alpha=0.5, model="resnet50", device="cuda")
            ctx.compress(g, r, slots[t % 2])
            ctx.exchange_peer(t % 2, dense)
            torch.cuda.synchronize()
            out.append((slots[t % 2].cpu().numpy().copy(), dense.cpu().numpy().copy()))
            dist.barrier()     # the peer's slot is re-used two iterations later; keep the copies consistent
        ctx.sync()
        dist.barrier()
        ctx.close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_two_process_ipc_peer_exchange():
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
    ctx = ld.Context(sizes, density_ppm=10000, world=2, rank=0)
    want = torch.empty(sum(sizes), device="cuda")
    for t in range(T):
        gathered = torch.from_numpy(np.concatenate([res[0][t][0], res[1][t][0]])).cuda()
        ctx.merge(2, gathered, want)
        w = want.cpu().numpy()
        for rank in (0, 1):
            assert np.array_equal(res[rank][t][1].view(np.uint32), w.view(np.uint32)), (t, rank)
    ctx.close()
