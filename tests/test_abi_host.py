"""CPU-only checks of the product library (no GPU): it loads, exports every symbol that
include/lowdiff.h declares, and its host-side logic (scalar derivation, CRC-32C, file
serialisers, chain scan) agrees with the oracle and with the stated rules."""
import os
import re

import numpy as np
import pytest

import paper_2509_04084_b200 as ld
from paper_2509_04084_b200 import lowdiff as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lowdiff.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lowdiff_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = B.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == {"lowdiff_" + n for n in B.EXPORTED}
    assert L.lowdiff_abi_version() == 1


def test_library_is_sm100a_and_links_nccl():
    so = B.LIB_PATH
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "libnccl.so.2" in deps


def test_scalars_and_consts_match_oracle(ref):
    for t in (1, 2, 7, 100, 5000):
        for lr in (1e-3, 0.1, 3e-4):
            s = ld.derive_step_scalars(t, lr)
            o = ref.step_scalars(t, lr)
            assert np.array_equal(np.array([s.lr, s.bc1_inv, s.bc2_inv], np.float32), o)
    c = ld.derive_adam_consts()
    assert np.array_equal(np.array([c.beta1, c.one_minus_beta1, c.beta2, c.one_minus_beta2, c.eps], np.float32),
                          ref.adam_consts())


def test_crc32c_matches_oracle(ref):
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 9, 63, 1000, 4097):
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert ld.crc32c(data) == ref.crc32c(data)


SIZES = [1000, 10, 3000, 7, 20000]


def _opts(tmp, **kw):
    o = ld.Options(density_ppm=20000, ckpt_dir=str(tmp), **kw)
    return o


def test_host_batch_writer_is_byte_identical_to_oracle(ref, tmp_path):
    for world, rank in ((1, 0), (4, 3)):
        o = _opts(tmp_path, world=world, rank=rank, nccl_id=b"\0" * 128 if world > 1 else None)
        K = sum(ref.k_table(SIZES, o.density_ppm))
        rng = np.random.default_rng(world)
        blocks = rng.integers(0, 2**32, (3, 2 * K), dtype=np.uint64).astype(np.uint32)
        scal = [ld.derive_step_scalars(t, 1e-3) for t in (11, 12, 13)]
        ld.write_batch_host(SIZES, o, 11, scal, blocks)
        got = open(os.path.join(tmp_path, ref.batch_name(rank, 11)), "rb").read()
        want = ref.batch_serialize(rank, world, 11, SIZES, o.density_ppm, ref.ADAM, ref.FLAG_EF | ref.FLAG_MEAN,
                                   ref.adam_consts(), np.stack([ref.step_scalars(t, 1e-3) for t in (11, 12, 13)]),
                                   blocks)
        assert got == want


def test_host_full_writer_is_byte_identical_to_oracle(ref, tmp_path):
    psi = sum(SIZES)
    rng = np.random.default_rng(9)
    p, m, v = (rng.standard_normal(psi).astype(np.float32) for _ in range(3))
    for world in (1, 3):
        for rank in range(world):
            o = _opts(tmp_path, world=world, rank=rank, nccl_id=b"\0" * 128 if world > 1 else None)
            ld.write_full_host(SIZES, o, 5, p, m, v)
            got = open(os.path.join(tmp_path, ref.full_name(rank, 5)), "rb").read()
            assert got == ref.full_serialize(rank, world, 5, ref.ADAM, 3, ref.adam_consts(), p, m, v)
    o = _opts(tmp_path, optim=ld.SGD)
    ld.write_full_host(SIZES, o, 6, p)
    assert open(os.path.join(tmp_path, ref.full_name(0, 6)), "rb").read() == \
        ref.full_serialize(0, 1, 6, ref.SGD, 3, ref.adam_consts(), p)


def test_chain_scan_rules(ref, tmp_path):
    o = _opts(tmp_path)
    K = sum(ref.k_table(SIZES, o.density_ppm))
    psi = sum(SIZES)
    z = np.zeros(psi, np.float32)
    blk = lambda n: np.zeros((n, 2 * K), np.uint32)
    sc = lambda a, n: [ld.derive_step_scalars(t, 1e-3) for t in range(a, a + n)]
    with pytest.raises(ld.LowDiffError) as e:
        ld.chain_scan(SIZES, o)
    assert e.value.code == B.E_GAP                      # no full checkpoint at all
    ld.write_full_host(SIZES, o, 100, z, z, z)
    assert ld.chain_scan(SIZES, o) == (100, 100)        # Full@100 only
    ld.write_batch_host(SIZES, o, 101, sc(101, 20), blk(20))
    ld.write_batch_host(SIZES, o, 121, sc(121, 17), blk(17))
    assert ld.chain_scan(SIZES, o) == (100, 137)        # Full@100 + 101..137
    assert ld.chain_scan(SIZES, o, 120) == (100, 120)
    ld.write_batch_host(SIZES, o, 139, sc(139, 2), blk(2))
    assert ld.chain_scan(SIZES, o) == (100, 137)        # 138 missing: the chain stops
    with pytest.raises(ld.LowDiffError) as e:
        ld.chain_scan(SIZES, o, 140)
    assert e.value.code == B.E_GAP
    ld.write_full_host(SIZES, o, 130, z, z, z)
    assert ld.chain_scan(SIZES, o) == (130, 137)
    assert ld.chain_scan(SIZES, o, 129) == (100, 129)


def test_crash_mid_write_leaves_only_tmp_files_which_recovery_ignores(ref, tmp_path):
    """Writer crash consistency (SPEC.md:287 atomic persist): a file is written
    as *.tmp and renamed, so a crash mid-write leaves a partial *.tmp at most.  Partial *.tmp files
    of the next batch and of a newer full checkpoint change neither the library's chain scan nor
    the oracle's recovery, and a complete file written later under the same name supersedes them."""
    o = _opts(tmp_path)
    K = sum(ref.k_table(SIZES, o.density_ppm))
    psi = sum(SIZES)
    rng = np.random.default_rng(3)
    p0 = rng.standard_normal(psi).astype(np.float32)
    z = np.zeros(psi, np.float32)
    sc = lambda a, n: [ld.derive_step_scalars(t, 1e-3) for t in range(a, a + n)]
    blocks = []
    for _ in range(6):
        idx = np.sort(rng.choice(psi, K, replace=False)).astype(np.uint32)
        blocks.append(np.concatenate([idx, (rng.standard_normal(K) * 1e-2).astype(np.float32).view(np.uint32)]))
    blocks = np.stack(blocks)
    ld.write_full_host(SIZES, o, 0, p0, z, z)
    ld.write_batch_host(SIZES, o, 1, sc(1, 4), blocks[:4])
    want = ref.recover(tmp_path, 1, SIZES, o.density_ppm, -1)
    assert ld.chain_scan(SIZES, o) == (0, 4) and want[3] == 4
    # the crash: a partial next batch and a partial newer full checkpoint, as *.tmp
    full_bytes = open(tmp_path / ref.full_name(0, 0), "rb").read()
    (tmp_path / (ref.batch_name(0, 5) + ".tmp")).write_bytes(b"LDB1" + bytes(100))
    (tmp_path / (ref.full_name(0, 4) + ".tmp")).write_bytes(full_bytes[: len(full_bytes) // 3])
    assert ld.chain_scan(SIZES, o) == (0, 4)
    got = ref.recover(tmp_path, 1, SIZES, o.density_ppm, -1)
    assert got[3] == 4 and np.array_equal(got[0], want[0]) and np.array_equal(got[2], want[2])
    # after the restart the batch is written again, completely: the chain extends past the crash
    ld.write_batch_host(SIZES, o, 5, sc(5, 2), blocks[4:6])
    assert ld.chain_scan(SIZES, o) == (0, 6)
    assert ref.recover(tmp_path, 1, SIZES, o.density_ppm, -1)[3] == 6


def _gloo_worker(rank, world, port, tmp, q):
    import torch.distributed as dist
    import paper_2509_04084_b200 as ld2
    import oracle as ref2
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import torch
        # rank 0 makes the NCCL unique id and broadcasts it (the bootstrap lowdiff_create expects)
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt = torch.frombuffer(bytearray(ld2.nccl_unique_id()), dtype=torch.uint8).clone()
        dist.broadcast(idt, 0)
        nid = bytes(idt.tolist())
        o = ld2.Options(density_ppm=20000, ckpt_dir=tmp, world=world, rank=rank, nccl_id=nid)
        K = sum(ref2.k_table(SIZES, o.density_ppm))
        psi = sum(SIZES)
        rng = np.random.default_rng(0)   # same on every rank: the replicated state
        p = rng.standard_normal(psi).astype(np.float32)
        ld2.write_full_host(SIZES, o, 0, p, p * 0, p * 0)
        blocks = np.random.default_rng(100 + rank).integers(0, 2**32, (4, 2 * K), dtype=np.uint64).astype(np.uint32)
        ld2.write_batch_host(SIZES, o, 1, [ld2.derive_step_scalars(t, 1e-3) for t in range(1, 5)], blocks)
        dist.barrier()
        full, last = ld2.chain_scan(SIZES, o)
        dist.barrier()
        if rank == 1:
            os.remove(os.path.join(tmp, ref2.batch_name(0, 1)))
        dist.barrier()
        try:
            ld2.chain_scan(SIZES, o, 2)
            gap = None
        except ld2.LowDiffError as e:
            gap = e.code
        q.put((rank, full, last, gap, len(set(nid)) > 1))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e), None, None))


def test_two_rank_gloo_sharded_files_and_chain(tmp_path):
    """World-size-2 host path: NCCL-id bootstrap over torch.distributed (gloo), each rank writes its
    own shard and its own differential blocks, the chain is complete only with every rank's files."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, full, last, gap, idok in res:
        assert full == 0 and last == 4, res
        assert gap == B.E_GAP and idok
    files = sorted(os.listdir(tmp_path))
    assert "ld_full_r000_000000000000.ldf" in files and "ld_full_r001_000000000000.ldf" in files


@pytest.mark.parametrize("model", ["gpt2_xl", "bert_large", "resnet50", "mlp"])
@pytest.mark.parametrize("min_mb", [0, 1, 4, 64])
def test_bucket_plan_covers_backward_order_minimal_runs(model, min_mb):
    """LowDiff+ buckets: contiguous runs in backward order that tile the whole
    layer table; every bucket but the one holding layer 0 reaches min_bytes and is minimal (dropping
    its lowest layer falls below min_bytes), so the 6.4 KB LayerNorm/bias tensors never travel alone
    once min_bytes exceeds them."""
    from inputs import table
    sizes = table(model)
    mb = min_mb << 20
    plan = ld.bucket_plan(sizes, mb)
    assert plan[0][0] + plan[0][1] == len(sizes) and plan[-1][0] == 0
    for (f0, c0), (f1, c1) in zip(plan, plan[1:]):
        assert f1 + c1 == f0                                  # contiguous, descending
    for f, c in plan:
        assert c >= 1
        b = 4 * sum(sizes[f:f + c])
        if f > 0:
            assert b >= mb and (c == 1 or 4 * sum(sizes[f + 1:f + c]) < mb)
    if mb == 0:
        assert plan == [(l, 1) for l in range(len(sizes) - 1, -1, -1)]
    if mb >= 4 << 20 and model == "gpt2_xl":
        assert all(c > 1 or sizes[f] * 4 >= mb for f, c in plan[:-1])


def test_bucket_plan_errors():
    import ctypes as C
    L = B.lib()
    first, count, nb = (C.c_int32 * 4)(), (C.c_int32 * 4)(), C.c_int32()
    sizes = (C.c_int64 * 3)(10, 0, 5)
    assert L.lowdiff_bucket_plan(3, sizes, 16, first, count, 4, C.byref(nb)) == 1       # numel < 1
    sizes = (C.c_int64 * 3)(10, 10, 5)
    assert L.lowdiff_bucket_plan(3, sizes, 0, first, count, 2, C.byref(nb)) == 2        # cap too small
    assert L.lowdiff_bucket_plan(3, sizes, 0, first, count, 3, C.byref(nb)) == 0 and nb.value == 3
    assert L.lowdiff_bucket_plan(3, sizes, 10**9, first, count, 1, C.byref(nb)) == 0
    assert nb.value == 1 and (first[0], count[0]) == (0, 3)


def test_bench_reference_arm_prints_one_json_line():
    """`bench.py --impl reference` (the oracle arm the driver runs) prints one JSON line with the
    contract's keys, on the CPU (MLP workload to keep it short)."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "mlp",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "mlp@10000ppm"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def _run_blocks(ref, sizes, ppm, seed, ts):
    """Valid send blocks (oracle compress of seeded gradients, EF on) for iterations ts."""
    psi = sum(sizes)
    r = np.zeros(psi, np.float32)
    out = []
    for t in ts:
        g = np.random.default_rng([seed, t]).standard_normal(psi).astype(np.float32)
        blk, r = ref.compress(sizes, ppm, g, r, ef=True)
        out.append(blk)
    return np.stack(out)


def test_restart_retires_the_abandoned_run(ref, tmp_path):
    """after a recovery to iteration 6, persisting restarts at 7 with another batch
    alignment.  The abandoned run's files holding iterations >= 7 (…05.ldb covers 5..8, …09.ldb
    9..10) must not splice into the new chain.  lowdiff_retire_from(7) truncates …05 to 5..6 and
    removes …09; the oracle then recovers exactly Full@0 + old 1..6 + new 7..12."""
    o = _opts(tmp_path)
    ppm, psi = o.density_ppm, sum(SIZES)
    K = sum(ref.k_table(SIZES, ppm))
    rng = np.random.default_rng(5)
    p0 = rng.standard_normal(psi).astype(np.float32)
    z = np.zeros(psi, np.float32)
    ld.write_full_host(SIZES, o, 0, p0, z, z)
    old = _run_blocks(ref, SIZES, ppm, 1, range(1, 11))
    new = _run_blocks(ref, SIZES, ppm, 2, range(7, 13))
    sc = lambda a, n: [ld.derive_step_scalars(t, 1e-3) for t in range(a, a + n)]
    for a, n in ((1, 4), (5, 4), (9, 2)):                       # old run, b = 4
        ld.write_batch_host(SIZES, o, a, sc(a, n), old[a - 1:a - 1 + n])
    ld.write_full_host(SIZES, o, 8, z, z, z)                    # an old full checkpoint of a state >= 7
    # without retiring, the old …09 file (first 9 > 7) would override blocks 9, 10 of the new …07 file
    ld.retire_from(SIZES, o, 7)
    names = sorted(os.listdir(tmp_path))
    assert ref.batch_name(0, 9) not in names and ref.full_name(0, 8) not in names
    raw = open(os.path.join(tmp_path, ref.batch_name(0, 5)), "rb").read()
    assert raw == ref.batch_serialize(0, 1, 5, SIZES, ppm, ref.ADAM, ref.FLAG_EF | ref.FLAG_MEAN, ref.adam_consts(),
                                      np.stack([ref.step_scalars(t, 1e-3) for t in (5, 6)]), old[4:6])
    assert ld.chain_scan(SIZES, o) == (0, 6)
    for a, n in ((7, 3), (10, 3)):                              # new run, b = 3
        ld.write_batch_host(SIZES, o, a, sc(a, n), new[a - 7:a - 7 + n])
    assert ld.chain_scan(SIZES, o) == (0, 12)
    P, M, V = p0.copy(), z.copy(), z.copy()
    blocks = list(old[:6]) + list(new)
    for t, blk in zip(range(1, 13), blocks):
        ref.adam_step(ref.exchange(blk, 1, K, psi), ref.adam_consts(), ref.step_scalars(t, 1e-3), P, M, V)
    q, mq, vq, it = ref.recover(str(tmp_path), 1, SIZES, ppm)
    assert it == 12 and np.array_equal(q, P) and np.array_equal(mq, M) and np.array_equal(vq, V)
    # nothing at or after 13 exists: retiring there changes nothing; another rank's files are not touched
    before = {n: open(os.path.join(tmp_path, n), "rb").read() for n in os.listdir(tmp_path)}
    ld.retire_from(SIZES, o, 13)
    ld.retire_from(SIZES, _opts(tmp_path, world=2, rank=1, nccl_id=b"\0" * 128), 0)
    assert {n: open(os.path.join(tmp_path, n), "rb").read() for n in os.listdir(tmp_path)} == before
