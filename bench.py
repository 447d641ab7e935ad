#!/usr/bin/env python
"""LowDiff hot-path benchmark (BASELINE.json metric: "compress+exchange+persist GB/s per iteration;
recovery replay params/s").

One step = one iteration of the per-iteration chain on every rank: lowdiff_compress (per-layer top-k
with error feedback) -> lowdiff_exchange (NCCL allgather + merge into the dense gradient) ->
lowdiff_batch_persist (D2H of the rank's own block into the pinned ring), on synthetic gradients
shaped like GPT-2 XL (BJ:10; 1,557,611,200 params, 580 tensors) at 1% density.  The timed region
ends when the last block has landed in host memory (lowdiff_wait_persist).  value = dense fp32
gradient bytes consumed per second by all ranks (4 * Psi * N / t_step).  Recovery replay (M2) is
timed in the same run and reported under "recovery".

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import gradient, table  # noqa: E402

METRIC = "compress+exchange+persist GB/s per iteration"
T_START = time.time()


def log(msg):
    """progress on stderr (elapsed wall seconds), so a slow leg is visible in the driver's log"""
    print(f"[bench {time.time() - T_START:7.1f}s] {msg}", file=sys.stderr, flush=True)
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "note": "fallback (B200_PROFILING.md)"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        d["note"] = "measured (MEASURED_PEAKS.json)"
        return d
    except OSError:
        return dict(PEAKS_FALLBACK)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.t.join(timeout=2)
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


def init_dist(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    return rank, world, local


def allmax(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def host_info():
    """The host the oracle is timed on (model, sockets x cores, SMT, NUMA, nproc)."""
    info = {"nproc": os.cpu_count()}
    try:
        txt = open("/proc/cpuinfo").read()
        models = [ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("model name")]
        info["model"] = models[0] if models else None
        info["sockets"] = len({ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("physical id")}) or None
        cores = {(a, b) for a, b in zip([ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("physical id")],
                                        [ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("core id")])}
        info["physical_cores"] = len(cores) or None
        info["smt"] = (len(models) // len(cores)) if cores else None
        info["numa_nodes"] = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])
    except (OSError, ValueError, ZeroDivisionError):
        pass
    return info


def workload_config(args, sizes, K, world):
    """The `config` object both arms print (same workload keys)."""
    psi = sum(sizes)
    return {"workload": f"{args.workload}@{args.ppm}ppm", "psi": psi, "layers": len(sizes), "k_total": K,
            "density_ppm": args.ppm, "batch_size": 4, "parallelism": f"dp{world}",
            "inputs": f"D4 row-sparse Gaussian, alpha=0.5 rank correlation; {N_GRADS} distinct gradient buffers of "
                      f"{4 * psi / 1e9:.2f} GB used in rotation (GPT-2 XL / BERT-L: > L2, no flush needed; "
                      "ResNet-50 / MLP: L2-resident, as the paper's small models would be)",
            "persist": "D2H of the rank's block into the pinned ring inside the timed region; "
                       "file writing measured separately (writer)"}


# --------------------------------------------------------------------------- oracle (CPU) legs
def oracle_sample(sizes_all, ppm, budget_s):
    """Time the oracle (as it stands, 1 thread) on a bounded sample of the workload: consecutive
    layers of the table starting after the embeddings, grown until ~budget_s of CPU work."""
    import oracle as ref
    ref.build()
    # calibrate on ~2M parameters
    start = 2
    cal = []
    n = 0
    i = start
    while n < 2_000_000 and i < len(sizes_all):
        cal.append(sizes_all[i])
        n += sizes_all[i]
        i += 1
    t_cal = _oracle_chain(ref, cal, ppm)[0]
    per_param = t_cal / sum(cal)
    target = max(sum(cal), int(budget_s / max(per_param, 1e-12)))
    sample, n, i = [], 0, start
    while i < len(sizes_all) and n + sizes_all[i] <= target:
        sample.append(sizes_all[i])
        n += sizes_all[i]
        i += 1
    if not sample:
        sample = cal
    t, K = _oracle_chain(ref, sample, ppm)
    return t, sample, (start, start + len(sample))


def _oracle_chain(ref, sizes, ppm):
    psi = sum(sizes)
    g = gradient(sizes, 0, 0, dist="D1", device="cpu").numpy()
    r = np.zeros(psi, np.float32)
    t0 = time.perf_counter()
    send, r = ref.compress(sizes, ppm, g, r, ef=True)
    K = send.size // 2
    ref.exchange(send, 1, K, psi)
    ref.batch_serialize(0, 1, 1, sizes, ppm, ref.ADAM, 3, ref.adam_consts(), ref.step_scalars(1, 1e-3)[None],
                        send[None])
    return time.perf_counter() - t0, K


def _oracle_part(args_):
    sizes, ppm = args_
    torch.set_num_threads(1)   # one core per worker process
    import oracle as ref
    return _oracle_chain(ref, sizes, ppm)[0]


def oracle_pool(n_sample_layers):
    """Worker processes for oracle_all_cores, one per host core (at most one per sample layer).
    spawn, not fork: a child forked from a process whose torch/OpenMP thread pool is live can
    deadlock on a lock held at the fork (seen on the GPU box: the leg never returned)."""
    import multiprocessing as mp
    cores = max(1, min(os.cpu_count() or 1, n_sample_layers))
    pool = mp.get_context("spawn").Pool(cores)
    pool.map(_oracle_part, [([64], 10000)] * cores)   # workers up, oracle loaded
    return pool, cores


def oracle_all_cores(sample, ppm, pool, cores):
    """The same oracle work on every host core: the sample's layers in `cores` size-balanced parts
    (compression is per layer, the merge per element), one process per part (the oracle is kept
    single-threaded as written).  Returns (wall seconds, cores used)."""
    parts = [[] for _ in range(cores)]
    load = [0] * cores
    for n in sorted(sample, reverse=True):   # greedy: largest layer to the least loaded part
        i = load.index(min(load))
        parts[i].append(n)
        load[i] += n
    parts = [p_ for p_ in parts if p_]
    t0 = time.perf_counter()
    pool.map(_oracle_part, [(p_, ppm) for p_ in parts])
    return time.perf_counter() - t0, len(parts)


def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sizes = table(args.workload)
    per_step_budget = max(0.5, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    import oracle as ref
    ref.build()
    _, sample, (a, b) = oracle_sample(sizes, args.ppm, per_step_budget)
    psi_s = sum(sample)
    for _ in range(args.warmup):
        _oracle_chain(ref, sample, args.ppm)
    times = [_oracle_chain(ref, sample, args.ppm)[0] for _ in range(args.steps)]
    t1 = sum(times) / len(times)
    # the host's cores: the same sample split over one oracle process per core
    pool, ncores = oracle_pool(len(sample))
    with pool:
        times_all = [oracle_all_cores(sample, args.ppm, pool, ncores) for _ in range(args.steps)]
    t = sum(x for x, _ in times_all) / len(times_all)
    cores = times_all[0][1]
    if t1 <= t:   # a sample too small to pay for the processes: the single thread is the baseline
        t, cores = t1, 1
    value = 4 * psi_s / t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, sizes, sum(ref.k_table(sizes, args.ppm)), args.gpus),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle", "host": host_info(),
                             "one_thread": {"value": 4 * psi_s / t1 / 1e9, "ms_per_step": t1 * 1e3},
                             "sample": f"{args.workload} layers [{a},{b}) = {psi_s} params per step "
                                       f"(compress + exchange + batch serialize, 1 rank), split over {cores} "
                                       "single-threaded oracle processes by layer"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
N_GRADS = 4      # distinct gradient buffers in rotation (a 2-periodic input biased the band)
EF_SETTLE = 20   # 20 warm-up iterations, which error feedback needs to reach steady state


def run_ours(args):
    import paper_2509_04084_b200 as ld

    # the first calls of a context admit 3-9x K candidates while the EF residual grows
    # (tools/spec_ratio.py); the JSON line reports the warm-up count actually run
    args.warmup = max(args.warmup, EF_SETTLE)

    rank, world, local = init_dist(args.gpus)
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    B_HBM = peaks["hbm_gbs"] * 1e9
    sizes = table(args.workload)
    psi = sum(sizes)
    nid = None
    if world > 1:
        import torch.distributed as dist
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(ld.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nid = bytes(t.cpu().tolist())
    tmp = tempfile.mkdtemp(prefix="lowdiff_bench_")
    ctx = ld.Context(sizes, density_ppm=args.ppm, rank=rank, world=world, nccl_id=nid, device=local,
                     ckpt_dir=tmp, batch_size=4, ring_slots=8, write_files=False, optim=ld.ADAM)
    K = ctx.K
    grads = [gradient(sizes, rank, i, dist="D4", alpha=0.5, model=args.workload, device=dev) for i in range(N_GRADS)]
    r = torch.zeros(psi, device=dev)
    dense = torch.empty(psi, device=dev)
    # double-buffered send blocks: the D2H of iteration t's block overlaps the
    # compress of t+1; the library makes a compress wait only for the D2H of the buffer it overwrites
    if args.exchange == "peer":
        # NEXT-1: the send slots are library-owned and mapped by every peer (CUDA IPC); the merge
        # reads the peers' blocks directly (no gathered buffer)
        if world > 1:
            sends = ctx.peer_setup(2)
        else:
            sends, _ = ctx.peer_alloc(2, handles=False)
            ctx.peer_set([ctx.peer_ptrs + [ctx.peer_flags_ptr]])
    else:
        sends = [torch.empty(2 * K, dtype=torch.int32, device=dev) for _ in range(2)]
    send = sends[0]
    gathered = torch.empty(world * 2 * K, dtype=torch.int32, device=dev) if world > 1 else None
    scal = [ld.derive_step_scalars(t, 1e-3) for t in range(1, args.warmup + 2 * args.steps + args.trace_calls + 60)]
    it = [0]

    def step(g=None):
        t = it[0]
        sd = sends[t % 2]
        ctx.compress(grads[t % N_GRADS] if g is None else g, r, sd)
        if args.persist_first:
            ctx.batch_persist(t + 1, scal[t], sd)   # D2H overlaps this exchange + the next compress
        if args.exchange == "peer":
            ctx.exchange_peer(t % 2, dense)
        else:
            ctx.exchange(sd, gathered, dense)
        if not args.persist_first:
            # Q.put after Sync (Alg. 1 l.5-6): the D2H overlaps the next compress, whose long scan
            # kernel covers it (a copy-engine D2H costs each kernel boundary it overlaps)
            ctx.batch_persist(t + 1, scal[t], sd)
        it[0] += 1
        return sd

    log("warm-up + timed steps")
    if not args.no_graphs:
        ctx.set_graphs(True)          # compress + merge replayed as captured CUDA graphs
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.sync()
    l0 = ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = Clocks(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    e0.record()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        step()
        marks[i].record()   # per-step spread (compute stream; the last block's D2H ends the region)
    ctx.wait_persist()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    raw = [e0.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i]) for i in range(1, args.steps)]
    per = sorted(raw)
    spread = {"p10": per[len(per) // 10], "p50": per[len(per) // 2], "p90": per[(9 * len(per)) // 10],
              "steps_ms": [round(x, 4) for x in raw],
              "note": "compute-stream time per step (event after each step); value uses the whole region"}
    barrier(world)
    ms = allmax(e0.elapsed_time(e1), world)
    launches = ctx.kernel_launches() - l0
    # per-kernel breakdown: a separate pass of the same steps with CUDA events recorded on the
    # launching streams (profiling replaces the graphs by plain launches; not the timed region)
    n_prof = max(3, min(args.steps, 10))
    ctx.prof_enable(True)
    for _ in range(n_prof):
        step()
    ctx.wait_persist()
    torch.cuda.synchronize()
    kern = {}
    for name in ("small_layer", "scan", "select", "emit", "merge", "peer_merge", "allgather", "d2h"):
        tot, n = ctx.prof_read(name)
        if n:
            kern[name] = {"ms_per_launch": tot / n, "launches": n, "share_of_step": tot / n_prof / (ms / args.steps)}
    ctx.prof_enable(False)
    # per-layer miss trace (lowdiff_compress_trace after each call of a further untimed run of the
    # same loop): which large layers left the speculative band and were refilled
    trace_calls = []
    for _ in range(max(args.trace_calls, 0)):
        step()
        _, lev, cand, _ = ctx.compress_trace()
        trace_calls.append({"refilled": int((lev == 1).sum()), "direct_segments": ctx.stats()["direct_segments"]})
    ctx.sync()
    st = ctx.stats()
    ms_step = ms / args.steps
    value = world * 4 * psi / (ms_step / 1e3) / 1e9

    # roofline of the dominant kernel: the scan (EF add + residual write + candidate compaction)
    psi_large = sum(n for n in sizes if n > 4096)   # layers above kSmallMax go through the scan
    scan_bytes = 12 * psi_large
    scan_ms = kern.get("scan", {}).get("ms_per_launch", float("nan"))
    achieved = scan_bytes / (scan_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"scan@{args.workload}")
    except (OSError, ValueError):
        pass
    roofline = {"kernel": "scan_kernel (lowdiff_compress pass A)", "bound": "hbm", "achieved": achieved,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "algorithmic_bytes_per_launch": scan_bytes, "peak_source": peaks["note"]}

    # live optimizer step from the gathered blocks (NEXT-1 second half): exchange_update never
    # materialises G; compared with exchange (merge) + a dense Adam step in the algorithmic-byte model
    update = None
    log("update (live merge + Adam)")
    if not args.no_update:
        p = torch.randn(psi, device=dev) * 0.02
        m = torch.zeros(psi, device=dev)
        v = torch.zeros(psi, device=dev)
        sd = sends[0]
        for t in range(2):
            ctx.exchange_update(sd, gathered, scal[t], p, m, v)
        torch.cuda.synchronize()
        n_u = 5
        u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        u0.record()
        for t in range(n_u):
            ctx.exchange_update(sd, gathered, scal[t + 2], p, m, v)
        u1.record()
        torch.cuda.synchronize()
        ums = allmax(u0.elapsed_time(u1), world) / n_u
        fused_b = 24 * psi + 8 * world * K
        unfused_b = (4 * psi + 8 * world * K) + 28 * psi
        update = {"ms_per_step": ums, "algorithmic_bytes": fused_b, "gbs": fused_b / (ums / 1e3) / 1e9,
                  "frac_of_hbm": fused_b / (ums / 1e3) / B_HBM,
                  "unfused_model_bytes": unfused_b, "unfused_floor_ms": unfused_b / B_HBM * 1e3,
                  "note": "allgather + update_kernel (tile merge in smem + streaming Adam); p, m, v fp32 in HBM"}
        if args.exchange == "peer":
            # NEXT-1 fully fused: the peers' entries read over peer memory straight into the tile merge
            # + Adam (lowdiff_exchange_peer_update): local HBM 24 B/param + this rank's own entries;
            # the other ranks' entries of each tile arrive over NVLink ((N - 1) 8 K bytes per step)
            for t in range(2):
                ctx.exchange_peer_update(0, scal[t], p, m, v)
            torch.cuda.synchronize()
            barrier(world)
            u0.record()
            for t in range(n_u):
                ctx.exchange_peer_update(0, scal[t + 2], p, m, v)
            u1.record()
            torch.cuda.synchronize()
            pms = allmax(u0.elapsed_time(u1), world) / n_u
            local_b = 24 * psi + 8 * K
            update["peer_fused"] = {"ms_per_step": pms, "local_hbm_bytes": local_b,
                                    "nvlink_bytes_in": 8 * K * (world - 1),
                                    "local_gbs": local_b / (pms / 1e3) / 1e9,
                                    "frac_of_hbm": local_b / (pms / 1e3) / B_HBM,
                                    "note": "lowdiff_exchange_peer_update: no gathered buffer, no dense G"}
        del p, m, v

    # BJ:5 gate: T_floor / t_chain; PCIe D2H bandwidth measured here
    # (one block-sized copy timed with CUDA events, best of 10 after a warm-up copy: a single
    # wall-clock sample of a 2 MB copy once read 2.8 GB/s and turned the gate into nonsense)
    host = torch.empty(2 * K, dtype=torch.int32, pin_memory=True)
    host.copy_(send, non_blocking=True)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ca.record()
        host.copy_(send, non_blocking=True)
        cb.record()
        cb.synchronize()
        best = min(best, ca.elapsed_time(cb) / 1e3)
    b_pcie = 8 * K / best
    t_c = (12 * psi + 8 * K) / B_HBM
    nvl = float(peaks.get("nvlink_gbs", 770.0))   # MEASURED_PEAKS.json has none: B200_PROFILING.md's measured
    t_ag = (world - 1) * 8 * K / (nvl * 1e9)       # peer copy, 770 GB/s per direction (unmeasurable on 1 GPU)
    t_m = (4 * psi + 8 * world * K) / B_HBM
    t_d2h = (8 * K + 32) / b_pcie
    t_floor = t_c + max(t_ag + t_m, t_d2h)
    t_pipe = max(t_c + t_ag + t_m, t_d2h)   # floor when the D2H of t overlaps the compress of t+1
    gate = {"t_floor_ms": t_floor * 1e3, "t_chain_ms": ms_step, "frac": t_floor / (ms_step / 1e3),
            "t_floor_pipelined_ms": t_pipe * 1e3, "frac_pipelined": t_pipe / (ms_step / 1e3),
            "pcie_d2h_gbs_measured": b_pcie / 1e9, "nvlink_gbs": nvl,
            "nvlink_source": ("MEASURED_PEAKS.json" if "nvlink_gbs" in peaks else
                              "B200_PROFILING.md measured peer copy (770 GB/s per direction); not measurable on the "
                              "1-GPU boxes of this round"),
            "note": "send blocks double-buffered: D2H(t) overlaps compress(t+1)"}

    # e2e: the same chain through the C ABI with the gradient in pinned HOST memory
    e2e = None
    log("e2e (host buffers)")
    if not args.no_e2e:
        hg = torch.empty(psi, dtype=torch.float32, pin_memory=True)
        hg.copy_(grads[0].cpu())
        hout = torch.empty(2 * K, dtype=torch.int32, pin_memory=True)
        # the H2D of step t+1's gradient (copy stream, double-buffered device gradient) overlaps
        # step t's chain, and the result's D2H runs on a third stream (PCIe is full duplex): every
        # step still moves its 4 Psi bytes in and its 8 K bytes out inside the timed region
        gbuf = [grads[1], grads[2]]
        cs_in, cs_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        comp = torch.cuda.current_stream(dev)
        n_e2e = max(2, min(args.steps, 4))
        gbuf[0].copy_(hg, non_blocking=True)
        step(gbuf[0])
        torch.cuda.synchronize()
        barrier(world)
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        out = [torch.cuda.Event() for _ in range(2)]
        done = torch.cuda.Event()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(comp)
        cs_in.wait_stream(comp)
        cs_out.wait_stream(comp)
        with torch.cuda.stream(cs_in):
            gbuf[0].copy_(hg, non_blocking=True)          # host -> device: step 0's gradient
            ready[0].record(cs_in)
        for i in range(n_e2e):
            b = i % 2
            if i + 1 < n_e2e:                             # host -> device: step i+1's, into the other buffer
                with torch.cuda.stream(cs_in):
                    if i >= 1:
                        cs_in.wait_event(free[1 - b])     # step i-1 has read that buffer
                    gbuf[1 - b].copy_(hg, non_blocking=True)
                    ready[1 - b].record(cs_in)
            comp.wait_event(ready[b])
            if i >= 2:
                comp.wait_event(out[b])                   # the send block this step overwrites is out
            sd = step(gbuf[b])
            free[b].record(comp)
            cs_out.wait_stream(comp)
            with torch.cuda.stream(cs_out):
                hout.copy_(sd, non_blocking=True)         # device -> host: this step's compressed result
                out[b].record(cs_out)
        ctx.wait_persist()
        done.record(cs_out)
        comp.wait_event(done)
        f1.record(comp)
        torch.cuda.synchronize()
        ems = allmax(f0.elapsed_time(f1), world) / n_e2e
        e2e = {"value": world * 4 * psi / (ems / 1e3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 4 * psi,
               "d2h_bytes_per_step": 8 * K, "ms_per_step": ems, "steps": n_e2e,
               "note": "H2D of step t+1 overlaps step t (double-buffered device gradient); result D2H on a third stream"}
        del hg, hout
    ctx.sync()

    # full checkpoint (a7): the producer waits only for the D2D stage of the rank's 12 Psi / N shard;
    # the D2H from the stage follows on the side stream (p, m, v stand-ins: the gradient buffers)
    fullck = None
    log("full checkpoint")
    if not args.no_full:
        fs = (psi * (rank + 1) // world) - (psi * rank // world)
        ctx.full_ckpt(0, grads[0], grads[1], grads[0])   # warm-up: allocates the stage and pinned host
        ctx.wait_persist()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        barrier(world)
        e0.record()
        ctx.full_ckpt(1, grads[0], grads[1], grads[0])
        e1.record()
        ctx.wait_persist()
        e2.record()
        torch.cuda.synchronize()
        stall = allmax(e0.elapsed_time(e1), world)
        done = allmax(e0.elapsed_time(e2), world)
        fullck = {"shard_bytes": 12 * fs, "producer_stall_ms": stall, "d2h_done_ms": done,
                  "stall_gbs": 12 * fs / (stall / 1e3) / 1e9, "d2h_gbs": 12 * fs / (done / 1e3) / 1e9,
                  "note": "producer waits for the D2D stage only (DESIGN.md 4.4); the D2H runs behind it"}

    # recovery replay (M2): n steps of gathered blocks resident in HBM, fused Adam replay
    recovery = None
    ctx.set_graphs(False)   # the recovery leg compresses into 100 different blocks: plain launches
    log("recovery replay")
    if not args.no_recovery:
        del dense
        step_bytes = world * 8 * K
        free, _ = torch.cuda.mem_get_info()
        n_rep = int(max(1, min(args.replay_steps, (free - 3 * 4 * psi - 2 * 2**30) * 0.8 // (step_bytes * 1.1))))
        diffs = torch.empty((n_rep, world * 2 * K), dtype=torch.int32, device=dev)
        dn = torch.empty(psi, device=dev)
        rsend = torch.empty(2 * K, dtype=torch.int32, device=dev)   # not a peer slot
        for t in range(n_rep):
            if world > 1:
                ctx.compress(grads[t % N_GRADS], r, rsend)
                ctx.exchange(rsend, diffs[t], dn)
            else:
                ctx.compress(grads[t % N_GRADS], r, diffs[t])
        del dn
        torch.cuda.synchronize()
        # sharded recovery (NEXT-2): every rank replays only its parameter range
        lo, hi = psi * rank // world, psi * (rank + 1) // world
        p = torch.randn(hi - lo, device=dev) * 0.02
        m = torch.zeros(hi - lo, device=dev)
        v = torch.zeros(hi - lo, device=dev)
        rscal = [ld.derive_step_scalars(t, 1e-3) for t in range(1, n_rep + 1)]
        ctx.replay_range(ld.ADAM, world, n_rep, diffs, rscal, lo, hi, p, m, v)   # warm-up (sizes the scratch)
        torch.cuda.synchronize()
        ctx.prof_enable(True)
        barrier(world)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        ctx.replay_range(ld.ADAM, world, n_rep, diffs, rscal, lo, hi, p, m, v)
        g1.record()
        torch.cuda.synchronize()
        rms = allmax(g0.elapsed_time(g1), world)
        rk_ms, _ = ctx.prof_read("replay")
        ri_ms, _ = ctx.prof_read("replay_index")
        ctx.prof_enable(False)
        t_rep = rms / 1e3
        S = hi - lo
        unfused = n_rep * (24 * S + 8 * world * K)
        fused = 24 * S + n_rep * 8 * world * K
        alu_peak = 148 * 128 * (peaks.get("sm_max_mhz", 1965.0) * 1e6)   # fp32 lane-instr/s
        recovery = {"metric": "recovery replay params/s", "value": n_rep * psi / t_rep,
                    "unit": "param-steps/s", "optimizer": "adam", "steps": n_rep, "ranks_per_step": world,
                    "sharded": f"each of {world} rank(s) replays its 1/{world} of Psi (lowdiff_replay_range)",
                    "ms": rms, "replay_kernel_ms": rk_ms, "index_kernel_ms": ri_ms,
                    "effective_unfused_gbs_per_rank": unfused / t_rep / 1e9,
                    "frac_of_hbm_unfused_model": unfused / t_rep / B_HBM,
                    "fused_algorithmic_gbs_per_rank": fused / t_rep / 1e9,
                    "alu_lane_instr_per_param_step_at_peak": alu_peak * t_rep / (n_rep * S)}
        # ncu's executed instructions of the same kernel (this round's capture, profiles/): the issue
        # bound at that count, and this run's fraction of it
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                ipp = json.load(f).get(f"replay_instr_per_param_step@{args.workload}")
        except (OSError, ValueError):
            ipp = None
        if ipp:
            recovery["ncu_thread_instr_per_param_step"] = ipp
            recovery["issue_bound_param_steps_per_s"] = alu_peak / ipp
            recovery["frac_of_issue_bound"] = (n_rep * psi / t_rep) / (alu_peak / ipp) if world == 1 else None
        # SGD replay of the same blocks (SURVEY §8(d) M2, C4 SGD row): HBM model n (8 S + 8 N K)
        ctx.replay_range(ld.SGD, world, n_rep, diffs, rscal, lo, hi, p)   # warm-up
        torch.cuda.synchronize()
        barrier(world)
        g0.record()
        ctx.replay_range(ld.SGD, world, n_rep, diffs, rscal, lo, hi, p)
        g1.record()
        torch.cuda.synchronize()
        sms_ = allmax(g0.elapsed_time(g1), world)
        unf_sgd = n_rep * (8 * S + 8 * world * K)
        recovery["sgd"] = {"value": n_rep * psi / (sms_ / 1e3), "unit": "param-steps/s", "steps": n_rep, "ms": sms_,
                           "effective_unfused_gbs_per_rank": unf_sgd / (sms_ / 1e3) / 1e9,
                           "frac_of_hbm_unfused_model": unf_sgd / (sms_ / 1e3) / B_HBM,
                           "fused_algorithmic_gbs_per_rank": (8 * S + n_rep * 8 * world * K) / (sms_ / 1e3) / 1e9}
        del diffs, p, m, v
        # C4's per-rank recovery work at N = 8 on this one GPU: every
        # step carries 8 ranks' blocks and this rank replays only its 1/8 of Psi (lowdiff_replay_range)
        if world == 1 and not args.no_c4_shape:
            W8 = 8
            torch.cuda.empty_cache()
            free, _ = torch.cuda.mem_get_info()
            n8 = int(max(1, min(args.replay_steps, (free - 4 * 2**30) * 0.85 // (W8 * 8 * K))))
            blk8 = torch.empty((W8, 2 * K), dtype=torch.int32, device=dev)
            for q in range(W8):   # 8 distinct blocks (the residual keeps evolving)
                ctx.compress(grads[q % N_GRADS], r, blk8[q])
            d8 = blk8.reshape(1, -1).expand(n8, -1).contiguous()   # the same 8 blocks at every step
            del blk8
            lo8, hi8 = 0, psi // W8
            S8 = hi8 - lo8
            p8 = torch.randn(S8, device=dev) * 0.02
            m8, v8 = torch.zeros(S8, device=dev), torch.zeros(S8, device=dev)
            sc8 = [ld.derive_step_scalars(t, 1e-3) for t in range(1, n8 + 1)]
            ctx.replay_range(ld.ADAM, W8, n8, d8, sc8, lo8, hi8, p8, m8, v8)   # warm-up
            torch.cuda.synchronize()
            g0.record()
            ctx.replay_range(ld.ADAM, W8, n8, d8, sc8, lo8, hi8, p8, m8, v8)
            g1.record()
            torch.cuda.synchronize()
            ms8 = g0.elapsed_time(g1)
            unf8 = n8 * (24 * S8 + 8 * W8 * K)
            recovery["c4_shape_rank_of_8"] = {
                "steps": n8, "ranks_per_step": W8, "range": [lo8, hi8], "ms": ms8,
                "param_steps_per_s_per_rank": n8 * S8 / (ms8 / 1e3),
                "param_steps_per_s_8_ranks": W8 * n8 * S8 / (ms8 / 1e3),
                "effective_unfused_gbs": unf8 / (ms8 / 1e3) / 1e9, "frac_of_hbm_unfused_model": unf8 / (ms8 / 1e3) / B_HBM,
                "note": "one rank's share of an 8-GPU recovery (8 ranks' blocks per step, 1/8 of Psi), timed on one GPU"}
            del d8, p8, m8, v8

    # recovery end to end from files (opt-in, --recovery-files n): Full@0 + n differentials written
    # by the library, then lowdiff_recover (chain scan, CRC checks, H2D, fused replay) timed by wall
    # clock; storage + PCIe + replay, reported beside the resident replay (M2)
    recovery_files = None
    if args.recovery_files and rank == 0:
        rdir = tempfile.mkdtemp(prefix="lowdiff_rf_")
        try:
            fctx = ld.Context(sizes, density_ppm=args.ppm, ckpt_dir=rdir, batch_size=4, optim=ld.ADAM)
            pf = torch.randn(psi, device=dev) * 0.02
            mf, vf = torch.zeros(psi, device=dev), torch.zeros(psi, device=dev)
            t_w0 = time.perf_counter()
            fctx.full_ckpt(0, pf, mf, vf)
            rf = torch.zeros(psi, device=dev)
            sf = torch.empty(2 * K, dtype=torch.int32, device=dev)
            for t in range(1, args.recovery_files + 1):
                fctx.compress(grads[t % 2], rf, sf)
                fctx.batch_persist(t, ld.derive_step_scalars(t, 1e-3), sf)
            fctx.sync()
            t_w = time.perf_counter() - t_w0
            del rf, sf
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            got = fctx.recover(pf, mf, vf)
            torch.cuda.synchronize()
            t_r = time.perf_counter() - t0
            fbytes = sum(os.path.getsize(os.path.join(rdir, f)) for f in os.listdir(rdir))
            recovery_files = {"steps": got, "seconds": t_r, "file_bytes": fbytes, "gbs": fbytes / t_r / 1e9,
                              "write_seconds": t_w,
                              "note": "lowdiff_recover from Full@0 + the .ldb chain on local storage (wall clock)"}
            fctx.close()
            del pf, mf, vf
        except Exception as exc:   # storage limits on the box: report, do not fail the bench line
            recovery_files = {"error": str(exc)[:200]}
        subprocess.run(["rm", "-rf", rdir])

    # writer throughput (files, CRC-32C, rename) on this box's storage, reported separately
    writer = None
    log("writer")
    if not args.no_writer and rank == 0:
        wdir = tempfile.mkdtemp(prefix="lowdiff_w_")
        wctx = ld.Context(sizes, density_ppm=args.ppm, ckpt_dir=wdir, batch_size=2, ring_slots=4, write_files=True)
        t0 = time.perf_counter()
        for t in range(1, 5):
            wctx.batch_persist(t, scal[t], send)
        wctx.sync()
        dt = time.perf_counter() - t0
        ws = wctx.stats()
        writer = {"files": ws["files_written"], "bytes": ws["bytes_written"], "seconds": dt,
                  "gbs": ws["bytes_written"] / dt / 1e9, "dir": "tempfile.mkdtemp()"}
        wctx.close()
        subprocess.run(["rm", "-rf", wdir])

    # LowDiff+ CPU replica: host Adam over one rank's shard of an 8-GPU job,
    # fed by the snapshot of the synced gradient (only the shard crosses PCIe); reported separately
    replica = None
    log("replica")
    if not args.no_replica and rank == 0:
        rw = 8
        rctx = ld.Context(sizes, density_ppm=args.ppm, world=rw, rank=0)
        S = psi // rw
        rp = torch.randn(S, device=dev)
        rm = torch.zeros(S, device=dev)
        rv = torch.zeros(S, device=dev)
        threads = max(1, min(32, os.cpu_count() or 1))
        rctx.replica_init(0, rp, rm, rv, threads=threads)
        n_w, n_r = 2, 4
        for t in range(1, n_w + 1):   # warm-up: pins both snapshot buffers
            rctx.snapshot_layer(t, 0, len(sizes), grads[t % 2])
            rctx.wait_persist()
            rctx.replica_step(t, scal[t])
        rctx.replica_wait()
        busy0 = rctx.stats()["replica_busy_ns"]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in range(n_w + 1, n_w + n_r + 1):
            rctx.snapshot_layer(t, 0, len(sizes), grads[t % 2])
            rctx.wait_persist()
            rctx.replica_step(t, scal[t])
        rctx.replica_wait()
        dt = time.perf_counter() - t0
        rs = rctx.stats()
        busy = (rs["replica_busy_ns"] - busy0) / 1e9 / n_r
        replica = {"shard_params": S, "of_world": rw, "threads": threads, "steps": n_r,
                   "host_adam_ms_per_step": busy * 1e3, "pipeline_ms_per_step": dt / n_r * 1e3,
                   "stall_ms_total": rs["replica_stall_ns"] / 1e6,
                   "snapshot_bytes_per_step": 4 * S,
                   "host_param_steps_per_s": S / busy if busy > 0 else None,
                   "host_algorithmic_gbs": 28 * S / busy / 1e9 if busy > 0 else None,
                   "bytes_model": "28 B/param-step: G read 4 + p, m, v read+write 24 (host DRAM)"}
        rctx.close()
        del rp, rm, rv

    # union-compacted differentials (NEXT-4): the union of 8 ranks' blocks (8 simulated ranks with
    # rank-correlated gradients, D4 with alpha = 0.5) compacted over rank 0's shard and over all of Psi
    union = None
    log("union")
    if not args.no_union and rank == 0:
        NU = 8
        uctx = ld.Context(sizes, density_ppm=args.ppm, world=NU, rank=0, device=local)
        g8 = torch.empty(NU * 2 * K, dtype=torch.int32, device=dev)
        rz = torch.zeros(psi, device=dev)
        for q in range(NU):
            gq = gradient(sizes, q, 0, dist="D4", alpha=0.5, model=args.workload, device=dev)
            rz.zero_()
            uctx.compress(gq, rz, g8[q * 2 * K:(q + 1) * 2 * K])
            del gq
        del rz
        res_u = {}
        for name, (lo, hi) in (("shard0", (0, psi // NU)), ("all", (0, psi))):
            cap = min(NU * K, hi - lo)
            out = torch.empty(2 * cap, dtype=torch.int32, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            uctx.union_compact(NU, g8, lo, hi, out, cap, cnt)
            torch.cuda.synchronize()
            u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            u0.record()
            for _ in range(5):
                uctx.union_compact(NU, g8, lo, hi, out, cap, cnt)
            u1.record()
            torch.cuda.synchronize()
            ums = u0.elapsed_time(u1) / 5
            n_u = int(cnt.item())
            share = NU * K * (hi - lo) / psi          # gathered entries falling in the range (expected)
            alg = 8 * share + 8 * n_u                 # gathered entries in range read once + union written
            res_u[name] = {"range": [lo, hi], "entries": n_u, "ms": ums,
                           "bytes_union": 8 * n_u, "bytes_gathered_share": int(8 * share),
                           "ratio_to_gathered": n_u / share, "algorithmic_gbs": alg / (ums / 1e3) / 1e9}
            del out, cnt
        uctx.close()
        del g8
        union = {"ranks": NU, "inputs": "D4, alpha = 0.5 rank correlation, one iteration per rank", **res_u,
                 "note": "union = indices of any rank's block with the merged value (R-29); persisted per shard"}

    # M3: LowDiff+ layer-wise dense snapshot.  A proxy backward pass (not our
    # code: torch copies, HBM-bound, duration proportional to each bucket's size) finalises the
    # gradient bucket by bucket in backward order; after each bucket lowdiff_snapshot_layer queues
    # its D2H.  M3 = dense bytes / (last D2H done - first bucket ready); interference = slowdown of
    # the proxy backward while the snapshots stream out over PCIe.
    snapshot = None
    log("snapshot")
    if not args.no_snapshot:
        plan = ld.bucket_plan(sizes, 4 << 20)
        offs = [0]
        for n_ in sizes:
            offs.append(offs[-1] + n_)
        sctx = ld.Context(sizes, density_ppm=args.ppm, rank=rank, world=1, device=local)
        g = grads[0]
        scratch = torch.empty(max(offs[f + c] - offs[f] for f, c in plan), device=dev)
        reps = args.snapshot_reps

        def backward(t, snap):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            for i, (f, c) in enumerate(plan):
                a, b = offs[f], offs[f + c]
                for _ in range(reps):   # an SM kernel (copy_ would use the copy engines the D2H needs)
                    torch.mul(g[a:b], 1.0, out=scratch[:b - a])
                if i == 0:
                    ev[1].record()
                if snap:
                    sctx.snapshot_layer(t, f, c, g[a:b])
            ev[2].record()
            if snap:
                sctx.wait_persist()
            ev[3].record()
            return ev

        backward(1, True)                 # warm-up: pins the snapshot buffers
        backward(2, True)
        torch.cuda.synchronize()
        alone, with_snap, m3 = [], [], []
        for t in range(3, 6):
            ev = backward(t, False)
            torch.cuda.synchronize()
            alone.append(ev[0].elapsed_time(ev[2]))
            ev = backward(t, True)
            torch.cuda.synchronize()
            with_snap.append(ev[0].elapsed_time(ev[2]))
            m3.append(ev[1].elapsed_time(ev[3]))
        sctx.snapshot_wait(5)
        sctx.close()
        # sharded: as rank 0 of 8, only its 1/8 of every bucket crosses PCIe
        sctx = ld.Context(sizes, density_ppm=args.ppm, rank=0, world=8, device=local)
        sctx.snapshot_shard(True)
        backward(1, True)
        backward(2, True)
        torch.cuda.synchronize()
        m3s, with_s = [], []
        for t in range(3, 6):
            ev = backward(t, True)
            torch.cuda.synchronize()
            with_s.append(ev[0].elapsed_time(ev[2]))
            m3s.append(ev[1].elapsed_time(ev[3]))
        sctx.close()
        del scratch
        shard_bytes = 4 * (psi // 8)
        t_m3s = allmax(statistics.median(m3s), world)
        t_m3 = allmax(statistics.median(m3), world)
        t_a, t_w = statistics.median(alone), statistics.median(with_snap)
        snapshot = {"metric": "LowDiff+ snapshot GB/s", "value": 4 * psi / (t_m3 / 1e3) / 1e9, "unit": "GB/s",
                    "bytes_per_iteration": 4 * psi, "buckets": len(plan), "min_bucket_bytes": 4 << 20,
                    "first_ready_to_last_d2h_ms": t_m3, "frac_of_pcie_measured": 4 * psi / (t_m3 / 1e3) / b_pcie,
                    "proxy_backward_ms_alone": t_a, "proxy_backward_ms_with_snapshot": t_w,
                    "interference": t_w / t_a - 1.0,
                    "proxy": f"{reps} torch.mul(g, 1.0) kernels over each bucket's gradient (8 B/param each), backward order",
                    "sharding": "unsharded: every rank copies all of its dense gradient",
                    "sharded_1_of_8": {"bytes_per_iteration": shard_bytes, "first_ready_to_last_d2h_ms": t_m3s,
                                       "gbs": shard_bytes / (t_m3s / 1e3) / 1e9,
                                       "proxy_backward_ms_with_snapshot": statistics.median(with_s),
                                       "interference": statistics.median(with_s) / t_a - 1.0,
                                       "note": "lowdiff_snapshot_shard: rank 0 of 8 copies its 1/8 of each bucket"}}

    log("cpu baseline (oracle)")
    cpu = None
    if rank == 0 and not args.no_cpu:   # (N > 1: rank 0 alone, on the same bounded sample)
        t_o, sample, (a, b) = oracle_sample(sizes, args.ppm, args.cpu_budget)
        pool, ncores = oracle_pool(len(sample))
        with pool:
            t_all, cores = oracle_all_cores(sample, args.ppm, pool, ncores)
        if t_o <= t_all:
            t_all, cores = t_o, 1
        cpu = {"value": 4 * sum(sample) / t_all / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
               "host": host_info(), "one_thread": {"value": 4 * sum(sample) / t_o / 1e9, "seconds": t_o},
               "sample": f"{args.workload} layers [{a},{b}) = {sum(sample)} params, one iteration of compress "
                         f"+ exchange + batch serialize: {t_o:.1f} s on 1 thread, {t_all:.1f} s split by layer "
                         f"over {cores} single-threaded oracle processes (value)"}

    ctx.close()
    subprocess.run(["rm", "-rf", tmp])
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "warmup_note": f"at least {EF_SETTLE} untimed iterations (EF steady state, SURVEY 8(d) M1)",
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload_config(args, sizes, K, world), "exchange": args.exchange,
                       "cuda_graphs": not args.no_graphs},
            "roofline": roofline, "gate_bj5": gate, "kernels": kern, "per_step_ms": spread, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk, "recovery": recovery, "writer": writer, "full_ckpt": fullck, "update": update,
            "replica": replica, "snapshot": snapshot, "union": union, "recovery_files": recovery_files,
            "spec": {"hits": st["spec_hits"], "misses": st["spec_misses"],
                     "trace": {"calls": len(trace_calls),
                               "calls_with_a_miss": sum(1 for t in trace_calls if t["refilled"]),
                               "refilled_layers": sum(t["refilled"] for t in trace_calls),
                               "direct_segments_per_call": [t["direct_segments"] for t in trace_calls]}},
            "scratch": {"compress_scratch_bytes": st["compress_scratch_bytes"],
                        "compress_scratch_bytes_per_param": st["compress_scratch_bytes"] / psi,
                        "library_device_bytes": st["device_bytes"],
                        "note": "bounded candidate slots (DESIGN.md 4.1) + plan; library_device_bytes adds the "
                                "merge/replay scratch and the full-checkpoint stage allocated so far"}}
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: one rank per GPU via torch.distributed.run
    on this node (the driver's own launch form), or a loud failure when the node has fewer GPUs."""
    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but this node has {n_dev} CUDA device(s); refusing to run "
              f"{args.gpus} ranks on fewer GPUs", file=sys.stderr, flush=True)
        sys.exit(2)
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="gpt2_xl", choices=["gpt2_xl", "bert_large", "resnet50", "mlp"])
    ap.add_argument("--ppm", type=int, default=10000)
    ap.add_argument("--replay-steps", type=int, default=100)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-recovery", action="store_true")
    ap.add_argument("--no-c4-shape", action="store_true", help="skip the 8-ranks-per-step replay leg")
    ap.add_argument("--no-writer", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-replica", action="store_true")
    ap.add_argument("--no-full", action="store_true")
    ap.add_argument("--no-update", action="store_true")
    ap.add_argument("--no-snapshot", action="store_true")
    ap.add_argument("--no-union", action="store_true")
    ap.add_argument("--trace-calls", type=int, default=40,
                    help="untimed calls after the timed region whose per-layer refill trace is reported")
    ap.add_argument("--recovery-files", type=int, default=0,
                    help="n > 0: also time lowdiff_recover from Full@0 + n differentials on local storage")
    ap.add_argument("--no-graphs", action="store_true", help="plain launches instead of captured CUDA graphs")
    ap.add_argument("--persist-first", action="store_true",
                    help="issue the block's D2H before the exchange instead of after it")
    ap.add_argument("--snapshot-reps", type=int, default=20,
                    help="proxy backward: HBM passes over each bucket (20 ~ 38 ms for GPT-2 XL, about the backward "
                         "of 8K tokens at ~1.2 PFLOP/s)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="nccl: ncclAllGather + merge; peer: merge reading the peers' slots (NEXT-1)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        spawn_ranks(args)   # (the reference arm runs on rank 0 only: nothing to spawn)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
