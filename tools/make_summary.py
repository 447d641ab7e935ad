"""Regenerate profiles/r01_summary.md from the committed bench lines and ncu summaries (not product).

  python tools/make_summary.py
"""
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def load(name):
    with open(os.path.join(P, name)) as f:
        return json.load(f)


def main():
    d = load("r01_bench_gpt2xl.json")
    rows = {}
    for r in csv.DictReader(open(os.path.join(P, "r01_ncu_full_summary.csv"))):
        rows[r["kernel"].split("(")[0].split("::")[-1].split("<")[0]] = r

    def g(k, m):
        try:
            return float(rows[k][m])
        except (KeyError, ValueError):
            return float("nan")

    cfg = {f: load(f"r01_bench_{f}.json") for f in ["resnet50", "bert_large", "gpt2_1000", "gpt2_2500", "gpt2_5000"]}
    rf = load("r01_bench_recovery_files_gpt2xl.json")["recovery_files"]
    k, rec, sn, un = d["kernels"], d["recovery"], d["snapshot"], d["union"]
    sh = sn["sharded_1_of_8"]
    t = f"""# Round 1 profile summary (B200, sm_100a)

All numbers: one B200 (148 SMs, SM clock {d['clocks']['sm_mhz']:.0f} MHz under load, no throttle reasons), GPT-2 XL
layer table (Ψ = 1,557,611,200, 580 tensors), density 1% (K = 15,576,112), error feedback on, D4
synthetic gradients, CUDA graphs on, unless a config says otherwise. Peaks from `MEASURED_PEAKS.json`
(HBM copy {d['roofline']['peak']} GB/s, "of measured"). Regenerate with `python tools/make_summary.py`.

Files (all from the same code, final refresh of round 1):
- `r01_bench_gpt2xl.json` — the default `bench.py --steps 20` line (every leg; 20 warm-up iterations).
- `r01_bench_{{resnet50,bert_large,gpt2_1000,gpt2_2500,gpt2_5000}}.json` — `tools/run_configs.sh`:
  C2, C3 and the C4 density sweep (0.1 / 0.25 / 0.5%); `r01_bench_snapshot_gpt2xl.json` — M3 leg;
  `r01_bench_recovery_files_gpt2xl.json` — `--recovery-files 100` (recovery from local files).
- `r01_launches_gpt2xl.csv` — ncu launch list (`gpu__time_duration.sum`, DRAM bytes, warps active;
  `--clock-control none`, serialised cold-cache launches; our kernels only, steady state);
  `r01_launches_gpt2xl_agg.txt` = its per-kernel aggregate (`python tools/launches.py … agg`).
- `r01_ncu_full_summary.csv` — `ncu --set full` of scan / chunk_prep / emit / merge1 / update /
  replay / union, one steady-state launch each (call 21 of the step loop) (`python tools/ncu_summary.py …`).
- `ncu_traffic.json` — DRAM bytes per scan launch (feeds `roofline.traffic`).
- `r01_stream_probe*.txt` — achievable HBM bandwidth for the access patterns (copy 6.77 TB/s,
  `r += g` 7.11 TB/s, 2-stream read 7.40 TB/s with full grids).
- `r01_d2h_interference_probe.txt` — what a concurrent D2H does to HBM-bound kernels (a cost per
  kernel boundary, DESIGN.md §4.4); `r01_sanitizer.txt` — compute-sanitizer memcheck / racecheck /
  synccheck / initcheck; `r01_pdl_ab.txt` — A/B records of the late variants (programmatic
  dependent launch adopted; persistent merge, wider tile index grid, candidate unroll 8 dropped).

## Bench line (bench.py, N = 1)

| quantity | value |
|---|---|
| M1 compress+exchange+persist | **{d['value']:.0f} GB/s** of dense gradient ({d['ms_per_step']:.2f} ms per iteration; p10/p50/p90 {d['per_step_ms']['p10']:.2f}/{d['per_step_ms']['p50']:.2f}/{d['per_step_ms']['p90']:.2f} ms) |
| BJ:5 gate `T_floor / t_chain` (PCIe {d['gate_bj5']['pcie_d2h_gbs_measured']:.1f} GB/s measured) | **{d['gate_bj5']['frac']:.2f}** (≥ 0.60; above 1 because the D2H of t overlaps the compress of t+1) |
| same against the pipelined floor `max(t_c + t_m, t_d2h)` | {d['gate_bj5']['frac_pipelined']:.2f} |
| e2e (gradient H2D from pinned host each step) | {d['e2e']['value']:.1f} GB/s — PCIe bound (6.23 GB H2D per step) |
| M2 recovery: fused Adam replay, 100 steps resident | **{rec['value']:.3g} param-steps/s** ({rec['ms']:.0f} ms); {rec['effective_unfused_gbs_per_rank']/1e3:.1f} TB/s under the unfused per-step byte model = {rec['frac_of_hbm_unfused_model']:.2f}× HBM (gate ≥ 0.5) |
| M2 SGD replay, 100 steps | {rec['sgd']['ms']:.0f} ms ({rec['sgd']['value']:.3g} param-steps/s, {rec['sgd']['frac_of_hbm_unfused_model']:.2f}× the unfused HBM model) |
| recovery end to end from local files (Full@0 + 100 differentials, {rf['file_bytes']/1e9:.1f} GB) | {rf['seconds']:.2f} s ({rf['gbs']:.1f} GB/s; chain scan, CRC, H2D, replay) |
| live update (`exchange_update`: merge + Adam, no dense G) | {d['update']['ms_per_step']:.2f} ms, {d['update']['gbs']/1e3:.2f} TB/s algorithmic = {d['update']['frac_of_hbm']:.2f} of the HBM copy peak |
| full checkpoint (18.7 GB at N = 1) | producer held {d['full_ckpt']['producer_stall_ms']:.2f} ms (D2D stage); D2H done after {d['full_ckpt']['d2h_done_ms']:.0f} ms |
| M3 LowDiff+ snapshot (194 buckets ≥ 4 MB) | {sn['value']:.1f} GB/s = {sn['frac_of_pcie_measured']:.2f} of measured PCIe; proxy backward {sn['proxy_backward_ms_alone']:.1f} → {sn['proxy_backward_ms_with_snapshot']:.1f} ms while it streams |
| M3 sharded (rank 0 of 8 copies its 1/8) | {sh['bytes_per_iteration']/1e9:.2f} GB per iteration; proxy backward interference {100*sh['interference']:.0f}% (paper: 8.2–10.1%) |
| union-compacted differential, 8 ranks, α = 0.5 | {un['shard0']['ratio_to_gathered']:.2f} of the 8 fixed-K blocks; shard compaction {un['shard0']['ms']:.2f} ms, all of Ψ {un['all']['ms']:.2f} ms |
| CPU replica (1/8 shard, {d['replica']['threads']} threads) | {d['replica']['host_adam_ms_per_step']:.1f} ms host Adam per step |
| writer (CRC-32C + writev + rename to local disk) | {d['writer']['gbs']:.2f} GB/s |
| oracle, 1 thread | {d['cpu_baseline']['value']:.3f} GB/s ({d['cpu_baseline']['sample']}) |

## Dominant kernel: `scan_kernel<EF=1, REFILL=0>` (lowdiff_compress pass A)

| metric | value |
|---|---|
| duration | bench CUDA events {k['scan']['ms_per_launch']:.2f} ms avg; ncu full set {g('scan_kernel','gpu__time_duration.sum'):.2f} ms |
| share of the step | {k['scan']['share_of_step']:.2f} (bench events) / 0.67 of our summed device time (launch list) |
| DRAM read / write | {g('scan_kernel','dram__bytes_read.sum'):.2f} GB / {g('scan_kernel','dram__bytes_write.sum'):.2f} GB per launch (algorithmic 12Ψ_large = 18.69 GB; +2.8%: candidates) |
| achieved (algorithmic bytes / event time) | **{d['roofline']['achieved']/1e3:.2f} TB/s = {d['roofline']['frac']:.2f} of measured HBM peak** |
| warps active / issue active | {g('scan_kernel','sm__warps_active.avg.pct_of_peak_sustained_active'):.0f}% / {g('scan_kernel','smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f}% |
| registers | {g('scan_kernel','launch__registers_per_thread'):.0f} (full occupancy: 16 CTAs × 4 warps per SM) |

Evolution of this kernel in round 1 (same workload, bench events):

| variant | scan ms | frac of HBM |
|---|---|---|
| 512-thread CTA per chunk, registers, 3 block barriers, CTA-ordered compaction | 4.27 | 0.67 |
| TMA (cp.async.bulk + mbarrier) 3-stage ring, persistent, block-ordered compaction | 4.79 | 0.60 |
| warp-specialised TMA producer + 16 consumer warps, per-warp segments | 4.47 | 0.64 |
| full-grid streaming, 256-element warp segments, 2×32-bit candidate arrays | 3.96 | 0.72 |
| 1024-element segments, 64-bit interleaved candidates | 3.62 | 0.79 |
| + chunk-local 32-bit offsets, 1 float4/lane/round, 32 registers | 3.15 | 0.90 |
| + candidates staged per warp in smem, 256-byte runs (L2 write sectors 308 M → 235 M) | 3.12 | 0.91 |
| + round r+1's loads issued before round r is processed (31 registers) | **3.06** | **0.92** |
| (tried) L2 prefetch of the warp's whole segment at its start | 3.18 | 0.90 |
| (tried) 2 / 8 / 16 warps per CTA | 3.09 / 3.14 / 3.16 | ≤ 0.92 |
| (tried) the prefetch with 40 / 48 registers (12 / 10 CTAs per SM) | 3.22 / 3.44 | 0.87 / 0.82 |

The probes explain the ordering: a plain full-grid `r = r + g` reaches 7.1 TB/s, and everything
that lowers resident warps (registers, block barriers, persistent CTAs with serial phases) costs
bandwidth; TMA staging added barrier/latency structure without adding bytes in flight.

## Per-iteration chain (ms per launch; a separate profiled pass, plain launches)

| stage | ms | note |
|---|---|---|
| small_layer (layers ≤ 4096) | {k['small_layer']['ms_per_launch']:.2f} | forked stream, concurrent with the scan |
| scan | {k['scan']['ms_per_launch']:.2f} | above |
| select (prep, find, 2 digit, count, layer scan; refill grids) | {k['select']['ms_per_launch']:.2f} | ~1.5 k candidates per k; includes launch gaps of the profiled pass |
| emit | {k['emit']['ms_per_launch']:.2f} | lazy residual zeroing: no scattered writes |
| merge (tile index + merge1) | {k['merge']['ms_per_launch']:.2f} | 6.18 GB written at {6.18 / (k['merge']['ms_per_launch'] / 1e3) / 1e3:.1f} TB/s (write-only stream) |
| D2H of the 124.6 MB block | {k['d2h']['ms_per_launch']:.2f} (side stream) | overlapped with the next compress (double-buffered send blocks) |

## Other configs (tools/run_configs.sh; same bench, N = 1, CUDA graphs on)

| config | ms / step (p10–p90) | BJ:5 gate | scan frac of HBM | 100-step Adam replay |
|---|---|---|---|---|
"""
    names = {"resnet50": "C2 ResNet-50 1%", "bert_large": "C3 BERT-large 1%", "gpt2_5000": "C4 GPT-2 XL 0.5%",
             "gpt2_2500": "C4 GPT-2 XL 0.25%", "gpt2_1000": "C4 GPT-2 XL 0.1%"}
    for f in ["resnet50", "bert_large", "gpt2_5000", "gpt2_2500", "gpt2_1000"]:
        x = cfg[f]
        t += (f"| {names[f]} | {x['ms_per_step']:.3f} ({x['per_step_ms']['p10']:.3f}–{x['per_step_ms']['p90']:.3f}) | "
              f"{x['gate_bj5']['frac']:.2f} | {x['roofline']['frac']:.2f} | {x['recovery']['ms']:.1f} ms |\n")
    t += f"""| C4 GPT-2 XL 1% (default line) | {d['ms_per_step']:.3f} ({d['per_step_ms']['p10']:.3f}–{d['per_step_ms']['p90']:.3f}) | {d['gate_bj5']['frac']:.2f} | {d['roofline']['frac']:.2f} | {rec['ms']:.1f} ms |

ResNet-50 sits just below the gate (0.53 with the PCIe rate timed by CUDA events, best of 10; earlier
lines read 0.57–0.68 against a slower wall-clock PCIe sample, which inflated the floor): its 17
dependent kernels per step take 3–50 µs each
(latency, not bytes), the CUDA graphs remove the launch gaps (197 → 168–182 µs), and the block's
D2H, which overlaps the next compress, adds a cost per kernel boundary while it is in flight
(DESIGN.md §4.4). Its replay of 20 Adam steps at N = 8 (gate ≤ 3.15 ms) is far inside the bound.

## Recovery replay (`replay_kernel<Adam>`)

{rec['ms']:.0f} ms for 100 steps over 1.56 G params ({rec['value']:.3g} param-steps/s). ncu (10-step capture):
issue active {g('replay_kernel','smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f}%, warps active {g('replay_kernel','sm__warps_active.avg.pct_of_peak_sustained_active'):.0f}%, {g('replay_kernel','launch__registers_per_thread'):.0f} registers,
DRAM {(g('replay_kernel','dram__bytes_read.sum') + g('replay_kernel','dram__bytes_write.sum')):.1f} GB per 10 steps (ALU-bound). Round-1 path: 480 → 304 (paired fp32) → 265 (paired
adds through an opaque −0 FMA addend) → 255 (selp) → 216 (128 threads × 16 elements, warp-synchronous
steps) → 208 ms kernel (fmax clamp instead of a select). ~40 thread-instructions per param-step;
the fp32 issue bound at that count is 0.91 T param-steps/s, measured {rec['value']/1e12:.2f} T.

## Oracle (CPU)

`cpu_baseline`: the oracle as it stands (sort-based top-k, bitwise CRC, one thread) on a bounded
sample of the same workload: {d['cpu_baseline']['value']:.3f} GB/s on {d['cpu_baseline']['host'].get('model')}
({d['cpu_baseline']['host'].get('nproc')} threads available, 1 used). The GPU/oracle ratio (~{d['value'] / d['cpu_baseline']['value']:,.0f}×) says
nothing about kernel quality; the roofline fraction does.
"""
    with open(os.path.join(P, "r01_summary.md"), "w") as f:
        f.write(t)


if __name__ == "__main__":
    main()
