"""Summarise an ncu --csv launch list (per-launch device time, DRAM bytes) by kernel.

  python tools/launches.py gpurun_out/launches.csv [first_n | agg]
Not part of the product: a reading aid for the profiles committed under profiles/.
"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "%": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = collections.OrderedDict()
    for r in data:
        d = launches.setdefault(r[idi], {"name": r[ki].split("(")[0].split("<")[0].replace("void ", "")
                                         .replace("(anonymous namespace)::", "").split("::")[-1]})
        d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    return list(launches.values())


def aggregate(ls):
    """Per kernel name: launches, mean us, share of the summed device time, DRAM GB per launch."""
    agg = collections.OrderedDict()
    for d in ls:
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"{'kernel':24s} {'n':>5s} {'mean us':>10s} {'share':>7s} {'DRAM GB/launch':>15s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:24s} {n:5d} {t / n:10.1f} {t / tot:7.3f} {b / n:15.3f}")


def main():
    ls = load(sys.argv[1])
    if len(sys.argv) > 2 and sys.argv[2] == "agg":
        aggregate(ls)
        return
    n = int(sys.argv[2]) if len(sys.argv) > 2 else len(ls)
    print(f"{'kernel':24s} {'us':>10s} {'read GB':>9s} {'write GB':>9s} {'GB/s':>8s} {'warps%':>7s}")
    for d in ls[:n]:
        t = d.get("gpu__time_duration.sum", 0.0)
        rb, wb = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        bw = (rb + wb) / (t * 1e-6) if t else 0.0
        print(f"{d['name']:24s} {t:10.1f} {rb:9.3f} {wb:9.3f} {bw:8.0f} "
              f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0.0):7.1f}")


if __name__ == "__main__":
    main()
