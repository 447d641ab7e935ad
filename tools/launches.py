"""Summarise an ncu --csv launch list (per-launch device time, DRAM bytes) by kernel.

  python tools/launches.py gpurun_out/launches.csv [first_n]
Not part of the product: a reading aid for the profiles committed under profiles/.
"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
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


def main():
    ls = load(sys.argv[1])
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
