"""Summarise `ncu --set full` reports (.ncu-rep) into one CSV row per kernel launch.

  python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/rNN_ncu_full_summary.csv
Not part of the product: a reading aid for the profiles committed under profiles/.
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "GB"),
    ("dram__bytes_write.sum", "GB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    ("launch__registers_per_thread", ""),
    ("launch__grid_size", ""),
    ("launch__block_size", ""),
    ("lts__t_sectors_op_write.sum", "M"),
    ("smsp__inst_executed.sum", ""),
]
SCALE = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "KB": 1e-6, "MB": 1e-3, "GB": 1.0, "B": 1e-9}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    head, units, data = r[0], r[1], r[2:]
    res = []
    for d in data:
        row = {"kernel": d[head.index("Kernel Name")]}
        for m, unit in METRICS:
            if m not in head:
                row[m] = ""
                continue
            i = head.index(m)
            try:
                v = float(d[i].replace(",", ""))
            except ValueError:
                row[m] = d[i]
                continue
            if unit in ("ms", "GB"):
                v *= SCALE.get(units[i], 1.0)
            elif unit == "M":
                v /= 1e6
            row[m] = round(v, 6)
        res.append(row)
    return res


def main():
    w = csv.writer(sys.stdout)
    w.writerow(["kernel"] + [m for m, _ in METRICS])
    for p in sys.argv[1:]:
        for row in rows(p):
            w.writerow([row["kernel"]] + [row[m] for m, _ in METRICS])


if __name__ == "__main__":
    main()
