"""Summarise an ncu report (raw page) or an ncu launch-list CSV into profiles/.

    python tools/ncu_summary.py full  <report.ncu-rep> <out.csv>
    python tools/ncu_summary.py list  <launches.csv>   <out.csv>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    idx = [h.index(k) if k in h else None for k in KEYS]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([f"{k} [{units[i]}]" if i is not None and units[i] else k for k, i in zip(KEYS, idx)])
        for r in data:
            w.writerow([r[i] if i is not None else "" for i in idx])


def launch_list(src, out):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = {"nsecond": v / 1000.0, "ns": v / 1000.0, "usecond": v, "us": v, "msecond": v * 1000.0, "ms": v * 1000.0}.get(r[ui], v)
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(v)
    total = sum(sum(v) for v in agg.values())
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "avg_us", "total_us", "share_of_listed_time"])
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            w.writerow([k, len(v), f"{sum(v) / len(v):.2f}", f"{sum(v):.1f}", f"{sum(v) / total:.3f}"])


if __name__ == "__main__":
    {"full": full, "list": launch_list}[sys.argv[1]](sys.argv[2], sys.argv[3])
