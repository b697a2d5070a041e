"""Summarise ncu output into profiles/.

    python tools/ncu_summary.py full  <out.csv> <report.ncu-rep>...   one row per captured launch
    python tools/ncu_summary.py list  <launches.csv> <out.csv>        per-kernel aggregate of a launch list
    python tools/ncu_summary.py train-traffic <report.ncu-rep> <out.json>
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def full(out, *reps):
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["report"] + KEYS[:3] + ["duration_us", "dram_read_MB", "dram_write_MB"] + [k for k in KEYS[6:]])
        for rep in reps:
            h, units, data = raw(rep)
            idx = {k: h.index(k) for k in KEYS if k in h}
            for r in data:
                def val(k):
                    if k not in idx:
                        return ""
                    v = r[idx[k]].replace(",", "")
                    try:
                        return float(v) * SCALE.get(units[idx[k]], 1.0)
                    except ValueError:
                        return v
                dur = val("gpu__time_duration.sum")
                rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
                w.writerow([os.path.basename(rep), r[idx["Kernel Name"]].split("(")[0][:90], r[idx["Grid Size"]],
                            r[idx["Block Size"]], f"{dur:.2f}", f"{rd / 1e6:.3f}", f"{wr / 1e6:.3f}"] +
                           [r[idx[k]] if k in idx else "" for k in KEYS[6:]])


def launch_list(src, out):
    txt = open(src).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        per.setdefault((int(r[ii]), r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    agg = collections.OrderedDict()
    for (_, name), m in per.items():
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "avg_us", "total_us", "share_of_listed_time", "avg_dram_MB_per_launch"])
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k, a[0], f"{a[1] / a[0]:.2f}", f"{a[1]:.1f}", f"{a[1] / total:.3f}",
                        f"{(a[2] + a[3]) / a[0] / 1e6:.3f}"])


def train_traffic(rep, out):
    """DRAM bytes per launch of the training step's GEMM kernels (chain fwd, chain dZ, split-K / grouped wgrad)
    from one --set full capture -> profiles/ncu_traffic.json (bench.py roofline.traffic)."""
    h, units, data = raw(rep)
    k = h.index("Kernel Name")
    rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    per = {}
    for r in data:
        name = r[k].split("(")[0]
        if not any(s in name for s in ("mlp_chain", "wgrad_group", "wgrad_sk")):
            continue
        b = float(r[rd].replace(",", "")) * SCALE[units[rd]] + float(r[wr].replace(",", "")) * SCALE[units[wr]]
        per.setdefault(name, []).append(b)
    kern = {n: sum(v) / len(v) for n, v in per.items()}
    json.dump({"gemm_bytes_per_launch": sum(kern.values()) / max(len(kern), 1), "per_kernel_bytes": kern,
               "gemm_bytes_per_step": sum(kern.values()), "source": os.path.basename(rep),
               "note": "ncu --set full replays with cold caches: an upper bound on the step's DRAM traffic"},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "full":
        full(sys.argv[2], *sys.argv[3:])
    elif cmd == "list":
        launch_list(sys.argv[2], sys.argv[3])
    else:
        train_traffic(sys.argv[2], sys.argv[3])
