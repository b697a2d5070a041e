"""Print an ncu --metrics launch list (csv with warnings on top) as one line per launch."""
import csv
import io
import sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
ki, mi, vi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
d = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    d.setdefault((int(r[ii]), r[ki].split("(")[0][:70]), {})[r[mi]] = (r[vi], r[ui])
for (i, k), v in sorted(d.items()):
    print(i, k, " ".join(f"{m.split('__')[1]}={val}{u}" for m, (val, u) in sorted(v.items())))
