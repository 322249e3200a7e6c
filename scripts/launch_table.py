"""Summarise an ncu --csv launch list (metrics per launch) by kernel name."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
i = h.index
data = collections.defaultdict(dict)
for r in rows[1:]:
    data[(r[i("ID")], r[i("Kernel Name")])][r[i("Metric Name")]] = r[i("Metric Value")]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, None])
for (_, k), m in data.items():
    a = agg[k]
    a[0] += 1
    a[1] += float(m.get("gpu__time_duration.sum", 0))
    a[2] += float(m.get("dram__bytes_read.sum", 0)) + float(m.get("dram__bytes_write.sum", 0))
    a[3] = m.get("launch__registers_per_thread")
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    bw = a[2] / a[1] if a[1] else 0
    print(f"{k[:58]:58s} n={a[0]:4d} {a[1]/1e3:9.1f} us {100*a[1]/tot:5.1f}% {bw:7.0f} GB/s regs={a[3]}")
