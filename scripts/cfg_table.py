"""Print bench_configs.py logs side by side: python scripts/cfg_table.py A.log [B.log]"""
import json
import sys


def load(path):
    res = {}
    for line in open(path):
        if line.startswith("c") and "{" in line:
            n, m, j = line.split(" ", 2)
            res[f"{n}_{m}"] = json.loads(j)
    return res


runs = [load(p) for p in sys.argv[1:]]
for k in runs[0]:
    cols = []
    for r in runs:
        d = r.get(k)
        if d:
            cols.append(f"{d['mpix_s']:8.0f} Mpx/s ({d['ms']:.4f} ms r{d.get('range_ms', 0):.3f} c{d.get('conv_ms', 0):.3f} t{d.get('tonal_ms', 0):.3f})")
    print(f"{k:10s} " + " | ".join(cols))
