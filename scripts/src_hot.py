"""Hot SASS lines per kernel of an `ncu --page source --csv` dump: python scripts/src_hot.py FILE [min_pct] [name filter]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1.2
flt = sys.argv[3] if len(sys.argv) > 3 else ""
ker = None; blocks = {}
for r in rows:
    if r and r[0] == "Kernel Name":
        ker = r[1] + "#" + str(len(blocks)); blocks[ker] = []; continue
    if ker: blocks[ker].append(r)
seen = set()
for k, b in blocks.items():
    name = k.split("#")[0]
    if name in seen or flt not in name: continue
    seen.add(name)
    hdr = b[0]
    try:
        iS = hdr.index("# Samples"); iI = hdr.index("Instructions Executed"); iSrc = hdr.index("Source")
    except ValueError:
        continue
    data = [(int(r[iS] or 0), int(r[iI] or 0), r[iSrc]) for r in b[1:] if len(r) > iS]
    tot = sum(d[0] for d in data)
    print("=====", name[:70], "samples", tot, "warp-instr", sum(d[1] for d in data))
    acc = 0
    for i, d in enumerate(data):
        acc += d[0]
        if d[0] >= tot * thr / 100:
            print(i, f"{100*d[0]/tot:.1f}%", d[1], d[2][:80], f"cum {100*acc/tot:.0f}%")
