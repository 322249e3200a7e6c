"""Summarise an ncu report (and optionally a launch-list CSV) into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_X.ncu-rep profiles/r1_NAME [--launches gpurun_out/launches.csv]
        [--images-per-launch N]

Writes <out>.json (per-kernel key metrics, dram bytes per launch = the bench
`roofline.traffic`) and <out>.md (human summary with stall breakdown).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
]


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def main():
    rep, out = sys.argv[1], Path(sys.argv[2])
    launches = None
    if "--launches" in sys.argv:
        launches = sys.argv[sys.argv.index("--launches") + 1]
    hdr, units, rows = raw_rows(rep)
    kernels = []
    for row in rows:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        rec = {"kernel": name}
        for k in KEYS:
            if k in d:
                rec[k] = to_float(d[k])
                rec[k + ".unit"] = u.get(k)
        stalls = {}
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                v = to_float(d[h])
                if v:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        rec["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        rb, wb = rec.get("dram__bytes_read.sum"), rec.get("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if rb is not None and wb is not None:
            rec["dram_bytes_per_launch"] = rb * scale.get(rec["dram__bytes_read.sum.unit"], 1) + \
                wb * scale.get(rec["dram__bytes_write.sum.unit"], 1)
        kernels.append(rec)
    summary = {"report": rep, "kernels": kernels}
    if "--images-per-launch" in sys.argv:
        summary["images_per_launch"] = int(sys.argv[sys.argv.index("--images-per-launch") + 1])
    if launches:
        per = defaultdict(list)
        step_bytes = [0.0]
        with open(launches) as fh:
            lines = [l for l in fh if l.startswith('"')]
        rd = list(csv.reader(lines))
        h = rd[0]
        for r in rd[1:]:
            dd = dict(zip(h, r))
            if dd.get("Metric Name") == "gpu__time_duration.sum":
                per[dd["Kernel Name"].split("(")[0]].append(to_float(dd["Metric Value"]))
            elif dd.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                # one hot-path step (bench --profile-step); the SE-spectrum launches at plan
                # creation (tile kernels with SPEC = 1) are not part of it
                if not dd["Kernel Name"].rstrip().endswith("1>(TileArgs)"):
                    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(dd.get("Metric Unit"), 1)
                    step_bytes[0] += (to_float(dd["Metric Value"]) or 0.0) * sc
        summary["launch_list"] = {k: {"launches": len(v), "total": sum(x for x in v if x), "mean": sum(x for x in v if x) / max(len(v), 1)}
                                  for k, v in per.items()}
        if step_bytes[0] > 0 and "--step-images" in sys.argv:
            n_img = int(sys.argv[sys.argv.index("--step-images") + 1])
            summary["dram_bytes_per_step"] = step_bytes[0]
            summary["dram_bytes_per_image"] = step_bytes[0] / n_img
        tot = sum(s["total"] for s in summary["launch_list"].values())
        for s in summary["launch_list"].values():
            s["share"] = s["total"] / tot if tot else None
    out.parent.mkdir(parents=True, exist_ok=True)
    out.with_suffix(".json").write_text(json.dumps(summary, indent=1))
    md = [f"# ncu summary: {Path(rep).name}", ""]
    for k in kernels:
        md.append(f"## {k['kernel'][:110]}")
        for key in KEYS:
            if key in k and k[key] is not None:
                md.append(f"- {key}: {k[key]} {k.get(key + '.unit') or ''}")
        if "dram_bytes_per_launch" in k:
            md.append(f"- dram bytes per launch (read+write): {k['dram_bytes_per_launch']:.4g}")
        md.append("- stalls per issued instruction: " + ", ".join(f"{a}={b:.2f}" for a, b in list(k["stalls_per_issue"].items())[:8]))
        md.append("")
    if launches:
        md.append("## launch list (gpu__time_duration.sum, cold-cache serialised: compare shares)")
        for name, s in summary["launch_list"].items():
            md.append(f"- {name[:80]}: {s['launches']} launches, total {s['total']:.4g}, share {s['share']:.3f}")
    out.with_suffix(".md").write_text("\n".join(md) + "\n")
    print(out.with_suffix(".md").read_text())


if __name__ == "__main__":
    main()
