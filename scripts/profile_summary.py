#!/usr/bin/env python
"""Write the committed profile summary from a launch-list CSV and an ncu --set full report.

usage: python scripts/profile_summary.py TAG [WORKLOAD]   (reads gpurun_out/launches_TAG.csv,
gpurun_out/prof_TAG.ncu-rep; WORKLOAD = the bench.py --workload the capture ran, default c3)
writes profiles/TAG_launches.csv, profiles/TAG_ncu_raw.csv, profiles/TAG_summary.md and the WORKLOAD entry of
profiles/ncu_summary.json (bench.py reads roofline.traffic from it)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if not name.startswith("sigattn::"):
            continue
        per.setdefault(name, []).append(float(r[vi].replace(",", "")))
    return per


TITLES = {"c3": "C3 bench step: B=32 N=8192 H=12 d=64 jagged, bf16",
          "c4": "C4 bench step: one 160M-encoder layer, B=16 N=8192 H=12 d=64, bf16",
          "c5": "C5 bench step: N=16384 H=16 d=128 key-split CP, bf16"}


def main(tag, workload="c3"):
    out = os.path.join(ROOT, "profiles")
    lpath = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    shutil.copy(lpath, os.path.join(out, f"{tag}_launches.csv"))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    open(os.path.join(out, f"{tag}_ncu_raw.csv"), "w").write(raw)
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    kern = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        d = {}
        for k in want:
            if k in h:
                v, u = r[h.index(k)].replace(",", ""), units[h.index(k)]
                try:
                    fv = float(v)
                    fv *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(u, 1.0)
                    d[k] = fv
                except ValueError:
                    d[k] = v
        kern[name] = d
    per = launch_shares(lpath)
    tot = sum(sum(v) for v in per.values())
    lines = [f"# Profile summary `{tag}` ({TITLES.get(workload, workload)})", "",
             "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised;",
             "compare shares, not absolutes):", "", "| kernel | launches | mean us | share of step |", "|---|---|---|---|"]
    for k, v in per.items():
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    lines += ["", "`ncu --set full` (one launch each):", "", "| metric | " + " | ".join(kern) + " |",
              "|---|" + "---|" * len(kern)]
    for k in want:
        lines.append(f"| {k} | " + " | ".join(
            (f"{kern[n].get(k):.4g}" if isinstance(kern[n].get(k), float) else str(kern[n].get(k))) for n in kern) + " |")
    open(os.path.join(out, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    bwd = next((v for n, v in kern.items() if "bwd_kernel" in n or "bwd128_kernel" in n), {})
    fwd = next((v for n, v in kern.items() if "fwd_kernel" in n or "fwd2_kernel" in n), {})
    entry = {"tag": tag,
            "bwd_kernel": {"dram_bytes_per_launch": bwd.get("dram__bytes_read.sum", 0) + bwd.get("dram__bytes_write.sum", 0),
                           "duration_ms": bwd.get("gpu__time_duration.sum")},
            "fwd_kernel": {"dram_bytes_per_launch": fwd.get("dram__bytes_read.sum", 0) + fwd.get("dram__bytes_write.sum", 0),
                           "duration_ms": fwd.get("gpu__time_duration.sum")}}
    jp = os.path.join(out, "ncu_summary.json")
    summ = json.load(open(jp)) if os.path.exists(jp) else {}
    if "tag" in summ:   # round-1 flat format: the C3 capture
        summ = {"c3": summ}
    summ[workload] = entry
    json.dump(summ, open(jp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "c3")
