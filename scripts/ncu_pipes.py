#!/usr/bin/env python
"""Print per-kernel pipe utilisation, issue, DRAM/L2 and duration from an ncu report (raw page).

usage: python scripts/ncu_pipes.py gpurun_out/prof_X.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "cycles"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu(MUFU)%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible/cyc"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem(tc)%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem(lsu)%"),
    ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("launch__registers_per_thread", "regs"),
]


def main(rep, out_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "")
        d = {}
        for k, lab in KEYS:
            if k in h:
                v = r[h.index(k)].replace(",", "")
                u = units[h.index(k)]
                try:
                    fv = float(v)
                    if u == "Kbyte":
                        fv *= 1e3
                    elif u == "Mbyte":
                        fv *= 1e6
                    elif u == "Gbyte":
                        fv *= 1e9
                    elif u == "usecond":
                        fv *= 1e3
                    elif u == "msecond":
                        fv *= 1e6
                    d[lab] = fv
                except ValueError:
                    d[lab] = v
        res.setdefault(short, []).append(d)
    for k, lst in res.items():
        print(k)
        for d in lst:
            print("   " + "  ".join(f"{a}={b:.4g}" if isinstance(b, float) else f"{a}={b}" for a, b in d.items()))
    if out_json:
        json.dump(res, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--json" else None)
