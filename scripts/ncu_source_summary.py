#!/usr/bin/env python
"""Summarise an `ncu --page source --csv` SASS dump: total stall reasons and the hottest instructions.

usage: ncu -i rep --page source --csv --kernel-name regex:K > src.csv; python scripts/ncu_source_summary.py src.csv [N]
"""
import csv
import sys
from collections import Counter


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    idx = {n: i for i, n in enumerate(h)}
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    tot = Counter()
    insts = []
    for r in rows[hi + 1:]:
        if len(r) < len(h) or not r[idx["Instructions Executed"]].replace(",", "").isdigit():
            continue
        s = int((r[idx["Warp Stall Sampling (All Samples)"]] or "0").replace(",", ""))
        for c in stall_cols:
            tot[c] += int((r[idx[c]] or "0").replace(",", ""))
        insts.append((s, r[idx["Address"]], r[idx["Source"]].strip(), int(r[idx["Instructions Executed"]].replace(",", "")),
                      {c: int((r[idx[c]] or "0").replace(",", "")) for c in stall_cols}))
    all_s = sum(tot.values())
    print(f"total samples {all_s}")
    for c, v in tot.most_common():
        if v:
            print(f"  {c:28s} {v:8d} {100 * v / max(all_s, 1):5.1f}%")
    print(f"\ntop {top} instructions by samples:")
    for s, a, src, ex, st in sorted(insts, key=lambda x: -x[0])[:top]:
        main_st = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{s:7d} {a[-5:]} {src[:60]:60s} exec={ex:9d} {main_st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
