"""Summarise an ncu report's SASS source page: hottest instructions by stall samples.

    python tools/ncu_hot.py gpurun_out/X.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    lines = txt.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    stall_cols = [c for c in rows[0] if c.startswith("stall_")]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    inst = sum(int(r["Instructions Executed"] or 0) for r in rows)
    print(f"total samples {tot}, warp instructions {inst}")
    agg = Counter()
    for r in rows:
        for c in stall_cols:
            agg[c] += int(r[c] or 0)
    print("stall reasons:", ", ".join(f"{k[6:]}={v/tot:.1%}" for k, v in agg.most_common(8)))
    ops = Counter()
    for r in rows:
        op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
        if op.startswith("@"):
            op = r["Source"].strip().split()[1]
        ops[op.split(".")[0]] += int(r["Instructions Executed"] or 0)
    print("opcode mix:", ", ".join(f"{k}={v/inst:.1%}" for k, v in ops.most_common(14)))
    rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        top_st = max(stall_cols, key=lambda c: int(r[c] or 0))
        print(f"{s/tot:6.1%} {int(r['Instructions Executed'] or 0):>10} {r['Address'][-5:]} {top_st[6:]:>18}  {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()
