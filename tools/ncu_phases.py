"""Sum an ncu report's per-source-line instruction counts by file and line range
(phase attribution for the profiles/ notes).

    python tools/ncu_phases.py gpurun_out/X.ncu-rep [min_pct]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    lim = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, header = [], "?", None
    for line in txt.splitlines():
        if line.startswith('"File Path"'):
            fname = next(csv.reader(io.StringIO(line)))[1].split("/")[-1]
            continue
        if line.startswith('"Line No"'):
            header = next(csv.reader(io.StringIO(line)))
            continue
        if header is None:
            continue
        r = next(csv.reader(io.StringIO(line)))
        if r and r[0] not in ("", "-") and r[0].isdigit():
            d = dict(zip(header, r))
            try:
                inst = float(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                inst = 0.0
            rows.append((fname, int(r[0]), r[1].strip()[:100], inst))
    tot = sum(r[3] for r in rows) or 1.0
    for f, ln, src, inst in sorted(rows, key=lambda t: (t[0], t[1])):
        if 100 * inst / tot >= lim:
            print(f"{100 * inst / tot:6.2f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
