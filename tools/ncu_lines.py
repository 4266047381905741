"""Per-CUDA-source-line view of an ncu report (needs -lineinfo + --import-source on):
warp instructions executed, stall samples and shared-memory wavefronts per line.

    python tools/ncu_lines.py gpurun_out/X.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    header = None
    for line in txt.splitlines():
        if line.startswith('"File Path"'):
            fname = next(csv.reader(io.StringIO(line)))[1].split("/")[-1]
            continue
        if line.startswith('"Line No"'):
            header = next(csv.reader(io.StringIO(line)))
            continue
        if header is None or line.startswith('"Function Name"'):
            continue
        r = next(csv.reader(io.StringIO(line)))
        if r and r[0] not in ("", "-"):
            d = dict(zip(header, r))
            rows.append((fname, r[0], r[1].strip()[:90], d))
    def num(d, k):
        try:
            return float(d.get(k, "0") or 0)
        except ValueError:
            return 0.0
    inst = sum(num(d, "Instructions Executed") for *_, d in rows)
    samp = sum(num(d, "Warp Stall Sampling (All Samples)") for *_, d in rows)
    wf_key = "L1 Wavefronts Shared"
    wf = sum(num(d, wf_key) for *_, d in rows)
    print(f"warp instructions {inst:.4g}, stall samples {samp:.0f}, shared wavefronts {wf:.4g}")
    rows.sort(key=lambda t: -num(t[3], "Warp Stall Sampling (All Samples)"))
    print(f"{'samples%':>8} {'inst%':>6} {'wf%':>6}  file:line  source")
    for f, ln, src, d in rows[:top]:
        print(f"{100 * num(d, 'Warp Stall Sampling (All Samples)') / max(samp, 1):8.1f} "
              f"{100 * num(d, 'Instructions Executed') / max(inst, 1):6.1f} {100 * num(d, wf_key) / max(wf, 1):6.1f}  "
              f"{f}:{ln}  {src}")


if __name__ == "__main__":
    main()
