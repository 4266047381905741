"""Compact summary of an ncu --set full report (for profiles/).

    python tools/ncu_summary.py gpurun_out/X.ncu-rep [points_per_launch] > profiles/rN_X.md
Also prints the per-launch DRAM traffic used as bench.py's roofline.traffic.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput % (incl. shared)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared wavefronts % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid size"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main():
    rep = sys.argv[1]
    npts = float(sys.argv[2]) if len(sys.argv) > 2 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        print(f"kernel: `{d.get('Kernel Name', ('?', ''))[0][:120]}`\n")
        print("| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in d:
                v, u = d[key]
                print(f"| {label} (`{key}`) | {v} {u} |")
        try:
            rd = float(d["dram__bytes_read.sum"][0]) * _scale(d["dram__bytes_read.sum"][1])
            wr = float(d["dram__bytes_write.sum"][0]) * _scale(d["dram__bytes_write.sum"][1])
            print(f"| DRAM traffic per launch | {rd + wr:.4e} B |")
            if npts:
                print(f"| DRAM bytes per point | {(rd + wr) / npts:.3f} |")
                inst = float(d["sm__inst_executed.sum"][0].replace(",", ""))
                print(f"| thread instructions per point | {inst * 32 / npts:.1f} |")
        except (KeyError, ValueError):
            pass
        print()


def _scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


if __name__ == "__main__":
    main()
