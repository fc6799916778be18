"""Summary of an ncu --set full report (read here, no GPU): per kernel the
duration, DRAM bytes, occupancy, pipe utilisation and top stall reasons.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--alg-bytes K=BYTES ...]
"""
import argparse
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "lts__t_sector_hit_rate.pct"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print("==", v[h.index("Kernel Name")][:90])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"   {w:62s} {v[i]:>16s} {units[i]}")
        st = [(n, v[i]) for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
        st = sorted(((n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(x))
                     for n, x in st if x.replace(".", "", 1).isdigit()), key=lambda t: -t[1])
        print("   stalls/issue: " + ", ".join(f"{n}={x:.2f}" for n, x in st[:8]))


if __name__ == "__main__":
    sys.exit(main())
