"""Summarise an ncu --set full report: per-kernel time, DRAM bytes, pipe usage, top stalls."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__inst_executed.sum', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.avg.per_second',
        'launch__grid_size', 'launch__block_size']


def main(path):
    out = subprocess.check_output(['ncu', '-i', path, '--page', 'raw', '--csv'], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')]
        print(f"== {name}")
        for w in WANT:
            if w in hdr:
                print(f"   {w:70s} {r[hdr.index(w)]}")
        vals = []
        for h, v in zip(hdr, r):
            if 'average_warps_issue_stalled' in h and 'not_issued' not in h:
                try:
                    vals.append((float(v), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
                except ValueError:
                    pass
        print("   stalls/issue:", ", ".join(f"{h}={v:.2f}" for v, h in sorted(vals, reverse=True)[:8]))


if __name__ == '__main__':
    main(sys.argv[1])
