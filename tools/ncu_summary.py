"""Summarise an .ncu-rep (raw page) into the few numbers we track per kernel."""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name", "?")[:80])
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]} {u.get(k, '')}")
        st = [(float(d[k].replace(",", "")), k) for k in hdr
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        print("  stall cycles per issued instruction:")
        for v, k in sorted(st, reverse=True)[:8]:
            print(f"    {v:6.3f}  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
