"""Print the headline counters and the top stall reasons of every kernel in an ncu report."""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
stall = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:60])
    for w in want:
        if w in h:
            print(f"   {w:60s} {r[h.index(w)]} {rows[1][h.index(w)]}")
    st = sorted(((float(r[h.index(c)] or 0), c) for c in stall), reverse=True)
    print("   stalls/issue: " + ", ".join(f"{c[34:-29]} {v:.2f}" for v, c in st[:8]))
