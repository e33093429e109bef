"""Record the DRAM traffic of the two roofline kernels from tools/ncu_roofline.sh captures into
profiles/latest_ncu_summary.json (read by bench.py) and profiles/<R>_roofline_ncu.txt.
usage: python tools/roof_summary.py R  (reads gpurun_out/roof_R*.ncu-rep)"""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
out, found = [], {}
for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"roof_{R}*.ncu-rep"))):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        vals = {}
        for k in KEYS:
            if k in h:
                v = float(r[h.index(k)].replace(",", "") or 0)
                vals[k] = v * SCALE.get(units[h.index(k)], 1.0)
        found.setdefault(name, vals)
for name, vals in found.items():
    out.append(f"== {name}\n" + "".join(f"  {k}: {v:,.3f}\n" for k, v in vals.items()))
    tr = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    out.append(f"  DRAM traffic per launch: {tr / 1e6:.1f} MB\n")
open(os.path.join(ROOT, "profiles", f"{R}_roofline_ncu.txt"), "w").write(
    f"ncu --set full of the roofline kernels as bench.py times them (tools/ncu_roofline.sh, E=32^3 p=7)\n\n"
    + "".join(out))
p = os.path.join(ROOT, "profiles", "latest_ncu_summary.json")
js = json.load(open(p))
for name, vals in found.items():
    tr = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    if "k_axw" in name and "EWrite" in name and "double" in name:
        js["ax_dram_bytes_per_launch"] = tr
        js["ax_traffic_source"] = f"{R}_roofline_ncu.txt"
    if "k_rasw<10, float, 0>" in name:
        js["ras_dram_bytes_per_launch"] = tr
        js["ras_traffic_source"] = f"{R}_roofline_ncu.txt"
json.dump(js, open(p, "w"), indent=1)
print("".join(out))
