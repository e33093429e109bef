"""Turn a tools/gpu_profile.sh run into the committed evidence under profiles/:
  <R>_bench.json          the bench line of that run
  <R>_launches.csv        the launch list itself (id, kernel, us per launch)
  <R>_launch_share.txt    share of device time per kernel over the timed solve (ncu launch list)
  <R>_ncu_full.txt        per-kernel key metrics of the --set full capture (means over launches)
  latest_ncu_summary.json DRAM bytes per launch of the roofline kernel (read by bench.py)
usage: python tools/profile_summary.py R [workload]"""
import collections
import csv
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def short(name):
    name = re.sub(r"\(Slab.*|\(const .*|\(double.*|\(int.*|\(long.*", "", name)
    name = re.sub(r"sb::|\(anonymous namespace\)::|<unnamed>::|unnamed>::|void ", "", name)
    return name.strip()[:70]


def launch_share(R):
    rows = list(csv.reader(open(os.path.join(OUT, f"launches_{R}.csv"))))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    compact = ["id,kernel,us"]
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", "nsecond"), 1e-3)
        a = agg[short(d["Kernel Name"])]
        a[0] += 1
        a[1] += v
        compact.append(f'{d["ID"]},"{short(d["Kernel Name"])}",{v:.2f}')
    open(os.path.join(PROF, f"{R}_launches.csv"), "w").write("\n".join(compact) + "\n")
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    lines = [f"ncu launch list of `python bench.py --steps 1 --warmup 3 --no-cpu-baseline`, NVTX range 'timed'",
             f"(one c4 solve; --clock-control none, per-launch cold-cache serialised times)",
             f"total {tot / 1e3:.1f} ms of kernel time over {n} launches", "",
             f"{'share':>7} {'launches':>8} {'avg us':>10}  kernel"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{t / tot * 100:6.2f}% {c:8d} {t / c:10.1f}  {k}")
    return "\n".join(lines) + "\n"


def full_summary(R):
    reps = sorted(glob.glob(os.path.join(OUT, f"full_{R}*.ncu-rep")))
    per = collections.defaultdict(list)
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            per[short(r[hdr.index("Kernel Name")])].append((hdr, units, r))
    names = ", ".join("gpurun_out/" + os.path.basename(r) for r in reps)
    out, js = [f"ncu --set full captures ({names}), means over the captured launches", ""], {}
    for name, rs3 in per.items():
        hdr, units = rs3[0][0], rs3[0][1]
        rs = [r for _, _, r in rs3]
        out.append(f"== {name}  ({len(rs)} launches)")
        m = {}
        for k in KEYS:
            if k not in hdr:
                continue
            i = hdr.index(k)
            vals = [float(r[i].replace(",", "")) for r in rs if r[i] not in ("", "n/a")]
            if not vals:
                continue
            v = sum(vals) / len(vals)
            u = units[i]
            if u in SCALE and k.startswith("dram__bytes"):
                v, u = v * SCALE[u], "byte"
            m[k] = v
            out.append(f"  {k}: {v:,.3f} {u}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                vals = [float(r[i]) for r in rs if r[i] not in ("", "n/a")]
                if vals:
                    st.append((h.split("stalled_")[1].split("_per")[0], sum(vals) / len(vals)))
        st.sort(key=lambda kv: -kv[1])
        out.append("  stalls (warps per issue): " + ", ".join(f"{a}={b:.2f}" for a, b in st[:6]))
        js[name] = m
    return "\n".join(out) + "\n", js


def main():
    R = sys.argv[1]
    workload = sys.argv[2] if len(sys.argv) > 2 else "c4"
    os.makedirs(PROF, exist_ok=True)
    bl = [l for l in open(os.path.join(OUT, f"bench_{R}.log")) if l.startswith("{")]
    if bl:
        open(os.path.join(PROF, f"{R}_bench.json"), "w").write(bl[-1])
    open(os.path.join(PROF, f"{R}_launch_share.txt"), "w").write(launch_share(R))
    txt, js = full_summary(R)
    open(os.path.join(PROF, f"{R}_ncu_full.txt"), "w").write(txt)
    ax = [v for k, v in js.items() if "k_axw" in k and "EWrite" in k and "double" in k]
    latest = {"round": R, "workload": workload, "kernels": js}
    if ax:
        latest["ax_dram_bytes_per_launch"] = ax[0]["dram__bytes_read.sum"] + ax[0]["dram__bytes_write.sum"]
    ras = [v for k, v in js.items() if "k_rasw<10, float, 0>" in k]
    if ras:
        latest["ras_dram_bytes_per_launch"] = ras[0]["dram__bytes_read.sum"] + ras[0]["dram__bytes_write.sum"]
    json.dump(latest, open(os.path.join(PROF, "latest_ncu_summary.json"), "w"), indent=1)
    print(open(os.path.join(PROF, f"{R}_launch_share.txt")).read()[:3000])
    print(txt[:6000])


if __name__ == "__main__":
    main()
