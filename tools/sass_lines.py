"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.
ncu's SASS page (addresses + samples) is matched by instruction offset against the line table
nvdisasm prints for the same locally built object (built with -lineinfo).
usage: python tools/sass_lines.py REPORT KERNEL_REGEX OBJ MANGLED_SUBSTR [top] [ncu source column]
(column e.g. "Instructions Executed" for the instruction mix instead of stall samples)"""
import collections
import csv
import re
import subprocess
import sys
import tempfile
import os


def main():
    rep, kre, obj, mang = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    col = sys.argv[6] if len(sys.argv) > 6 else "Warp Stall Sampling (All Samples)"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                          "--kernel-id", f"::regex:{kre}:1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    si, ai = h.index(col), h.index("Address")
    samples = []
    for r in rows[hi + 1:]:
        if len(r) > si and r[ai].startswith("0x"):
            samples.append((int(r[ai], 16), float(r[si] or 0), r[h.index("Source")].strip()))
    base = samples[0][0]
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-c", "-g", "--print-line-info", os.path.join(tmp, cub)],
                         capture_output=True, text=True).stdout.splitlines()
    line_of, cur, infn, cur_line = {}, None, False, None
    for l in dis:
        if l.startswith("//---") and ".text." in l:
            infn = mang in l
            continue
        if not infn:
            continue
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if "//## File" in l and m:
            f = m.group(1).split("/")[-1]
            cur_line = int(m.group(2)) if f == os.path.basename(obj).split(".")[0] + ".cu" else f"{f}:{m.group(2)}"
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m:
            line_of[int(m.group(1), 16)] = cur_line
    agg = collections.Counter()
    tot = 0.0
    for addr, v, _ in samples:
        agg[line_of.get(addr - base)] += v
        tot += v
    src = {}
    for f in ("paper_2110_07663_b200/csrc/k_fdm.cu", "paper_2110_07663_b200/csrc/k_space.cu",
              "paper_2110_07663_b200/csrc/k_mg.cu"):
        if f.split("/")[-1].split(".")[0] in obj:
            src = dict(enumerate(open(f).read().splitlines(), 1))
    print(f"{len(samples)} SASS instructions, {tot:.0f} samples, {len(line_of)} mapped offsets")
    for ln, v in agg.most_common(top):
        print(f"{v / tot * 100:5.1f}%  {ln!s:>5}  {src.get(ln, '')[:100].strip()}")


if __name__ == "__main__":
    main()
