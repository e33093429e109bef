"""DRAM traffic per launch of the bench's roofline kernels from ncu --set full captures ->
profiles/latest_ncu_summary.json (read by bench.py for the `traffic` fields).
usage: python tools/traffic_summary.py AXE64.ncu-rep AXE32.ncu-rep FACE.ncu-rep RAS.ncu-rep
The Ax entries add the element kernel (k_axe) and its face-gather launch (k_face_epi7)."""
import csv
import json
import os
import subprocess
import sys


def dram(rep, regex=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if regex and regex not in name:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[h.index("dram__bytes_read.sum")]) * scale[rows[1][h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * scale[rows[1][h.index("dram__bytes_write.sum")]]
        out.append((name, rd + wr))
    return out


def main():
    ax64, ax32, face, ras = sys.argv[1:5]
    f = dram(face)
    face_b = {"EWrite": next((b for n, b in f if "EWrite" in n), None)}
    a64 = dram(ax64)[0][1]
    a32 = dram(ax32)[0][1]
    r0 = dram(ras)[0][1]
    summ = {"workload": "c4", "dram_bytes_per_launch": {"ax64": a64 + (face_b["EWrite"] or 0),
                                                        "ax32": a32 + (face_b["EWrite"] or 0), "ras0": r0},
            "parts": {"k_axe<double>": a64, "k_axe<float>": a32, "k_face_epi7": face_b["EWrite"], "k_rasw": r0},
            "sources": [os.path.basename(x) for x in sys.argv[1:5]],
            "note": "ncu --set full (caches flushed between kernels: cold-cache traffic), one launch each"}
    path = sys.argv[5] if len(sys.argv) > 5 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "latest_ncu_summary.json")
    json.dump(summ, open(path, "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
