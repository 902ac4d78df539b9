"""Per-CUDA-source-line aggregation of an ncu report's source page: stall
samples, warp instructions, shared-memory wavefronts (and the ideal count, so
bank conflicts show as the excess) and global sectors.
Usage: python scripts/ncu_lines.py REP kernel-regex [top]"""
import csv
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fn = path = None
hdr = None
agg = {}
COLS = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Ideal", "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Ideal"]
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        fn = r[1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and r[2] == "-" and re.search(kre, fn or ""):
        key = (fn, path, int(r[0]), r[1].strip()[:60])
        a = agg.setdefault(key, [0] * len(COLS))
        for k, c in enumerate(COLS):
            if c in hdr:
                v = r[hdr.index(c)]
                a[k] += int(float(v)) if v.replace(".", "", 1).isdigit() else 0
for f in sorted(set(k[0] for k in agg)):
    items = sorted(((v, k) for k, v in agg.items() if k[0] == f), key=lambda x: -x[0][0])[:top]
    tot = [sum(v[i] for k, v in agg.items() if k[0] == f) for i in range(len(COLS))]
    print(f"== {f[:100]}\n   totals: " + ", ".join(f"{c.split('(')[0].strip()}={t}" for c, t in zip(COLS, tot)))
    print(f"   {'stall':>7} {'inst':>10} {'smemWF':>10} {'ideal':>10} {'l2sec':>10} {'ideal':>10}  line")
    for v, k in items:
        print(f"   {v[0]:>7} {v[1]:>10} {v[2]:>10} {v[3]:>10} {v[4]:>10} {v[5]:>10}  {k[1]}:{k[2]} {k[3]}")
