"""Summarise an ncu report here (CPU side): key raw metrics per kernel and
the top stall SASS lines. Usage: python scripts/ncu_summary.py REP [kernel-regex] [nlines]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 12
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if not re.search(kre, name):
        continue
    print(name[:90])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:60s} {r[i]:>16s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
blocks, cur = [], None
for r in csv.reader(src.splitlines()):
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]
        blocks.append(cur)
    elif r and r[0] != "Address" and cur is not None:
        cur[1].append(r)
seen = set()
for name, lines in blocks:
    if not re.search(kre, name) or name in seen:
        continue
    seen.add(name)
    tot = sum(int(x[2]) for x in lines if x[2].isdigit())
    print(f"{name[:80]}: {len(lines)} SASS, {tot} stall samples")
    for x in sorted(lines, key=lambda x: -int(x[2]) if x[2].isdigit() else 0)[:ntop]:
        print(f"   {x[2]:>7s} {x[0][-5:]} {x[1][:80]}")

# per CUDA source line (needs -lineinfo): aggregate stall samples
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fn, path, agg = None, None, {}
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        fn = r[1]
    elif r[0] == "Line No" or not re.search(kre, fn or ""):
        continue
    elif r[0] and r[0].isdigit() and r[2] == "-":
        key = (fn, path, int(r[0]), r[1].strip()[:70])
        agg[key] = agg.get(key, 0) + (int(r[4]) if r[4].isdigit() else 0)
for f in sorted(set(k[0] for k in agg)):
    items = sorted(((v, k) for k, v in agg.items() if k[0] == f), reverse=True)[:ntop]
    print(f"[source lines] {f[:80]}")
    for v, k in items:
        print(f"   {v:>7d} {k[1]}:{k[2]} {k[3]}")

# utilisation of every unit ncu reports as pct_of_peak (top 15), first matching kernel
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if not re.search(kre, name):
        continue
    util = []
    for i, h in enumerate(hdr):
        if h.endswith("pct_of_peak_sustained_elapsed") or h.endswith("pct_of_peak_sustained_active"):
            try:
                util.append((float(r[i]), h))
            except ValueError:
                pass
    print(f"[unit utilisation] {name[:80]}")
    for v, h in sorted(util, reverse=True)[:15]:
        print(f"   {v:7.2f} {h}")
