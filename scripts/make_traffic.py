"""Writes profiles/traffic.json (DRAM bytes per launch from an ncu --set full
capture, as bench.py's roofline.traffic) and the round's ncu summary.

    python scripts/make_traffic.py r02    # gpurun_out/r02_full_raw.csv (gpu_prof.sh):
                                          # the 8 kernels of one C2 step, launch order
    python scripts/make_traffic.py r01    # round-1 layout: gpurun_out/full_*_raw.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
# capture file -> bench profiler names of its rows, in launch order (gpu_prof.sh)
ROWS = {"hist": ["k4_part_hist", "p4_part_hist"], "msplit": ["k6a_multisplit", "k6b_multisplit"],
        "pbuild": ["k7_part_build"], "pprobe": ["k8p_probe_part"], "isect": ["k12_intersect"]}
KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
if os.path.exists(os.path.join(OUT, f"{tag}_full_raw.csv")):
    # one capture of a whole C2 step: build (K4, K6a, K6b, K7), probe (P4, P6a, P6b, K8p)
    ROWS = {f"{tag}_full": ["k4_part_hist", "k6a_multisplit", "k6b_multisplit", "k7_part_build",
                            "p4_part_hist", "p6a_multisplit", "p6b_multisplit", "k8p_probe_part"]}
traffic, summary = {}, []
for cap, names in ROWS.items():
    path = os.path.join(OUT, f"{cap}_raw.csv" if cap.endswith("_full") else f"full_{cap}_raw.csv")
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    data = rows[2:]
    if cap.endswith("_full"):
        # classify by kernel name in launch order; guarded no-op launches (the
        # slack layout's exact fallback, < 20 us) are skipped
        names, keep, phase, nsplit = [], [], "k", 0
        ti = hdr.index("gpu__time_duration.sum")
        for r in data:
            kn = r[hdr.index("Kernel Name")]
            if float(r[ti]) * UNIT.get(units[ti], 1.0) < 0.02:
                continue
            if kn.startswith("void k_part_hist"):
                nm = f"{phase}4_part_hist"
            elif kn.startswith("void k_multisplit"):
                nm = f"{phase}6{'ab'[nsplit % 2]}_multisplit"
                nsplit += 1
            elif kn.startswith("void k_part_build"):
                nm, phase, nsplit = "k7_part_build", "p", 0
            elif kn.startswith("void k_probe_part"):
                nm = "k8p_probe_part"
            else:
                continue
            names.append(nm)
            keep.append(r)
        data = keep
    for name, r in zip(names, data):
        def val(m):
            i = hdr.index(m)
            return float(r[i]) * UNIT.get(units[i], 1.0)
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        traffic[name] = int(rd + wr)
        ent = {"bench_name": name, "Kernel Name": r[hdr.index("Kernel Name")],
               "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
               "duration_ms": val("gpu__time_duration.sum")}
        for m in KEEP[3:]:
            if m in hdr:
                ent[m] = r[hdr.index(m)]
        summary.append(ent)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump({"source": f"ncu --set full --clock-control none, one launch per kernel ({tag}); "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch",
           "kernels": traffic},
          open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
json.dump(summary, open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
