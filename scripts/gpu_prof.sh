# Round profile pass: launch list of the bench step (one ncu --metrics pass)
# + one ncu --set full capture of every kernel of one C2 step (build: k4,
# k6a, k6b, k7; probe: p4, p6a, p6b, k8p), raw CSVs for profiles/
# (summarised here with scripts/ncu_summary.py / ncu_lines.py / make_traffic.py).
# usage: bash scripts/gpu_prof.sh TAG
set -x
TAG=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras --csv="
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras --csv= > gpurun_out/ncu_launch.log 2>&1
# warm-up = 3 steps: skip their launches, capture the 4th step's
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_hist|k_multisplit|k_part_build|k_probe_part" -s 24 -c 12 -o gpurun_out/${TAG}_full $B > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/${TAG}_full.ncu-rep . 30 > gpurun_out/${TAG}_lines.txt 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep . 10 > gpurun_out/${TAG}_summary.txt 2>&1
du -sh gpurun_out
# the report itself (12 kernels with source) exceeds gpurun's 64 MiB merge cap: compress it
xz -T0 -6 gpurun_out/${TAG}_full.ncu-rep 2>/dev/null
du -sh gpurun_out
