# Round profile pass: launch list of the bench step + one ncu --set full
# capture per hot kernel, raw metric CSVs for profiles/ (reports are read here
# with scripts/ncu_summary.py and scripts/make_traffic.py).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_launch.log 2>&1
# bench step = build (k_part_hist, k_multisplit x2, k_part_build) + probe (k_part_hist, k_multisplit x2, k_probe_part)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_hist -s 6 -c 2 -o gpurun_out/full_hist $B > gpurun_out/ncu_hist.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_multisplit -s 12 -c 2 -o gpurun_out/full_msplit $B > gpurun_out/ncu_msplit.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_build -s 3 -c 1 -o gpurun_out/full_pbuild $B > gpurun_out/ncu_pbuild.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_part -s 3 -c 1 -o gpurun_out/full_pprobe $B > gpurun_out/ncu_pprobe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_intersect -s 2 -c 1 -o gpurun_out/full_isect python scripts/prof_intersect.py > gpurun_out/ncu_isect.log 2>&1
tail -1 gpurun_out/ncu_*.log
for f in gpurun_out/full_*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
du -sh gpurun_out
for f in $(ls -S gpurun_out/full_*.ncu-rep); do
  if [ $(du -sm gpurun_out | cut -f1) -gt 58 ]; then rm -f $f; fi
done
du -sh gpurun_out
