# Round profile pass: launch list of the bench step + one ncu --set full
# capture per hot kernel (small reps), raw metric CSVs for profiles/.
set -x
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_launch.log 2>&1
for k in k_part_hist k_multisplit k_part_build k_probe_part; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 2 -o gpurun_out/full_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_$k.log 2>&1
  tail -2 gpurun_out/ncu_$k.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_intersect -s 2 -c 2 -o gpurun_out/full_k_intersect python scripts/prof_intersect.py > gpurun_out/ncu_k_intersect.log 2>&1
tail -2 gpurun_out/ncu_k_intersect.log
for f in gpurun_out/full_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null
done
ls -la gpurun_out
du -sh gpurun_out
# keep the reports only while the total stays under the 64 MiB copy-back limit
for f in $(ls -S gpurun_out/full_*.ncu-rep); do
  if [ $(du -sm gpurun_out | cut -f1) -gt 55 ]; then rm -f $f; fi
done
du -sh gpurun_out
