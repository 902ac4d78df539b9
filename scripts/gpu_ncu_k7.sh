timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_part_build|k_probe_part" -s 2 -c 2 -o gpurun_out/prof3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu3.log
