set -x
nvidia-smi -L; nproc
timeout 900 python -m pytest tests -m gpu -q -x --durations=12 2>&1 | tail -40
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_part_build|k_multisplit|k_probe_part|k_part_hist" -s 16 -c 8 -o gpurun_out/prof1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
