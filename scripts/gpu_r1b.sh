set -x
nvidia-smi -L; nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -q -x --durations=12 2>&1 | tail -30
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/benchref.json 2> gpurun_out/benchref.err; tail -3 gpurun_out/benchref.err; cat gpurun_out/benchref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_build|k_multisplit|k_probe|k_part_hist" -s 12 -c 10 -o gpurun_out/prof1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
