timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --no-e2e --csv= 2>gpurun_out/ab.err | tail -1 > gpurun_out/ab.json
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['ms_per_step'], d['value'], d['gpu_launches'], d['roofline'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_probe_pairs" -c 1 -o gpurun_out/c4b_full python scripts/prof_c3.py 28 c4 > gpurun_out/ncu_c4.log 2>&1
python scripts/ncu_lines.py gpurun_out/c4b_full.ncu-rep . 40 > gpurun_out/c4b_lines.txt 2>&1
python scripts/ncu_summary.py gpurun_out/c4b_full.ncu-rep . 10 > gpurun_out/c4b_summary.txt 2>&1
rm -f gpurun_out/c4b_full.ncu-rep
