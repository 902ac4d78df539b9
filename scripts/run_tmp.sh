timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --no-e2e --csv= > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step'],d['match_count'],d['key_comparisons']);print({k:v['avg_ms'] for k,v in d['kernels'].items()})" || tail gpurun_out/b.err
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_probe_part -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-extras --no-e2e --csv= 2>/dev/null | grep -E "duration|inst_executed"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
