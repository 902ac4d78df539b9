timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --no-e2e --csv= > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step'],d['match_count'],d['key_comparisons']);print({k:v['avg_ms'] for k,v in d['kernels'].items()})" || tail -5 gpurun_out/b.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sliced.py -q -x 2>&1 | tail -2
