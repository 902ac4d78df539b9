timeout 600 python scripts/prof_c3.py 28 c4 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --csv= > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step']);print({k:v['avg_ms'] for k,v in d['kernels'].items()});print(d['phases']['probe_new'])"
