timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --csv= 2>/dev/null | tail -1 > gpurun_out/ab.json
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['ms_per_step'], d['value'], d['gpu_launches'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step_reference_frac'])"
