timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 --csv=gpurun_out/r02e_bench_rows.csv > gpurun_out/r02e_bench_full.json 2> gpurun_out/r02e_bench_full.err; tail -1 gpurun_out/r02e_bench_full.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02e_bench_full.json'))
print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step_reference_frac'])
print({k: v['avg_ms'] for k,v in d['kernels'].items() if v['avg_ms']>0.05})
for L,x in d['phases']['c3_zipf'].items():
    if isinstance(x, dict): print(L, x['v2']['build_gkeys_s'], x['probe']['probe_ms'], x['probe']['gprobes_s'], x['probe']['match_count'], x['probe']['key_comparisons'])
PY
