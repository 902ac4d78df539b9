BENCH_DEBUG=x timeout 900 python bench.py --config c5 --steps 4 --warmup 3 > gpurun_out/bench_c5_x.json 2> gpurun_out/bench_c5_x.err
grep "step host" gpurun_out/bench_c5_x.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --no-e2e --csv= > gpurun_out/b.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step'])"
