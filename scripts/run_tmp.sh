lscpu | grep -E "Model name|^CPU\(s\)|Flags" | cut -c1-200 > gpurun_out/lscpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cp bench_rows.csv gpurun_out/bench_rows.csv 2>/dev/null
tail -3 gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/bench_ref.err
