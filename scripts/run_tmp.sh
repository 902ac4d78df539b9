timeout 900 python -m pytest tests/test_gpu_sliced.py tests/test_gpu_configs.py::test_sharded_engine_over_nccl_world1 tests/test_cpp_dropin.py -q 2>&1 | tail -30 > gpurun_out/t.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cp bench_rows.csv gpurun_out/bench_rows.csv 2>/dev/null
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
