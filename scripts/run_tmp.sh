timeout 600 python scripts/prof_c3.py 28 > gpurun_out/c3prof.log 2>&1
head -2 gpurun_out/c3prof.log
timeout 900 python -m pytest tests/test_gpu_sliced.py tests/test_gpu_configs.py -q -x 2>&1 | tail -3
