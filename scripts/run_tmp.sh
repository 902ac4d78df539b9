timeout 600 python scripts/prof_c3.py 28 c4 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_probe_new.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
