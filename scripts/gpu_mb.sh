timeout 300 ./scripts/microbench > gpurun_out/microbench.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
