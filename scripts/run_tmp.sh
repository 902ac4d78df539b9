timeout 300 python scripts/prof_c3.py 28 > gpurun_out/c3prof.txt 2>&1; cat gpurun_out/c3prof.txt | tail -4
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -5 gpurun_out/gputest.log
