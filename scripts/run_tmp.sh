timeout 300 python scripts/prof_c3.py 28 c4 > gpurun_out/c4prof.txt 2>&1; cat gpurun_out/c4prof.txt | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
