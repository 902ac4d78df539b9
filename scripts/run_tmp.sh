timeout 300 python scripts/prof_c3.py 28 > gpurun_out/c3prof.txt 2>&1; head -1 gpurun_out/c3prof.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
