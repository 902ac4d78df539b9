set -x
nvidia-smi -L; nproc
timeout 900 python bench.py --steps 10 --warmup 3 --csv=gpurun_out/r02d_bench_rows.csv > gpurun_out/r02d_bench_full.json 2> gpurun_out/r02d_bench_full.err; tail -2 gpurun_out/r02d_bench_full.err
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-extras --csv= > gpurun_out/r02d_bench_c5.json 2> gpurun_out/r02d_bench_c5.err; tail -2 gpurun_out/r02d_bench_c5.err
bash scripts/gpu_prof.sh r02d
