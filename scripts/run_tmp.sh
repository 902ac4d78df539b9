bash scripts/gpu_prof.sh r02
