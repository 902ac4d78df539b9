for v in 0 1 2 3 4; do
  HG_K8P=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-extras --no-e2e --csv= > gpurun_out/b$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b$v.json'));k=d['kernels'];print('var',$v,d['ms_per_step'],k['k8p_probe_part']['avg_ms'],d['match_count'],d['key_comparisons'])"
  HG_K8P=$v timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_probe_part -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-extras --no-e2e --csv= 2>/dev/null | grep -E "duration|inst_executed|wavefronts|throughput"
done
