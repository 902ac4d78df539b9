"""Profiling driver for the probe_new kernels (K12): builds two 2^28 u32
tables over one vertex range and runs probe_new_prepared count-only and with
pairs. Used under ncu by scripts/gpu_prof.sh (numbers printed here are not
bench values)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1907_02900_b200 as hg

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << log2n
keys = torch.empty(n, dtype=torch.int32, device="cuda")
probes = torch.empty(n, dtype=torch.int32, device="cuda")
hg.generate(keys, kind=0, seed=1)
hg.generate(probes, kind=0, seed=2)
res = torch.zeros(2, dtype=torch.int64, device="cuda")
ta = hg.build_v2(keys)
tb = hg.build_v2(probes, vertex_count=ta.num_vertices())
for _ in range(3):
    hg.probe_new_device(ta, tb, res)
pairs = torch.empty((1 << 25, 2), dtype=torch.int32, device="cuda")
for _ in range(2):
    hg.probe_new_device(ta, tb, res, pairs=pairs, pair_width=4, pair_cap=1 << 25)
torch.cuda.synchronize()
print("matches", res.tolist())
