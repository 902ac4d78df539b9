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
pairs = torch.empty((1 << 25, 2), dtype=torch.int32, device="cuda")
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
for _ in range(3):
    e0.record()
    hg.probe_new_device(ta, tb, res)
    e1.record()
    hg.probe_new_device(ta, tb, res, pairs=pairs, pair_width=4, pair_cap=1 << 25)
    e2.record()
    torch.cuda.synchronize()
    print(f"intersect count {e0.elapsed_time(e1):.3f} ms, pairs {e1.elapsed_time(e2):.3f} ms")
print("matches", res.tolist())
