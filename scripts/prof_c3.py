"""Per-kernel timeline of the C3 (Zipf, u64 key/value) builds and the C4
join probe (library event profiler; not a bench value)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import _lib

log2n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 28
only_c4 = "c4" in sys.argv[1:]
n = 1 << log2n
cdf = torch.tensor(hg.zipf_cdf(1 << 24, 1.0), dtype=torch.float64, device="cuda")
keys = torch.empty(n, dtype=torch.int64, device="cuda")
hg.generate(keys, kind=3, seed=1, ref=cdf)
vals = torch.arange(n, dtype=torch.int64, device="cuda")
for variant, b in (() if only_c4 else ((2, hg.build_v2), (1, hg.build_v1))):
    b(keys, vals=vals).close()
    torch.cuda.synchronize()
    _lib.profiler_enable(True)
    _lib.profiler_collect()
    t = b(keys, vals=vals)
    torch.cuda.synchronize()
    k = _lib.profiler_collect()
    _lib.profiler_enable(False)
    print(f"C3 v{variant}:", {a: round(x[1], 3) for a, x in sorted(k.items(), key=lambda z: -z[1][1])})
    t.close()
del keys, vals
c4n = 26 if "small" in sys.argv[1:] else 28
build = torch.empty(1 << c4n, dtype=torch.int32, device="cuda")
hg.generate(build, kind=2)
t = hg.build_v2(build)
m = 1 << (c4n + 1)
probes = torch.empty(m, dtype=torch.int32, device="cuda")
hg.generate(probes, kind=1, seed=3, hit=0.5, ref=build)
res = torch.zeros(2, dtype=torch.int64, device="cuda")
pairs = torch.empty((m, 2), dtype=torch.int32, device="cuda")
for it in range(2):
    _lib.profiler_enable(True)
    _lib.profiler_collect()
    hg.probe_device(t, probes, res, pairs=pairs, pair_width=4, pair_cap=m)
    torch.cuda.synchronize()
    k = _lib.profiler_collect()
    _lib.profiler_enable(False)
print("C4 h=0.5:", {a: round(x[1], 3) for a, x in sorted(k.items(), key=lambda z: -z[1][1])})
