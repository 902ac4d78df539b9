"""Per-kernel timeline of build_v2 at key multiplicity 1 vs 32 (keys from the
reference generator, acceptance criterion 4; library event profiler)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import _lib
from oracle.oracle import Reference

n = 1 << 28
ref = Reference()
keys = torch.empty(n, dtype=torch.int32, device="cuda")
for mult, seed in ((1.0, 101), (32.0, 102)):
    h = ref.generate(1, n, mult, seed).astype(np.uint32)
    keys.copy_(torch.from_numpy(h.view(np.int32)))
    cfg = hg.BuildConfig(hash_seed=9)
    hg.build_v2(keys, cfg).close()
    torch.cuda.synchronize()
    _lib.profiler_enable(True)
    _lib.profiler_collect()
    hg.build_v2(keys, cfg).close()
    torch.cuda.synchronize()
    k = _lib.profiler_collect()
    _lib.profiler_enable(False)
    print(f"mult {mult}:", {a: round(x[1], 3) for a, x in sorted(k.items(), key=lambda z: -z[1][1])})
