"""C5 at one GPU (2^32 keys + 2^32 probes): per-phase device time of the
sliced build and the sliced probe, and the kernel totals (library profiler)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import _lib

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 32
keys = torch.empty(n, dtype=torch.int32, device="cuda")
probes = torch.empty(n, dtype=torch.int32, device="cuda")
hg.generate(keys, kind=0, seed=1)
hg.generate(probes, kind=0, seed=2)
res = torch.zeros(2, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
mode = sys.argv[2] if len(sys.argv) > 2 else ""
if "clock" in mode:
    from bench import ClockSampler
    cs = ClockSampler(0)
    cs.__enter__()
for it in range(6):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    _lib.profiler_enable(it == 5 or "prof" in mode)
    t0 = time.perf_counter()
    e[0].record()
    t = hg.build_v2(keys, stream=s.cuda_stream)
    e[1].record()
    t1 = time.perf_counter()
    hg.probe_device(t, probes, res, stream=s.cuda_stream)
    e[2].record()
    t2 = time.perf_counter()
    t.close(s.cuda_stream)
    e[3].record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"it {it}: build {e[0].elapsed_time(e[1]):.1f} ms  probe {e[1].elapsed_time(e[2]):.1f} ms  "
          f"close {e[2].elapsed_time(e[3]):.1f} ms | host build {1e3*(t1-t0):.1f} probe {1e3*(t2-t1):.1f} "
          f"sync {1e3*(t3-t2):.1f}", flush=True)
k = _lib.profiler_collect()
tot = sum(v[1] for v in k.values())
print(f"kernels total {tot:.1f} ms:", {a: (b[0], round(b[1], 2)) for a, b in sorted(k.items(), key=lambda x: -x[1][1])})
print("matches", res.tolist())
