# A/B timing of alternate builds of the C-ABI (exp/*.so via HG_B200_LIB)
# against the in-tree build: C2 step kernels, 5 steps after 3 warm-ups.
# usage: bash scripts/ab.sh exp/libhg_var1.so [...]
for lib in "" "$@"; do
  HG_B200_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-extras --no-e2e --csv= > gpurun_out/ab.json 2>/dev/null
  python - "$lib" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
k = {n: v["avg_ms"] for n, v in d["kernels"].items() if v["avg_ms"] > 0.05}
print(sys.argv[1] or "in-tree", d["ms_per_step"], d["match_count"], d["key_comparisons"], k)
PY
done
