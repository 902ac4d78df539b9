#!/usr/bin/env python
"""HashGraph build + probe benchmark (BASELINE.json metric, config C2).

One step = one pass of the hot path over one batch of synthetic input:
  build a HashGraph over N = 2^28 uniform u32 keys (splitmix64 seed 1, load 1,
  binned V2 build unless --variant 1), then probe_standard with M = 2^28
  independent u32 probe keys (splitmix64 seed 2), count only (ProbeOptions{}).
value = (N + M) / step time in G keys/s, inputs resident in HBM; e2e = the
same step through the public API with the keys and probes in pinned HOST
memory (H2D inside the timed region, result scalars read back).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) the table is sharded by hash range (weak scaling: each
rank contributes N keys and M probes); see paper_1907_02900_b200/sharded.py.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "build and probe Gkeys/s (2^28 uint32 keys) at 1/2/4/8 B200; % of HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--log2n", type=int, default=None,
                   help="c2: keys (and probes) per GPU, default 28; c5: TOTAL keys, default 32")
    p.add_argument("--config", default="c2", choices=["c2", "c5"],
                   help="c2: the BASELINE metric config (weak scaling, 2^28 per GPU); c5: "
                        "2^32 keys + 2^32 probes in total split over the GPUs (strong scaling)")
    p.add_argument("--variant", type=int, default=2, choices=[1, 2])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the per-phase/variant breakdown")
    p.add_argument("--cpu-log2n", type=int, default=None,
                   help="reference-arm sample size (default: the B200 arm's own --log2n, "
                        "i.e. the same config)")
    p.add_argument("--csv", default="bench_rows.csv",
                   help="reference bench CSV rows (hashgraph_bench.cpp:47-49 + B200 columns)")
    a = p.parse_args()
    if a.log2n is None:
        a.log2n = 32 if a.config == "c5" else 28
    return a


def per_gpu_log2n(args, world: int) -> int:
    """log2 of the keys (= probes) each GPU holds."""
    if args.config == "c5":
        return args.log2n - (world.bit_length() - 1)
    return args.log2n


def workload_config(log2n: int, variant: int, world: int, config: str = "c2") -> dict:
    """The `config` of both arms' JSON lines (identical for the same args);
    log2n = keys per GPU."""
    n = 1 << log2n
    if config == "c5":
        tot = (1 << log2n) * world
        return {"workload": f"C5: build_v{variant} over {tot} uniform u32 keys in total "
                            f"(splitmix64 seed 1, global positions), load 1, hash-range sharded "
                            f"over {world} GPU(s) + probe_standard (count) of {tot} u32 probes "
                            f"(seed 2); strong scaling",
                "n_total": tot, "m_total": tot, "n_per_gpu": n, "m_per_gpu": n,
                "load_factor": 1.0, "variant": variant, "vertices": tot,
                "l2": "inputs larger than L2",
                "parallelism": f"hash-range shards x{world}" if world > 1 else "1 GPU"}
    return {"workload": f"C2: build_v{variant} over 2^{log2n} uniform u32 keys (splitmix64 "
                        f"seed 1) at load 1 + probe_standard (count) of 2^{log2n} u32 probes "
                        f"(seed 2), per GPU",
            "n_per_gpu": n, "m_per_gpu": n, "load_factor": 1.0, "variant": variant,
            "vertices": n,
            "l2": "inputs larger than L2 (1 GiB keys + 1 GiB probes per GPU vs 126 MB L2)",
            "parallelism": f"hash-range shards x{world}" if world > 1 else "1 GPU"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# SURVEY.md 8(d) reference-loop-nest bytes (the roofline numerators of the
# phase figures): sk/sv/so key/value/offset widths, sc = 4-byte counters.
def ref_bytes_build(variant, n, v, sk=4, sv=4, so=4, sc=4, bins=1 << 15):
    if variant == 1:
        return n * (3 * sk + sv) + v * (7 * sc + 2 * so) + so
    b = min(bins, v)
    return n * (6 * sk + 3 * sv) + (v + b) * (7 * sc + 2 * so) + 2 * so


def ref_bytes_probe(m, v, c, sk=4, so=4, sc=4):
    return m * sk + (v + 1) * so + c * sk + m * sc


def ref_bytes_probe_pairs(m, v, c, p, sk=4, so=4, sc=4, sv=4, si=4):
    return (ref_bytes_probe(m, v, c, sk, so, sc) + m * sc + (m + 1) * 8 +
            m * sk + (v + 1) * so + c * sk + 8 * m + p * sv + 2 * p * si)


def roof(bytes_, ms, peak):
    gbs = bytes_ / (ms * 1e-3) / 1e9
    return {"alg_bytes": int(bytes_), "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}


# ------------------------------------------------------------------ helpers

def splitmix_u32(seed: int, start: int, n: int) -> np.ndarray:
    """SURVEY.md Appendix B generator on the host (numpy, wrapping u64)."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z & np.uint64(0xFFFFFFFF)).astype(np.uint32)


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def alg_bytes(name: str, n: int, v: int, m: int, c: int, kb: int = 4, vb: int = 4,
              ob: int = 4, probe_ent: int = 4) -> int:
    """Algorithmic bytes of ONE launch of kernel `name`:
    compulsory traffic at array granularity -- each pass reads each input
    array once and writes each output array once. n build keys, v vertices,
    m probes, c key comparisons; kb/vb/ob key/value/offset widths; probe_ent
    = bytes of a partitioned probe entry (4: key only for count-only probes)."""
    e = kb + vb  # build entry (key, value)
    return {
        # simple build (V1)
        "k1_hash_count": n * kb + 2 * v * ob,
        "k2_scan": 2 * v * ob,
        "k3_scatter": n * kb + 2 * v * ob + n * e,
        # binned build (V2)
        "k4_part_hist": n * kb,
        "k6a_multisplit": n * kb + n * e,
        "k6b_multisplit": 2 * n * e,
        "k7_part_build": n * e + n * e + v * ob,
        # partitioned probe
        "p4_part_hist": m * kb,
        "p6a_multisplit": m * kb + m * probe_ent,
        "p6b_multisplit": 2 * m * probe_ent,
        "k8p_probe_part": m * probe_ent + (v + 1) * ob + n * kb,
        # direct probe
        "k8_probe_count": m * kb + (v + 1) * ob + c * kb,
    }.get(name, 0)


def reference_alg_bytes(variant: int, n: int, v: int, m: int, c: int, kb: int = 4, vb: int = 4,
                        ob: int = 4, sc: int = 4, bins: int = 1 << 15) -> int:
    """SURVEY.md 8(d) reference-loop-nest bytes of one step (build + count-only
    probe): V1 = N(3sk+sv) + V(7sc+2so) + so, V2 = N(6sk+3sv) + (V+B)(7sc+2so)
    + 2so, probe = M sk + (V+1) so + C sk + M sc."""
    if variant == 1:
        build = n * (3 * kb + vb) + v * (7 * sc + 2 * ob) + ob
    else:
        build = n * (6 * kb + 3 * vb) + (v + bins) * (7 * sc + 2 * ob) + 2 * ob
    return build + m * kb + (v + 1) * ob + c * kb + m * sc


# ------------------------------------------------------------------ reference arm

def cpu_reference_rate(variant: int, log2n: int, trials: int, warmup: int, threads=None):
    """The reference's own CPU implementation (oracle/_ref = the unmodified
    reference headers, -O3 x86-64-v4 on AVX-512 hosts; oracle port when _ref
    is absent) on the host cores: build + probe_standard of 2^log2n keys and
    probes of the same workload (table allocation inside the timed region, as
    in the reference bench)."""
    from oracle.oracle import Oracle, Reference, have_reference
    n = 1 << log2n
    keys = splitmix_u32(1, 0, n).astype(np.uint64)
    probes = splitmix_u32(2, 0, n).astype(np.uint64)
    threads = threads or os.cpu_count() or 1
    so = None
    if have_reference():
        ref, kind = Reference(), "reference"
        so = os.path.basename(ref.path)
        ref.set_threads(threads)

        def one():
            h = ref.build_handle(keys, variant=variant)
            r = ref.probe(h, probes)
            ref.free(h)
            return r["match_count"]
    else:  # pragma: no cover - the GPU box ships the prebuilt oracle/_ref
        ref, kind, threads = Oracle(), "port", 1

        def one():
            t = ref.build(keys, variant=variant)
            return ref.probe_standard(t, probes)["match_count"]
    for _ in range(warmup):
        one()
    times = []
    for _ in range(trials):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": 2 * n / med / 1e9, "unit": "Gkeys/s", "cores": threads, "kind": kind,
            "sample": f"build_v{variant} + probe_standard (count) of 2^{log2n} u32 keys "
                      f"(splitmix seed 1) and 2^{log2n} probes (seed 2), load 1; median of "
                      f"{trials} after {warmup} warm-up; HASHGRAPH_THREADS={threads}",
            "seconds_median": med, "seconds": times, "cpu_model": cpu_model(),
            "nproc": os.cpu_count(), "library": so}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on the box's
    host cores, all threads, on this arm's config (2^log2n keys + probes per
    step; at N > 1 rank 0 runs one GPU's share as the sample)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    own = per_gpu_log2n(args, world)
    log2n = args.cpu_log2n or min(own, 28)
    steps = max(1, args.steps)
    # each step is a full 2^28 build + probe (~10-20 s on 16 cores): cap the
    # warm-up so K steps + W warm-ups end within a few minutes
    warm = min(args.warmup, 1)
    res = cpu_reference_rate(args.variant, log2n, steps, warm)
    cfg = workload_config(own, args.variant, world, args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": "Gkeys/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": res["seconds_median"] * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c5" else "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": cfg,
        "same_config": log2n == own and world == 1 and args.config == "c2",
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample",
                                              "cpu_model", "nproc", "library")},
        "e2e": {"value": res["value"], "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ secondary configs

def log(msg: str) -> None:
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def _timed(torch, stream, fn, reps=3):
    """Average ms of fn() over reps (after one untimed call), CUDA events on `stream`."""
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def bench_c3(torch, hg, stream, sp, peak, rows, log2n=28):
    """C3: 2^28 u64 keys ~ Zipf(s = 1.0) over 2^24 ranks with u64 values,
    binned and simple builds across the load sweep (G keys/s = N / t), and
    probe_standard (count) of 2^28 probes of uniformly drawn ranks (seed 2)
    into each V2 table (G probes/s = M / t): every rank is probed equally, so
    the heavy ranks' long segments are walked (by the warp) about M / 2^24
    times each. (Zipf-distributed probes would make the join itself explode:
    the top rank holds ~6 % of both sides, ~2^48 comparisons.) Rooflines from
    SURVEY.md 8(d) bytes with the exact C."""
    n = 1 << log2n
    cdf = torch.tensor(hg.zipf_cdf(1 << 24, 1.0), dtype=torch.float64, device="cuda")
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    hg.generate(keys, kind=3, seed=1, ref=cdf)
    probes = torch.empty(n, dtype=torch.int64, device="cuda")
    ucdf = torch.arange(1, (1 << 24) + 1, dtype=torch.float64, device="cuda") / float(1 << 24)
    hg.generate(probes, kind=3, seed=2, ref=ucdf)  # uniform ranks through the same key map
    del ucdf
    vals = torch.arange(n, dtype=torch.int64, device="cuda")
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = {"workload": "2^28 u64 Zipf(1.0) keys over 2^24 ranks, u64 values = position; "
                       "2^28 probes of uniform ranks (seed 2)"}
    for load in (0.5, 1.0, 1.5, 2.0, 4.0):
        row = {}
        nv = hg.derived_vertex_count(n, load)
        so = 4 if nv <= (1 << 32) else 8
        for name, var, bfn in (("v2", 2, hg.build_v2), ("v1", 1, hg.build_v1)):
            cfg = hg.BuildConfig(load_factor=load)
            ms = _timed(torch, stream, lambda: bfn(keys, cfg, vals=vals, stream=sp).close(sp),
                        reps=2 if name == "v1" else 3)
            row[name] = {"build_ms": round(ms, 3), "build_gkeys_s": round(n / (ms * 1e-3) / 1e9, 3),
                         "roofline": roof(ref_bytes_build(var, n, nv, 8, 8, so), ms, peak)}
            rows.append(csv_row("build", f"hg_{name}", n, load, ms, n, mult="zipf1.0",
                                alg=row[name]["roofline"]))
        t = hg.build_v2(keys, hg.BuildConfig(load_factor=load), vals=vals, stream=sp)
        ms = _timed(torch, stream, lambda: hg.probe_device(t, probes, res, stream=sp))
        res.zero_()
        hg.probe_device(t, probes, res, stream=sp)
        mc, cmp = (int(x) for x in res.cpu().tolist())
        t.close(sp)
        row["probe"] = {"probe_ms": round(ms, 3), "gprobes_s": round(n / (ms * 1e-3) / 1e9, 3),
                        "match_count": mc, "key_comparisons": cmp,
                        "roofline": roof(ref_bytes_probe(n, nv, cmp, 8, so), ms, peak)}
        rows.append(csv_row("probe", "probe_standard", n, load, ms, n, mult="zipf1.0", matches=mc,
                            alg=row["probe"]["roofline"]))
        out[f"load_{load}"] = row
    del keys, vals, probes
    torch.cuda.empty_cache()
    return out


def bench_c4(torch, hg, stream, sp, peak, rows):
    """C4: probe_standard with pairs, 2^29 probes into 2^28 unique u32 build
    keys at hit ratio 0.1 / 0.5 / 1.0 (G probes/s = M / t, u32 pairs);
    roofline from SURVEY.md 8(d)'s pairs formula with the exact C and P."""
    n, m = 1 << 28, 1 << 29
    build = torch.empty(n, dtype=torch.int32, device="cuda")
    hg.generate(build, kind=2)
    t = hg.build_v2(build, stream=sp)
    probes = torch.empty(m, dtype=torch.int32, device="cuda")
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    pairs = torch.empty((m, 2), dtype=torch.int32, device="cuda")
    out = {"workload": "build 2^28 unique u32 (scramble31), probe 2^29 u32 with u32 pairs"}
    for h in (0.1, 0.5, 1.0):
        hg.generate(probes, kind=1, seed=3, hit=h, ref=build)
        ms = _timed(torch, stream, lambda: hg.probe_device(t, probes, res, pairs=pairs,
                                                           pair_width=4, pair_cap=m, stream=sp))
        res.zero_()
        hg.probe_device(t, probes, res, pairs=pairs, pair_width=4, pair_cap=m, stream=sp)
        mc, cmp = (int(x) for x in res.cpu().tolist())
        out[f"hit_{h}"] = {"probe_ms": round(ms, 3),
                           "gprobes_s": round(m / (ms * 1e-3) / 1e9, 3),
                           "match_count": mc, "key_comparisons": cmp,
                           "roofline": roof(ref_bytes_probe_pairs(m, n, cmp, mc), ms, peak)}
        rows.append(csv_row("probe", "probe_standard", m, 1.0, ms, m, mult=f"hit{h}", matches=mc,
                            alg=out[f"hit_{h}"]["roofline"]))
    t.close(sp)
    del build, probes, pairs
    torch.cuda.empty_cache()
    return out


def bench_multiplicity(torch, hg, stream, sp, peak, rows, log2n=28):
    """build_v2 at key multiplicity 1 vs 32 (acceptance_main.cpp:234-273,
    criterion 4; the paper reports < 15 % slowdown). Keys come
    from the reference's own generator (keygen.hpp:59-73, uniform_multiplicity,
    sequential mt19937_64 -- oracle/_ref) handed over as HGKEYS01 files and
    read straight into device memory (hg_keys_read)."""
    import tempfile
    from oracle.oracle import Reference, have_reference
    if not have_reference():
        return {"skipped": "oracle/_ref (compiled reference generator) absent"}
    n = 1 << log2n
    ref = Reference()
    out = {"workload": f"build_v2 of 2^{log2n} keys from keygen uniform_multiplicity "
                       f"(seeds 101 / 102, hash_seed 9 as acceptance criterion 4), u32 on device"}
    rates = {}
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    with tempfile.TemporaryDirectory() as d:
        for mult, seed in ((1.0, 101), (32.0, 102)):
            path = os.path.join(d, f"m{int(mult)}.keys")
            ref.write_keys(path, ref.generate(1, n, mult, seed))
            hg.read_keys(path, out=keys)
            os.unlink(path)
            cfg = hg.BuildConfig(hash_seed=9)
            ms = _timed(torch, stream, lambda: hg.build_v2(keys, cfg, stream=sp).close(sp))
            rates[mult] = n / (ms * 1e-3) / 1e9
            out[f"mult_{int(mult)}"] = {"build_ms": round(ms, 3),
                                       "build_gkeys_s": round(rates[mult], 3),
                                       "roofline": roof(ref_bytes_build(2, n, n), ms, peak)}
            rows.append(csv_row("build", "hg_v2", n, 1.0, ms, n, mult=str(mult), seed=seed,
                                alg=out[f"mult_{int(mult)}"]["roofline"]))
    out["slowdown_32_vs_1"] = round(1.0 - rates[32.0] / rates[1.0], 4)
    del keys
    torch.cuda.empty_cache()
    return out


CSV_HEADER = ("experiment,algo,n,load_factor,bins,multiplicity,seed,trials,threads,"
              "median_seconds,keys_per_second,match_count,truncated,"
              "gpus,bytes_algorithmic,roofline_achieved,dram_bytes_measured,cpu_cores")


def csv_row(experiment, algo, n, load, ms, keys, mult="1", seed=1, matches=0, alg=None,
            trials=3, gpus=1, threads=0, dram=""):
    """One row of the reference bench's CSV (hashgraph_bench.cpp:47-49,
    CsvWriter::row) extended per SURVEY.md 5 with gpus, bytes_algorithmic,
    roofline_achieved, dram_bytes_measured and cpu_cores."""
    sec = ms * 1e-3
    return (f"{experiment},{algo},{n},{load:g},{1 << 15},{mult},{seed},{trials},{threads},"
            f"{sec:.9f},{keys / sec:.3f},{matches},0,{gpus},"
            f"{alg['alg_bytes'] if alg else ''},{alg['frac'] if alg else ''},{dram},{threads}")


# ------------------------------------------------------------------ B200 arm

def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1907_02900_b200 as hg
    from paper_1907_02900_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c5 = args.config == "c5"
    if c5:  # the whole config is too large for the CPU arm and the pinned e2e copies
        args.no_cpu = args.no_e2e = args.no_extras = True
    log2n = per_gpu_log2n(args, world)
    n = m = 1 << log2n
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    keys = torch.empty(n, dtype=torch.int32, device=dev)
    probes = torch.empty(m, dtype=torch.int32, device=dev)
    hg.generate(keys, kind=0, seed=1, start=rank * n)
    hg.generate(probes, kind=0, seed=2, start=rank * m)
    result = torch.zeros(2, dtype=torch.int64, device=dev)
    build = hg.build_v2 if args.variant == 2 else hg.build_v1

    if world > 1:
        from paper_1907_02900_b200 import sharded
        engine = sharded.ShardedHashGraph(world, rank, variant=args.variant)

        def step():
            engine.build_and_probe(keys, probes, result)
    else:
        def step():
            t = build(keys, stream=sp)
            hg.probe_device(t, probes, result, stream=sp)
            t.close(sp)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    nv = hg.derived_vertex_count(n, 1.0)
    if world > 1:
        engine.exchange_events = None  # the timed steps run un-instrumented

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region (device-resident inputs; each input 1 GiB > 126 MB L2)
    # The step time comes from this un-instrumented region; the per-kernel
    # averages (roofline, launch count) from an identical pass right after it
    # with the library's event timeline on (its 2 events per launch cost ~2 %
    # of the step, so they stay out of `value`).
    dbg = os.environ.get("BENCH_DEBUG", "")
    _lib.profiler_enable(False)
    _lib.profiler_collect()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local if "noclock" not in dbg else 10 ** 6)
    barrier()
    with clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            h0 = time.perf_counter()
            step()
            if "sync" in dbg:
                torch.cuda.synchronize()
            if dbg:
                log(f"step host {1e3 * (time.perf_counter() - h0):.1f} ms")
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    _lib.profiler_enable("noprof" not in dbg)
    _lib.profiler_collect()
    if world > 1:
        engine.exchange_events = []  # the exchange timing comes from the instrumented pass too
    for _ in range(args.steps):
        step()
    barrier()
    _lib.profiler_enable(False)
    kern = _lib.profiler_collect()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * (n + m) / (ms * 1e-3) / 1e9
    nvlink = None
    if world > 1:
        # NVLink 5 roofline of the exchanges: bytes this rank sends to other
        # ranks per step (routed key records + probe keys) over the device
        # time of its all-to-alls, against 900 GB/s per direction per GPU
        xms = engine.exchange_ms() / args.steps
        xb = int(engine.last_build_bytes + engine.last_probe_bytes)
        t_ = torch.tensor([xms, float(xb)], device=dev, dtype=torch.float64)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        xms_max, xb_max = float(t_[0]), float(t_[1])
        nvlink = {"bytes_per_rank_per_step": xb, "exchange_ms_per_step": round(xms, 4),
                  "achieved_gbs": round(xb / (xms * 1e-3) / 1e9, 1) if xms else None,
                  "peak_gbs": 900.0, "peak_source": "NVLink 5, 900 GB/s per direction per GPU",
                  "frac": round(xb / (xms * 1e-3) / 1e9 / 900.0, 4) if xms else None,
                  "max_over_ranks": {"exchange_ms": round(xms_max, 4), "bytes": int(xb_max)},
                  "exchange_share_of_step": round(xms / ms, 4)}
    matches, comparisons = (int(x) for x in result.cpu().tolist())
    gpu_launches = sum(l for (l, _) in kern.values())

    # ---- roofline of the dominant kernel (algorithmic bytes / avg launch time)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks else "fallback 6.65 TB/s"
    local_n = n if world == 1 else int(engine.last_local_n)
    local_m = m if world == 1 else int(engine.last_local_m)
    local_v = nv if world == 1 else int(engine.local_vertices)
    if not kern:  # BENCH_DEBUG=noprof: step time only
        print(json.dumps({"ms_per_step": round(ms, 4), "value": round(value, 3)}))
        return
    dom = max((k for k in kern if alg_bytes(k, 1, 1, 1, 1) > 0), key=lambda k: kern[k][1])
    dl, dms = kern[dom]
    avg_ms = dms / dl
    # alg_bytes() is the kernel's traffic for the whole step (summed over its
    # launches when a sliced table launches it once per vertex-range slice)
    ab_step = alg_bytes(dom, local_n, local_v, local_m, comparisons if world == 1 else
                        int(engine.last_local_c))
    ab = ab_step * args.steps // dl  # per launch
    achieved = ab / (avg_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("kernels", {}).get(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "alg_bytes_per_launch": ab, "avg_launch_ms": round(avg_ms, 4),
                "peak_source": peak_src,
                "launch_times": "library CUDA-event timeline over K instrumented steps run right after the un-instrumented timed region",
                "step_alg_bytes": sum(alg_bytes(k, local_n, local_v, local_m, comparisons)
                                      for k in kern)}
    ref_bytes = reference_alg_bytes(args.variant, local_n, local_v, local_m,
                                    comparisons if world == 1 else int(engine.last_local_c))
    roofline["step_alg_frac"] = round(roofline["step_alg_bytes"] / (ms * 1e-3) / 1e9 / peak, 4)
    roofline["step_reference_alg_bytes"] = ref_bytes
    roofline["step_reference_frac"] = round(ref_bytes / (ms * 1e-3) / 1e9 / peak, 4)
    kernels = {k: {"launches": l, "avg_ms": round(t / l, 4), "share": round(t / sum(
        x[1] for x in kern.values()), 4)} for k, (l, t) in sorted(kern.items(), key=lambda x: -x[1][1])}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gkeys/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong" if c5 else "weak", "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": workload_config(log2n, args.variant, world, args.config),
        "roofline": roofline,
        "nvlink": nvlink,
        "clocks": clocks.summary(),
        "gpu_launches": gpu_launches,
        "match_count": matches, "key_comparisons": comparisons,
        "kernels": kernels,
    }

    # ---- per-phase / per-variant breakdown (device-resident, outside the timed region)
    rows = []
    rows.append(csv_row("join", f"hg_v{args.variant}+probe_standard", n, 1.0, ms, n + m,
                        matches=matches, trials=args.steps, gpus=world,
                        alg={"alg_bytes": roofline["step_alg_bytes"],
                             "frac": roofline["step_alg_frac"]}))
    if not args.no_extras and world == 1:
        extras = {}
        for var, bfn in ((1, hg.build_v1), (2, hg.build_v2)):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            reps = 3
            tb = tp = 0.0
            for _ in range(reps):
                e0.record(stream)
                t = bfn(keys, stream=sp)
                e1.record(stream)
                hg.probe_device(t, probes, result, stream=sp)
                e2.record(stream)
                t.close(sp)
                torch.cuda.synchronize()
                tb += e0.elapsed_time(e1)
                tp += e1.elapsed_time(e2)
            bms, pms = tb / reps, tp / reps
            extras[f"v{var}"] = {"build_ms": round(bms, 4),
                                 "build_gkeys_s": round(n / (bms * 1e-3) / 1e9, 3),
                                 "build_roofline": roof(ref_bytes_build(var, n, nv), bms, peak),
                                 "probe_ms": round(pms, 4),
                                 "probe_gkeys_s": round(m / (pms * 1e-3) / 1e9, 3),
                                 "probe_roofline": roof(ref_bytes_probe(m, nv, comparisons), pms,
                                                        peak)}
            rows.append(csv_row("build", f"hg_v{var}", n, 1.0, bms, n,
                                alg=extras[f"v{var}"]["build_roofline"]))
            rows.append(csv_row("probe", "probe_standard", m, 1.0, pms, m, matches=matches,
                                alg=extras[f"v{var}"]["probe_roofline"]))
        # probe_new (join.hpp:170-182): second table over the probes with the
        # shared V, then the K12 intersect (count only)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        tb = ti = 0.0
        reps = 3
        ta = hg.build_v2(keys, stream=sp)
        warm = hg.build_v2(probes, vertex_count=nv, stream=sp)  # pool warm-up (untimed)
        hg.probe_new_device(ta, warm, result, stream=sp)
        warm.close(sp)
        torch.cuda.synchronize()
        for _ in range(reps):
            e0.record(stream)
            tbl_b = hg.build_v2(probes, vertex_count=nv, stream=sp)
            e1.record(stream)
            hg.probe_new_device(ta, tbl_b, result, stream=sp)
            e2.record(stream)
            tbl_b.close(sp)
            torch.cuda.synchronize()
            tb += e0.elapsed_time(e1)
            ti += e1.elapsed_time(e2)
        ta.close(sp)
        pn_matches, pn_cmp = (int(x) for x in result.cpu().tolist())
        ib = (nv + 1) * 4 * 2 + (n + m) * 4  # offsets of both tables + both key arrays
        extras["probe_new"] = {
            "build_b_ms": round(tb / reps, 4), "intersect_ms": round(ti / reps, 4),
            "intersect_gkeys_s": round((n + m) / (ti / reps * 1e-3) / 1e9, 3),
            "intersect_alg_gbs": round(ib / (ti / reps * 1e-3) / 1e9, 1),
            "intersect_roofline": roof(ib, ti / reps, peak),
            "join_gkeys_s": round((n + m) / ((tb / reps + extras["v2"]["build_ms"] + ti / reps)
                                             * 1e-3) / 1e9, 3),
            "match_count": pn_matches, "key_comparisons": pn_cmp,
            "matches_equal_probe_standard": pn_matches == matches}
        rows.append(csv_row("probe", "probe_new", n + m, 1.0, ti / reps, n + m,
                            matches=pn_matches, alg=extras["probe_new"]["intersect_roofline"]))
        log("c3")
        extras["c3_zipf"] = bench_c3(torch, hg, stream, sp, peak, rows)
        log("c4")
        extras["c4_join"] = bench_c4(torch, hg, stream, sp, peak, rows)
        log("multiplicity")
        extras["multiplicity"] = bench_multiplicity(torch, hg, stream, sp, peak, rows)
        log("phases done")
        line["phases"] = extras

    # ---- e2e through the public API with pinned HOST buffers
    if not args.no_e2e and world == 1:
        log("e2e")
        hkeys = keys.cpu().pin_memory()
        hprobes = probes.cpu().pin_memory()
        torch.cuda.synchronize()

        def e2e_step():
            t = build(hkeys, stream=sp)           # H2D of the keys inside hg_build
            # H2D of the probes (chunked, overlapping the build still running:
            # the pinned buffer is final, HG_PROBE_HOST_READY), D2H of the totals
            r = hg.probe_standard(t, hprobes, host_ready=True)
            t.close(sp)
            return r

        e2e_step()
        e2e_step()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            r = e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        e_ms = f0.elapsed_time(f1) / args.steps
        assert r.match_count == matches, "e2e result differs from device-resident result"
        line["e2e"] = {"value": round((n + m) / (e_ms * 1e-3) / 1e9, 3), "unit": "Gkeys/s",
                       "ms_per_step": round(e_ms, 3), "h2d_bytes_per_step": 4 * (n + m),
                       "d2h_bytes_per_step": 16,
                       "path": "hashgraph.build_v2/probe_standard -> C-ABI hg_build/hg_probe "
                               "with pinned host buffers"}

    # ---- e2e at N > 1: every rank stages its pinned host slice (H2D inside
    # the timed region), runs the sharded step through ShardedHashGraph and
    # reads the global totals back; max over ranks
    if not args.no_e2e and world > 1:
        hkeys = keys.cpu().pin_memory()
        hprobes = probes.cpu().pin_memory()
        dk, dp = torch.empty_like(keys), torch.empty_like(probes)

        def e2e_step():
            dk.copy_(hkeys, non_blocking=True)
            dp.copy_(hprobes, non_blocking=True)
            engine.build_and_probe(dk, dp, result)
            return result.cpu()

        e2e_step()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            r = e2e_step()
        f1.record(stream)
        barrier()
        e_ms = torch.tensor([f0.elapsed_time(f1) / args.steps], device=dev)
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        assert int(r[0]) == matches, "e2e result differs from device-resident result"
        line["e2e"] = {"value": round(world * (n + m) / (e_ms * 1e-3) / 1e9, 3), "unit": "Gkeys/s",
                       "ms_per_step": round(e_ms, 3), "h2d_bytes_per_step": 4 * (n + m) * world,
                       "d2h_bytes_per_step": 16 * world,
                       "path": "pinned host slices -> ShardedHashGraph.build_and_probe (C-ABI "
                               "hg_route / hg_build / hg_probe, NCCL all_to_all) -> totals"}

    if not args.no_cpu and world == 1 and rank == 0:
        log("cpu baseline")
        # the reference on the host cores: the same 2^28 config, all threads,
        # two trials (~30 s of CPU work), plus a 1-thread row on a 2^22 sample
        try:
            keys_ = ("value", "unit", "cores", "kind", "sample", "cpu_model", "nproc", "library")
            cb = cpu_reference_rate(args.variant, args.cpu_log2n or log2n, trials=2, warmup=0)
            line["cpu_baseline"] = {k: cb[k] for k in keys_}
            c1 = cpu_reference_rate(args.variant, 22, trials=3, warmup=1, threads=1)
            line["cpu_baseline"]["threads_1"] = {k: c1[k] for k in ("value", "unit", "cores",
                                                                     "sample")}
            rows.append(csv_row("join", f"ref_hg_v{args.variant}+probe_standard", n, 1.0,
                                cb["seconds_median"] * 1e3, 2 * (1 << (args.cpu_log2n or log2n)),
                                trials=2, gpus=0, threads=cb["cores"]))
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0 and args.csv:
        with open(args.csv, "w") as f:
            f.write(CSV_HEADER + "\n" + "\n".join(rows) + "\n")
        line["csv"] = args.csv

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
