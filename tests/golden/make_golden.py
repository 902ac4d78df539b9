"""Regenerates tests/golden/golden.json from the REFERENCE ITSELF.

Runs in the build container only: it loads oracle/_ref/libhgref.so, i.e. the
unmodified reference headers (/root/reference/proj/include) compiled by
oracle/Makefile, and records their outputs. The JSON is committed so the
oracle and the GPU engine are pinned against the reference on machines where
/root/reference does not exist (the GPU box).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import HASH_IDENTITY, Oracle, Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def fold_table(o: Oracle, t):
    inter = np.stack([t.keys, t.index], 1).ravel() if len(t.keys) else np.zeros(0, np.uint64)
    return {"offsets_fold": hex(o.fold(t.offsets)), "edges_fold": hex(o.fold(inter))}


def main() -> None:
    r = Reference()
    o = Oracle()  # only for mt19937_64 inputs and the fold helper
    g: dict = {"generator": "tests/golden/make_golden.py (reference headers via oracle/_ref)"}

    xs = [0, 1, 2, 123456789, 0xFFFFFFFF, 0xFFFFFFFFFFFFFFFF, 0x9E3779B97F4A7C15, 42, 1 << 63]
    g["mix64"] = [[hex(x), hex(r.mix64(x))] for x in xs]
    hv = []
    for key in [0, 1, 7, 123456789, 0xFFFFFFFF, 0xFFFFFFFFFFFFFFFF, 10121]:
        for seed in [0, 1, 42, 0xDEADBEEF]:
            for nv in [1, 2, 3, 5059, 65536, 1000003, (1 << 28), (1 << 32) + 15, (1 << 40) + 7]:
                hv.append([hex(key), hex(seed), hex(nv), hex(r.hash_to_vertex(key, seed, nv))])
    g["hash_to_vertex"] = hv

    # Config-1 known answers.
    n = 1 << 20
    keys = o.mt19937_64(1, n, mask_u32=True)
    probe = o.mt19937_64(1, n, skip=n, mask_u32=True)
    h = r.build_handle(keys, variant=1, sequential=True)
    t = r.export(h)
    c1 = {"n": n, "generator": "mt19937_64(1) & 0xffffffff; probes = next 2^20 draws",
          **fold_table(o, t),
          "offsets_1_4": [int(x) for x in t.offsets[1:5]],
          "offsets_mid": int(t.offsets[n // 2]),
          "empty_vertices": int((np.diff(t.offsets) == 0).sum()),
          "max_segment": int(np.diff(t.offsets).max())}
    c1["self_probe"] = {k: v for k, v in r.probe(h, keys).items() if k != "pairs"}
    c1["indep_probe"] = {k: v for k, v in r.probe(h, probe).items() if k != "pairs"}
    c1["sort_merge_indep"] = r.sort_merge_join_count(keys, probe)
    r.free(h)
    t2 = r.build(keys, variant=2, sequential=True)
    c1["v2_equal_v1_sequential"] = bool((t2.offsets == t.offsets).all()
                                        and (t2.keys == t.keys).all()
                                        and (t2.index == t.index).all())
    g["config1"] = c1

    # Small random cases: full sequential tables (tiny) + probe results.
    cases = []
    rng = np.random.default_rng(7)
    specs = [(0, 1.0, 1 << 15, 0, 0), (1, 1.0, 1 << 15, 0, 0), (37, 0.5, 4, 3, 0),
             (500, 2.0, 64, 42, 0), (1000, 4.0, 1, 0, 0), (777, 1.5, 16, 9, 0),
             (64, 1.0, 1 << 15, 0, 0), (300, 1.0, 8, 0, 1), (5, 5.0, 1 << 15, 0, 0)]
    for (n, load, bins, seed, identity) in specs:
        kr = int(rng.integers(1, 200))
        ks = rng.integers(0, kr, size=n, dtype=np.uint64) if n else np.zeros(0, np.uint64)
        if n == 64:
            ks = np.full(n, 5, np.uint64)  # single heavy key
        ps = rng.integers(0, kr + 20, size=max(n // 2, 3), dtype=np.uint64)
        hk = HASH_IDENTITY if identity else 0
        case = {"keys": [int(x) for x in ks], "probes": [int(x) for x in ps], "load": load,
                "bins": bins, "seed": seed, "hash_kind": hk}
        for variant in (1, 2):
            h = r.build_handle(ks, variant=variant, load=load, bins=bins, seed=seed,
                               sequential=True, hash_kind=hk)
            t = r.export(h, seed, hk)
            case[f"v{variant}"] = {"num_vertices": t.num_vertices,
                                   "offsets": [int(x) for x in t.offsets],
                                   "keys": [int(x) for x in t.keys],
                                   "index": [int(x) for x in t.index]}
            if variant == 1 and hk == 0:
                pr = r.probe(h, ps, materialize=True, cap=1 << 20)
                case["probe"] = {"match_count": pr["match_count"],
                                 "key_comparisons": pr["key_comparisons"],
                                 "pairs": sorted([[int(a), int(b)] for a, b in pr["pairs"]])}
            r.free(h)
        cases.append(case)
    g["cases"] = cases

    # probe_new / probe_new_prepared (join.hpp:143-182), incl. the
    # test_join.cpp:134-260 scenarios: random pairs, empty sides, shared V from
    # the larger side (load 2), heavy single key (cap), identity collisions.
    pn = []
    rng = np.random.default_rng(21)
    pspecs = [(800, 150, 700, 120, 1.0, 0, 0), (0, 1, 3, 4, 1.0, 0, 0), (3, 4, 0, 1, 1.0, 0, 0),
              (8, 0, 2, 0, 2.0, 0, 0), (64, 0, 64, 0, 1.0, 0, 0), (5, 0, 3, 0, 5.0, 0, 1),
              (2000, 300, 1500, 300, 0.5, 77, 0), (1200, 40, 900, 40, 4.0, 5, 0)]
    for (na, ra, nb, rb, load, seed, identity) in pspecs:
        if ra:
            a = rng.integers(0, ra, size=na, dtype=np.uint64)
            b = rng.integers(0, rb, size=nb, dtype=np.uint64)
        elif na == 8:
            a, b = np.arange(1, 9, dtype=np.uint64), np.array([3, 4], np.uint64)
        elif na == 64:
            a, b = np.full(64, 5, np.uint64), np.full(64, 5, np.uint64)
        else:
            a = np.array([3, 9, 3, 10121, 7], np.uint64)
            b = np.array([3, 10121, 11], np.uint64)
        hk = HASH_IDENTITY if identity else 0
        res = r.probe_new(a, b, load=load, seed=seed, hash_kind=hk, materialize=True,
                          cap=1 << 20)
        pn.append({"a": [int(x) for x in a], "b": [int(x) for x in b], "load": load,
                   "seed": seed, "hash_kind": hk, "match_count": res["match_count"],
                   "key_comparisons": res["key_comparisons"],
                   "pairs": sorted([[int(x), int(y)] for x, y in res["pairs"]])})
    g["probe_new"] = pn
    with open(OUT, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
