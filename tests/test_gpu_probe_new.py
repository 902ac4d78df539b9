"""GPU parity for probe_new / probe_new_prepared (join.hpp:143-182; SURVEY.md
8(f) rank 1) through the C-ABI (K12 k_intersect) against the oracle and the
reference-generated golden vectors (tests/golden/golden.json "probe_new").

Bar: match_count and key_comparisons identical; pair arrays identical to the
oracle's sequential emission order (vertex, A position, B position), hence
identical sorted pair sets; under a cap the kept pairs are the first cap of
that order. Scenarios follow test_join.cpp:134-260."""
import json
import os

import numpy as np
import pytest

import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import BuildConfig, ExecMode, IdentityHasher, ProbeOptions

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


@pytest.fixture(autouse=True)
def _need_gpu(cuda):
    yield


def pair_list(r):
    return [[int(p["left_index"]), int(p["right_index"])] for p in r.pairs]


@pytest.mark.parametrize("ci", range(len(GOLDEN["probe_new"])))
def test_golden_probe_new(ci):
    case = GOLDEN["probe_new"][ci]
    cfg = BuildConfig(load_factor=case["load"], hash_seed=case["seed"])
    hasher = IdentityHasher() if case["hash_kind"] == 1 else None
    r = hg.probe_new(np.array(case["a"], np.uint64), np.array(case["b"], np.uint64), cfg,
                     ProbeOptions(materialize=True, pair_cap=1 << 20), hasher=hasher)
    assert r.match_count == case["match_count"]
    assert r.key_comparisons == case["key_comparisons"]
    assert sorted(pair_list(r)) == case["pairs"]
    assert not r.truncated


def _tables(a, b, load=1.0, seed=0, width=8, variant=2, mode=ExecMode.parallel):
    nv = hg.derived_vertex_count(max(len(a), len(b)), load)
    cfg = BuildConfig(load_factor=load, hash_seed=seed, mode=mode)
    dt = np.uint64 if width == 8 else np.uint32
    build = hg.build_v2 if variant == 2 else hg.build_v1
    return (build(np.asarray(a, dt), cfg, vertex_count=nv),
            build(np.asarray(b, dt), cfg, vertex_count=nv))


@pytest.mark.parametrize("width", [4, 8])
@pytest.mark.parametrize("mode", [ExecMode.sequential, ExecMode.parallel])
def test_random_vs_oracle_exact_order(oracle, width, mode):
    # test_join.cpp:134-150; with identical tables the pair ARRAY equals the
    # oracle's sequential emission order.
    rng = np.random.default_rng(333 + width)
    for _ in range(12):
        a = rng.integers(0, int(rng.integers(100, 5000)), size=int(rng.integers(1, 20000)),
                         dtype=np.uint64)
        b = rng.integers(0, int(rng.integers(100, 5000)), size=int(rng.integers(1, 20000)),
                         dtype=np.uint64)
        load = float(rng.choice([0.25, 0.5, 1.0, 1.5, 2.0]))
        ta, tb = _tables(a, b, load, width=width, mode=mode)
        r = hg.probe_new_prepared(ta, tb, ProbeOptions(materialize=True, pair_cap=1 << 23))
        # oracle over the GPU tables' exact layout (intra-segment order included)
        from oracle.oracle import Table
        oa = Table(ta.num_vertices(), ta.offsets(), ta.edge_keys(), ta.edge_index())
        ob = Table(tb.num_vertices(), tb.offsets(), tb.edge_keys(), tb.edge_index())
        ro = oracle.probe_new_prepared(oa, ob, materialize=True, cap=1 << 23)
        assert r.match_count == ro["match_count"] == oracle.sort_merge_join_count(a, b)
        assert r.key_comparisons == ro["key_comparisons"]
        assert pair_list(r) == ro["pairs"].tolist()
        # and the sorted pair set equals probe_new from the raw inputs
        rn = oracle.probe_new(a, b, load=load, materialize=True, cap=1 << 23)
        assert sorted(pair_list(r)) == sorted(rn["pairs"].tolist())


def test_symmetric_and_vs_probe_standard(oracle):
    # test_join.cpp:146-157
    rng = np.random.default_rng(444)
    a = rng.integers(0, 80, size=600, dtype=np.uint64)
    b = rng.integers(0, 80, size=900, dtype=np.uint64)
    assert hg.probe_new(a, b).match_count == hg.probe_new(b, a).match_count
    assert hg.probe_new(a, b).match_count == hg.probe_standard(hg.build_v2(a), b).match_count


def test_empty_sides():
    # test_join.cpp:159-165
    a = np.array([1, 2, 3], np.uint64)
    e = np.zeros(0, np.uint64)
    assert hg.probe_new(a, e).match_count == 0
    assert hg.probe_new(e, a).match_count == 0
    assert hg.probe_new(e, e).match_count == 0


def test_shared_vertex_range_and_mismatch():
    # test_join.cpp:167-186
    a = np.arange(1, 9, dtype=np.uint64)
    b = np.array([3, 4], np.uint64)
    cfg = BuildConfig(load_factor=2.0)
    v = hg.derived_vertex_count(len(a), 2.0)
    ta, tb = hg.build_v2(a, cfg, vertex_count=v), hg.build_v2(b, cfg, vertex_count=v)
    assert ta.num_vertices() == tb.num_vertices() == 4
    assert hg.probe_new_prepared(ta, tb).match_count == 2
    assert hg.probe_new(a, b, cfg).match_count == 2
    with pytest.raises(hg.InvalidArgument):
        hg.probe_new_prepared(hg.build_v2(np.array([1, 2, 3, 4], np.uint64)),
                              hg.build_v2(np.array([1, 2], np.uint64)))


def test_comparisons_equal_segment_products():
    # test_join.cpp:189-205
    rng = np.random.default_rng(555)
    a = rng.integers(0, 64, size=700, dtype=np.uint64)
    b = rng.integers(0, 64, size=500, dtype=np.uint64)
    ta, tb = _tables(a, b)
    expect = int((np.diff(ta.offsets()).astype(np.int64) * np.diff(tb.offsets()).astype(np.int64)).sum())
    assert hg.probe_new_prepared(ta, tb).key_comparisons == expect


def test_cap_truncation_heavy_key(oracle):
    # test_join.cpp:226-243: 64 x 64 copies of one key (a long segment pair,
    # warp-cooperative path); the kept pairs are the first cap in order.
    a = np.full(64, 5, np.uint64)
    b = np.full(64, 5, np.uint64)
    r = hg.probe_new(a, b, BuildConfig(), ProbeOptions(materialize=True, pair_cap=100))
    assert r.match_count == 4096 and r.truncated and len(r.pairs) == 100
    # sequential layout: segments in input order, so the first 100 pairs are
    # the reference's sequential first 100
    r = hg.probe_new(a, b, BuildConfig(mode=ExecMode.sequential),
                     ProbeOptions(materialize=True, pair_cap=100))
    assert pair_list(r) == [[i // 64, i % 64] for i in range(100)]
    r = hg.probe_new(a, b, BuildConfig(), ProbeOptions(materialize=True, pair_cap=4096))
    assert not r.truncated and len(r.pairs) == 4096
    assert sorted(pair_list(r)) == [[i, j] for i in range(64) for j in range(64)]


def test_collision_fixture_identity():
    # test_join.cpp:245-260
    a = np.array([3, 9, 3, 10121, 7], np.uint64)
    b = np.array([3, 10121, 11], np.uint64)
    r = hg.probe_new(a, b, BuildConfig(load_factor=5.0),
                     ProbeOptions(materialize=True), hasher=IdentityHasher())
    assert r.match_count == 3 and r.key_comparisons == 15
    assert sorted(pair_list(r)) == [[0, 0], [2, 0], [3, 1]]


def test_skewed_long_segments_mixed(oracle):
    # mixture of short segments and heavy keys across many tiles: exercises
    # the look-back slot assignment, the warp-cooperative long path and
    # tiles whose key slices exceed the staged capacity (global fallback)
    rng = np.random.default_rng(9)
    heavy = rng.integers(0, 1 << 20, size=40, dtype=np.uint64)
    a = np.concatenate([rng.integers(0, 1 << 20, size=200000, dtype=np.uint64),
                        np.repeat(heavy, rng.integers(1, 300, size=40))])
    b = np.concatenate([rng.integers(0, 1 << 20, size=150000, dtype=np.uint64),
                        np.repeat(heavy, rng.integers(1, 200, size=40))])
    rng.shuffle(a)
    rng.shuffle(b)
    ta, tb = _tables(a, b, load=1.0, width=4)
    from oracle.oracle import Table
    oa = Table(ta.num_vertices(), ta.offsets(), ta.edge_keys(), ta.edge_index())
    ob = Table(tb.num_vertices(), tb.offsets(), tb.edge_keys(), tb.edge_index())
    ro = oracle.probe_new_prepared(oa, ob, materialize=True, cap=1 << 23)
    for cap in (1 << 23, ro["match_count"] // 3):
        r = hg.probe_new_prepared(ta, tb, ProbeOptions(materialize=True, pair_cap=cap))
        assert r.match_count == ro["match_count"]
        assert r.key_comparisons == ro["key_comparisons"]
        assert pair_list(r) == ro["pairs"][:cap].tolist()
    # a low-load table: slices larger than the staged capacity
    ta, tb = _tables(a, b, load=64.0, width=8)
    oa = Table(ta.num_vertices(), ta.offsets(), ta.edge_keys(), ta.edge_index())
    ob = Table(tb.num_vertices(), tb.offsets(), tb.edge_keys(), tb.edge_index())
    ro = oracle.probe_new_prepared(oa, ob, materialize=True, cap=1 << 23)
    r = hg.probe_new_prepared(ta, tb, ProbeOptions(materialize=True, pair_cap=1 << 23))
    assert r.match_count == ro["match_count"] and r.key_comparisons == ro["key_comparisons"]
    assert pair_list(r) == ro["pairs"].tolist()
