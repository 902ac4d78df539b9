"""CPU: pin the oracle (plain-C restatement) against the reference itself.

(1) SURVEY.md Appendix A golden vectors and tests/golden/golden.json (written
by tests/golden/make_golden.py from the compiled reference headers);
(2) when oracle/_ref is present, direct comparison with the reference on
random inputs, including parallel-mode builds (canonical segments)."""
import json
import os

import numpy as np
import pytest

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def test_appendix_a_mix64(oracle):
    assert oracle.mix64(0) == 0
    assert oracle.mix64(1) == 0xB456BCFC34C2CB2C
    assert oracle.mix64(2) == 0x3ABF2A20650683E7
    assert oracle.mix64(123456789) == 0x8F7C29206384F886
    assert oracle.mix64(0xFFFFFFFF) == 0xCC71ECDA2AA8BCC6
    assert oracle.mix64(0xFFFFFFFFFFFFFFFF) == 0x64B5720B4B825F21
    assert oracle.hash_to_vertex(123456789, 42, 65536) == 3765
    assert oracle.hash_to_vertex(123456789, 0, 1000003) == 28752


def test_golden_hash_vectors(oracle):
    for x, y in GOLDEN["mix64"]:
        assert oracle.mix64(int(x, 16)) == int(y, 16)
    for k, s, v, out in GOLDEN["hash_to_vertex"]:
        assert oracle.hash_to_vertex(int(k, 16), int(s, 16), int(v, 16)) == int(out, 16)


def test_derived_vertex_count_table(oracle):
    # test_core.cpp:34-43
    assert oracle.derived_vertex_count(10, 1.0) == 10
    assert oracle.derived_vertex_count(10, 2.0) == 5
    assert oracle.derived_vertex_count(10, 0.5) == 20
    assert oracle.derived_vertex_count(10, 4.0) == 2
    assert oracle.derived_vertex_count(3, 10.0) == 1
    assert oracle.derived_vertex_count(0, 1.0) == 1
    for bad in (0.0, -1.0):
        with pytest.raises(ValueError):
            oracle.derived_vertex_count(10, bad)


def test_config1_known_answers(oracle):
    c1 = GOLDEN["config1"]
    n = c1["n"]
    keys = oracle.mt19937_64(1, n, mask_u32=True)
    probe = oracle.mt19937_64(1, n, skip=n, mask_u32=True)
    t = oracle.build(keys)
    assert hex(oracle.fold(t.offsets)) == c1["offsets_fold"] == "0xcda71121e0620fe2"
    inter = np.stack([t.keys, t.index], 1).ravel()
    assert hex(oracle.fold(inter)) == c1["edges_fold"] == "0xee658543c1303331"
    assert t.offsets[1:5].tolist() == c1["offsets_1_4"]
    assert int(t.offsets[n // 2]) == c1["offsets_mid"]
    assert int((np.diff(t.offsets) == 0).sum()) == c1["empty_vertices"]
    assert int(np.diff(t.offsets).max()) == c1["max_segment"]
    for pk, name in ((keys, "self_probe"), (probe, "indep_probe")):
        r = oracle.probe_standard(t, pk)
        assert r["match_count"] == c1[name]["match_count"]
        assert r["key_comparisons"] == c1[name]["key_comparisons"]
    assert oracle.sort_merge_join_count(keys, probe) == c1["sort_merge_indep"]
    t2 = oracle.build(keys, variant=2)
    assert (t2.offsets == t.offsets).all() and (t2.keys == t.keys).all()
    assert (t2.index == t.index).all()


@pytest.mark.parametrize("ci", range(len(GOLDEN["cases"])))
def test_golden_cases(oracle, ci):
    case = GOLDEN["cases"][ci]
    for variant in (1, 2):
        t = oracle.build(case["keys"], variant=variant, load=case["load"], bins=case["bins"],
                         seed=case["seed"], hash_kind=case["hash_kind"])
        g = case[f"v{variant}"]
        assert t.num_vertices == g["num_vertices"]
        assert t.offsets.tolist() == g["offsets"]
        assert t.keys.tolist() == g["keys"]
        assert t.index.tolist() == g["index"]
        assert oracle.validate_csr(t, len(case["keys"]), case["keys"]) == 0
    if "probe" in case:
        t = oracle.build(case["keys"], load=case["load"], seed=case["seed"])
        r = oracle.probe_standard(t, case["probes"], materialize=True, cap=1 << 20)
        assert r["match_count"] == case["probe"]["match_count"]
        assert r["key_comparisons"] == case["probe"]["key_comparisons"]
        assert sorted(r["pairs"].tolist()) == case["probe"]["pairs"]


def test_hand_traced_fixture(oracle):
    # test_core.cpp:45-62 (identity hash, keys [5,1,5,9], V=4)
    t = oracle.build([5, 1, 5, 9], hash_kind=1)
    assert t.offsets.tolist() == [0, 0, 4, 4, 4]
    assert t.segment(1) == [(5, 0), (1, 1), (5, 2), (9, 3)]
    # test_core.cpp:64-88 (collision fixture, V=5059)
    t = oracle.build([3, 9, 3, 10121, 7], vertex_count=5059, hash_kind=1)
    assert t.segment(3) == [(3, 0), (3, 2), (10121, 3)]
    assert oracle.count_instances(t, 3) == 2
    assert oracle.count_instances(t, 10121) == 1
    assert oracle.count_instances(t, 5059 + 3) == 0


def test_exclusive_prefix_sum(oracle):
    # test_parallel.cpp:127-165
    assert oracle.exclusive_prefix_sum([1, 2, 0, 3]).tolist() == [0, 1, 3, 3, 6]
    assert oracle.exclusive_prefix_sum([]).tolist() == [0]
    with pytest.raises(OverflowError):
        oracle.exclusive_prefix_sum([0xFFFFFFFFFFFFFFFF, 1])


def test_validate_negative_cases(oracle):
    # test_core.cpp:260-289
    t = oracle.build([1, 2, 3, 4])
    assert oracle.validate_csr(t, 4) == 0
    assert oracle.validate_csr(t, 5) != 0
    k = t.keys.copy()
    k[0], k[-1] = k[-1], k[0]
    from oracle.oracle import Table
    bad = Table(t.num_vertices, t.offsets, k, t.index)
    if not (k == t.keys).all():
        assert oracle.validate_csr(bad, 4) != 0
    idx = t.index.copy()
    idx[-1] = idx[0]
    assert oracle.validate_csr(Table(t.num_vertices, t.offsets, t.keys, idx), 4) != 0


def test_oracle_matches_reference_random(oracle, reference):
    rng = np.random.default_rng(11)
    for _ in range(40):
        n = int(rng.integers(0, 3000))
        kr = int(rng.integers(1, 2000))
        keys = rng.integers(0, kr, size=n, dtype=np.uint64)
        load = float(rng.choice([0.25, 0.5, 1.0, 1.5, 2.0, 4.0]))
        bins = int(rng.choice([1, 7, 64, 1 << 15]))
        seed = int(rng.integers(0, 1 << 62))
        for variant in (1, 2):
            ro = oracle.build(keys, variant, load, bins, seed)
            rr = reference.build(keys, variant, load, bins, seed, sequential=True)
            assert (ro.offsets == rr.offsets).all()
            assert (ro.keys == rr.keys).all() and (ro.index == rr.index).all()
            # parallel-mode reference: same offsets and canonical segments
            rp = reference.build(keys, variant, load, bins, seed, sequential=False)
            assert (rp.offsets == ro.offsets).all()
            for a, b in zip(rp.canonical_segments(), ro.canonical_segments()):
                assert (a == b).all()
        probes = rng.integers(0, kr + 50, size=int(rng.integers(0, 2000)), dtype=np.uint64)
        h = reference.build_handle(keys, 1, load, bins, seed, sequential=True)
        rr = reference.probe(h, probes, materialize=True, cap=1 << 30)
        reference.free(h)
        ro = oracle.probe_standard(oracle.build(keys, 1, load, bins, seed), probes,
                                   materialize=True, cap=1 << 30)
        assert rr["match_count"] == ro["match_count"]
        assert rr["key_comparisons"] == ro["key_comparisons"]
        assert sorted(map(tuple, rr["pairs"].tolist())) == sorted(map(tuple, ro["pairs"].tolist()))


def test_keygen_restatement(oracle, reference):
    for n, mult, seed in [(1000, 1.0, 7), (5000, 16.0, 3), (10, 0.5, 0)]:
        assert (oracle.generate_uniform(n, mult, seed) ==
                reference.generate(1, n, mult, seed)).all()


@pytest.mark.parametrize("ci", range(len(GOLDEN["probe_new"])))
def test_golden_probe_new(oracle, ci):
    # join.hpp:143-182; reference outputs recorded by make_golden.py
    case = GOLDEN["probe_new"][ci]
    r = oracle.probe_new(case["a"], case["b"], load=case["load"], seed=case["seed"],
                         hash_kind=case["hash_kind"], materialize=True, cap=1 << 20)
    assert r["match_count"] == case["match_count"]
    assert r["key_comparisons"] == case["key_comparisons"]
    assert sorted(r["pairs"].tolist()) == case["pairs"]


def test_probe_new_matches_reference_random(oracle, reference):
    # test_join.cpp:134-150 (random vs nested loop), :152-157 (symmetric count),
    # :189-205 (comparisons = segment-product sum)
    rng = np.random.default_rng(333)
    for _ in range(25):
        a = rng.integers(0, int(rng.integers(1, 150)), size=int(rng.integers(1, 800)),
                         dtype=np.uint64)
        b = rng.integers(0, int(rng.integers(1, 150)), size=int(rng.integers(1, 800)),
                         dtype=np.uint64)
        load = float(rng.choice([0.5, 1.0, 2.0]))
        ro = oracle.probe_new(a, b, load=load, materialize=True, cap=1 << 20)
        rr = reference.probe_new(a, b, load=load, materialize=True, cap=1 << 20)
        assert ro["match_count"] == rr["match_count"] == oracle.sort_merge_join_count(a, b)
        assert ro["key_comparisons"] == rr["key_comparisons"]
        assert sorted(ro["pairs"].tolist()) == sorted(rr["pairs"].tolist())
        assert oracle.probe_new(b, a)["match_count"] == ro["match_count"]
    # mismatched vertex ranges (test_join.cpp:182-186)
    ta, tb = oracle.build([1, 2, 3, 4], variant=2), oracle.build([1, 2], variant=2)
    with pytest.raises(ValueError):
        oracle.probe_new_prepared(ta, tb)
    ha = reference.build_handle([1, 2, 3, 4], variant=2)
    hb = reference.build_handle([1, 2], variant=2)
    with pytest.raises(ValueError):
        reference.probe_new_prepared(ha, hb)
    reference.free(ha)
    reference.free(hb)
