"""GPU parity: the sm_100a engine (through the C-ABI) against the oracle and
the golden vectors generated from the reference itself.

Bar: bit-identical offsets; identical per-vertex (key,
index) multisets (exact edge arrays in ExecMode::sequential); identical
match_count / key_comparisons; identical sorted pair sets."""
import json
import os

import numpy as np
import pytest

import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import BuildConfig, ExecMode, IdentityHasher, ProbeOptions

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
BUILDS = {1: hg.build_v1, 2: hg.build_v2}


@pytest.fixture(autouse=True)
def _need_gpu(cuda):
    yield


def canon(offsets, keys, index):
    nv = len(offsets) - 1
    seg = np.repeat(np.arange(nv, dtype=np.uint64), np.diff(offsets).astype(np.int64))
    order = np.lexsort((index, keys, seg))
    return keys[order], index[order]


def assert_same_table(t, o, exact: bool):
    assert t.num_vertices() == o.num_vertices
    assert t.num_edges() == len(o.keys)
    assert (t.offsets() == o.offsets).all(), "offsets differ"
    if exact:
        assert (t.edge_keys() == o.keys).all(), "edge keys differ (sequential layout)"
        assert (t.edge_index() == o.index).all(), "edge index differ (sequential layout)"
    else:
        a = canon(t.offsets(), t.edge_keys(), t.edge_index())
        b = canon(o.offsets, o.keys, o.index)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all(), "segment multisets differ"


@pytest.mark.parametrize("ci", range(len(GOLDEN["cases"])))
@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("mode", [ExecMode.sequential, ExecMode.parallel])
def test_golden_cases(ci, variant, mode):
    case = GOLDEN["cases"][ci]
    g = case[f"v{variant}"]
    cfg = BuildConfig(load_factor=case["load"], bin_count=case["bins"], hash_seed=case["seed"],
                      mode=mode)
    hasher = IdentityHasher() if case["hash_kind"] == 1 else None
    keys = np.array(case["keys"], np.uint64)
    t = BUILDS[variant](keys, cfg, hasher=hasher)
    assert t.num_vertices() == g["num_vertices"]
    assert t.offsets().tolist() == g["offsets"]
    if mode == ExecMode.sequential:
        assert t.edge_keys().tolist() == g["keys"]
        assert t.edge_index().tolist() == g["index"]
    else:
        a = canon(t.offsets(), t.edge_keys(), t.edge_index())
        b = canon(np.array(g["offsets"], np.uint64), np.array(g["keys"], np.uint64),
                  np.array(g["index"], np.uint64))
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    assert hg.validate_csr(t, len(keys), keys) is None
    if "probe" in case and variant == 1:
        r = hg.probe_standard(t, np.array(case["probes"], np.uint64),
                              ProbeOptions(materialize=True, pair_cap=1 << 20))
        assert r.match_count == case["probe"]["match_count"]
        assert r.key_comparisons == case["probe"]["key_comparisons"]
        got = sorted([[int(p["left_index"]), int(p["right_index"])] for p in r.pairs])
        assert got == case["probe"]["pairs"]
        assert not r.truncated


def test_hand_traced_identity_fixture():
    # test_core.cpp:45-62
    t = hg.build_v1([5, 1, 5, 9], BuildConfig(mode=ExecMode.sequential), hasher=IdentityHasher())
    assert t.num_vertices() == 4
    assert t.offsets().tolist() == [0, 0, 4, 4, 4]
    seg = t.vertex_entries(1)
    assert [(int(e["key"]), int(e["index"])) for e in seg] == [(5, 0), (1, 1), (5, 2), (9, 3)]
    for v in (0, 2, 3):
        assert len(t.vertex_entries(v)) == 0
    with pytest.raises(IndexError):
        t.vertex_entries(4)


def test_collision_fixture():
    # test_core.cpp:64-88
    t = hg.build_v1([3, 9, 3, 10121, 7], BuildConfig(mode=ExecMode.sequential), vertex_count=5059,
                    hasher=IdentityHasher())
    lens = np.diff(t.offsets())
    assert (lens == 3).sum() == 1 and lens.max() == 3
    assert [(int(e["key"]), int(e["index"])) for e in t.vertex_entries(3)] == \
        [(3, 0), (3, 2), (10121, 3)]
    assert hg.count_instances(t, 3) == 2
    assert hg.count_instances(t, 10121) == 1
    assert hg.count_instances(t, 5059 + 3) == 0


@pytest.mark.parametrize("variant", [1, 2])
def test_empty_input(variant):
    # test_core.cpp:90-100
    t = BUILDS[variant]([], BuildConfig(mode=ExecMode.sequential))
    assert t.num_vertices() == 1 and t.num_edges() == 0
    assert t.offsets().tolist() == [0, 0]
    assert hg.validate_csr(t, 0) is None
    assert hg.count_instances(t, 42) == 0
    assert hg.probe_standard(t, [1, 2, 3]).match_count == 0


@pytest.mark.parametrize("variant", [1, 2])
def test_duplicates_count_instances(variant):
    # test_core.cpp:102-109
    t = BUILDS[variant]([7, 7, 7, 2], BuildConfig(mode=ExecMode.sequential))
    assert hg.count_instances(t, 7) == 3
    assert hg.count_instances(t, 2) == 1
    assert hg.count_instances(t, 999) == 0


def test_config_errors():
    # test_core.cpp:291-299
    with pytest.raises(ValueError):
        hg.build_v1([1, 2, 3], BuildConfig(load_factor=0.0))
    with pytest.raises(ValueError):
        hg.build_v2([1, 2, 3], BuildConfig(bin_count=0))


def test_build_stats_exact_counts():
    # test_core.cpp:206-236
    keys = np.arange(3000, dtype=np.uint64) % 100
    s1 = hg.BuildStats()
    hg.build_v1(keys, BuildConfig(mode=ExecMode.sequential), stats=s1)
    assert (s1.hash_evals, s1.count_increments, s1.placement_writes) == (6000, 3000, 3000)
    assert s1.counter_zero_writes == 3000 and s1.bin_count_increments == 0
    s2 = hg.BuildStats()
    hg.build_v2(keys, BuildConfig(mode=ExecMode.sequential, bin_count=64), stats=s2)
    assert s2.hash_evals == 12000 and s2.bin_placement_writes == 3000
    assert s2.counter_zero_writes == 64 + 3000


@pytest.mark.parametrize("width", [4, 8])
@pytest.mark.parametrize("variant", [1, 2])
def test_config1_known_answers(oracle, width, variant):
    c1 = GOLDEN["config1"]
    n = c1["n"]
    keys = oracle.mt19937_64(1, n, mask_u32=True)
    probe = oracle.mt19937_64(1, n, skip=n, mask_u32=True)
    dt = np.uint32 if width == 4 else np.uint64
    t = BUILDS[variant](keys.astype(dt), BuildConfig(mode=ExecMode.sequential))
    assert hex(oracle.fold(t.offsets())) == c1["offsets_fold"]
    inter = np.stack([t.edge_keys(), t.edge_index()], 1).ravel()
    assert hex(oracle.fold(inter)) == c1["edges_fold"]
    for pk, name in ((keys, "self_probe"), (probe, "indep_probe")):
        r = hg.probe_standard(t, pk.astype(dt))
        assert r.match_count == c1[name]["match_count"]
        assert r.key_comparisons == c1[name]["key_comparisons"]
    # parallel mode: same offsets, same canonical segments
    tp = BUILDS[variant](keys.astype(dt))
    assert (tp.offsets() == t.offsets()).all()
    a = canon(tp.offsets(), tp.edge_keys(), tp.edge_index())
    b = canon(t.offsets(), t.edge_keys(), t.edge_index())
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()


RANDOM_CASES = [
    # n, key_range, load, seed, width, variant, aggregate, bins
    (5000, 1200, 0.5, 0, 8, 2, -1, 1 << 15),
    (20000, 5000, 1.0, 0, 4, 1, 1, 1 << 15),
    (20000, 5000, 1.0, 0, 4, 1, 0, 1 << 15),
    (3000, 700, 0.25, 17, 8, 1, -1, 256),
    (3000, 700, 4.0, 17, 8, 2, -1, 1),
    (65536, 1 << 32, 1.5, 99, 4, 2, -1, 1 << 15),
    (65536, 1 << 62, 1.0, 5, 8, 1, -1, 1 << 15),
    (100000, 97, 1.0, 0, 4, 2, -1, 1 << 15),   # heavy duplication
    (100000, 97, 1.0, 0, 8, 1, 0, 1 << 15),    # heavy duplication, no aggregation
    (40000, 1, 1.0, 0, 4, 2, -1, 1 << 15),     # one key
    (1 << 18, 1 << 32, 2.0, 3, 4, 2, -1, 1 << 15),
]


@pytest.mark.parametrize("n,kr,load,seed,width,variant,agg,bins", RANDOM_CASES)
def test_random_vs_oracle(oracle, n, kr, load, seed, width, variant, agg, bins):
    rng = np.random.default_rng(n + seed + width)
    keys = (rng.integers(0, kr, size=n, dtype=np.uint64) if kr < (1 << 63)
            else rng.integers(0, 1 << 63, size=n, dtype=np.uint64))
    if width == 4:
        keys &= np.uint64(0xFFFFFFFF)
    dt = np.uint32 if width == 4 else np.uint64
    o = oracle.build(keys, variant, load, bins, seed)
    for mode in (ExecMode.parallel, ExecMode.sequential):
        cfg = BuildConfig(load_factor=load, bin_count=bins, hash_seed=seed, mode=mode,
                          aggregate=agg)
        t = BUILDS[variant](keys.astype(dt), cfg)
        assert_same_table(t, o, exact=mode == ExecMode.sequential)
        assert hg.validate_csr(t, n, keys.astype(dt)) is None
    # keep the pair count bounded for heavily duplicated inputs
    npb = min(n // 3, max(64, 4_000_000 // max(1, n // max(kr, 1))))
    probes = np.concatenate([keys[:npb], rng.integers(0, max(kr, 2), size=npb,
                                                      dtype=np.uint64)])
    if width == 4:
        probes &= np.uint64(0xFFFFFFFF)
    ro = oracle.probe_standard(o, probes, materialize=True, cap=1 << 26, per_probe=True)
    exp = ro["pairs"][np.lexsort((ro["pairs"][:, 0], ro["pairs"][:, 1]))]
    for method in (1, 2):  # direct gathers, vertex-range partitioned
        r = hg.probe_standard(t, probes.astype(dt), ProbeOptions(materialize=True, pair_cap=1 << 26),
                              method=method)
        assert r.match_count == ro["match_count"]
        assert r.key_comparisons == ro["key_comparisons"]
        assert not r.truncated
        got = np.stack([r.pairs["left_index"], r.pairs["right_index"]], 1)
        got = got[np.lexsort((got[:, 0], got[:, 1]))]
        assert (got == exp).all()
        # per-probe counts == count_instances per key (count-only and with pairs)
        counts = np.zeros(len(probes), np.uint32)
        r2 = hg.probe_standard(t, probes.astype(dt), counts=counts, method=method)
        assert r2.match_count == ro["match_count"] and r2.key_comparisons == ro["key_comparisons"]
        assert (counts.astype(np.uint64) == ro["per_probe"]).all()
        counts[:] = 0
        hg.probe_standard(t, probes.astype(dt), ProbeOptions(materialize=True, pair_cap=1 << 26),
                          counts=counts, method=method)
        assert (counts.astype(np.uint64) == ro["per_probe"]).all()
        r3 = hg.probe_standard(t, probes.astype(dt), method=method)
        assert (r3.match_count, r3.key_comparisons) == (ro["match_count"], ro["key_comparisons"])


def test_probe_cap_truncation():
    # test_join.cpp:224-243
    a = np.full(64, 5, np.uint64)
    t = hg.build_v2(a)
    r = hg.probe_standard(t, a, ProbeOptions(materialize=True, pair_cap=100))
    assert r.match_count == 4096 and r.truncated and len(r.pairs) == 100
    assert (r.pairs["left_index"] < 64).all() and (r.pairs["right_index"] < 64).all()
    r = hg.probe_standard(t, a, ProbeOptions(materialize=True, pair_cap=4096))
    assert not r.truncated and len(r.pairs) == 4096
    assert len(set(zip(r.pairs["left_index"].tolist(), r.pairs["right_index"].tolist()))) == 4096


def test_probe_counts_duplicates():
    # test_join.cpp:85-116
    t = hg.build_v2([7, 7, 2])
    r = hg.probe_standard(t, [7, 3, 7])
    assert r.match_count == 4 and r.pairs is None and not r.truncated
    r = hg.probe_standard(t, [7, 3, 7], ProbeOptions(materialize=True))
    got = sorted(zip(r.pairs["left_index"].tolist(), r.pairs["right_index"].tolist()))
    assert got == [(0, 0), (0, 2), (1, 0), (1, 2)]


def test_probe_degenerate_single_vertex():
    # test_join.cpp:245-259 (V == 1: every key collides; full-key compares decide)
    a = [3, 9, 3, 10121, 7]
    b = [3, 10121, 11]
    t = hg.build_v2(a, BuildConfig(load_factor=float(len(a))), hasher=IdentityHasher())
    assert t.num_vertices() == 1
    r = hg.probe_standard(t, b, ProbeOptions(materialize=True))
    assert r.match_count == 3 and r.key_comparisons == len(a) * len(b)
    got = sorted(zip(r.pairs["left_index"].tolist(), r.pairs["right_index"].tolist()))
    assert got == [(0, 0), (2, 0), (3, 1)]


def test_long_segments_warp_cooperative(oracle):
    # heavy keys -> segments far beyond the per-thread walk limit
    rng = np.random.default_rng(5)
    keys = np.concatenate([np.full(5000, 11, np.uint64), np.full(300, 12, np.uint64),
                           rng.integers(0, 1 << 40, size=20000, dtype=np.uint64)])
    rng.shuffle(keys)
    o = oracle.build(keys, 1, 1.0, 1, 0)
    for variant in (1, 2):
        t = BUILDS[variant](keys, BuildConfig(mode=ExecMode.sequential))
        assert_same_table(t, o, exact=True)
    probes = np.array([11, 12, 13] * 50 + [11] * 3, np.uint64)
    ro = oracle.probe_standard(o, probes, materialize=True, cap=1 << 24)
    exp = ro["pairs"][np.lexsort((ro["pairs"][:, 0], ro["pairs"][:, 1]))]
    for method in (1, 2):
        r = hg.probe_standard(t, probes, ProbeOptions(materialize=True, pair_cap=1 << 24),
                              method=method)
        assert r.match_count == ro["match_count"] and r.key_comparisons == ro["key_comparisons"]
        got = np.stack([r.pairs["left_index"], r.pairs["right_index"]], 1)
        got = got[np.lexsort((got[:, 0], got[:, 1]))]
        assert (got == exp).all()


def test_device_tensors_in_place(oracle, cuda):
    torch = cuda
    n = 1 << 16
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    host = oracle.splitmix(1, n, mask_u32=True)
    assert (keys.cpu().numpy().view(np.uint32).astype(np.uint64) == host).all()
    t = hg.build_v2(keys)
    o = oracle.build(host, 2)
    assert_same_table(t, o, exact=False)
    counts = torch.zeros(n, dtype=torch.int32, device="cuda")
    r = hg.probe_standard(t, keys, counts=counts)
    ro = oracle.probe_standard(o, host, per_probe=True)
    assert r.match_count == ro["match_count"]
    assert (counts.cpu().numpy().view(np.uint32).astype(np.uint64) == ro["per_probe"]).all()


@pytest.mark.parametrize("log2n,width,load", [(22, 4, 1.0), (24, 4, 1.0), (23, 8, 0.5),
                                              (23, 4, 4.0), (22, 8, 1.5)])
def test_large_scale_vs_oracle(oracle, cuda, log2n, width, load):
    """Sizes where the partitioned (multi-pass) paths are the ones that run."""
    torch = cuda
    n = 1 << log2n
    dt = torch.int32 if width == 4 else torch.int64
    keys = torch.empty(n, dtype=dt, device="cuda")
    probes = torch.empty(n, dtype=dt, device="cuda")
    hg.generate(keys, kind=0, seed=11)
    hg.generate(probes, kind=0, seed=12)
    hk = keys.cpu().numpy().view(np.uint32 if width == 4 else np.uint64).astype(np.uint64)
    hp = probes.cpu().numpy().view(np.uint32 if width == 4 else np.uint64).astype(np.uint64)
    o = oracle.build(hk, 1, load)
    for variant in (1, 2):
        t = BUILDS[variant](keys, BuildConfig(load_factor=load))
        assert_same_table(t, o, exact=False)
        assert hg.validate_csr(t, n, keys) is None
    half = np.concatenate([hk[: n // 2], hp[: n // 2]])
    ro = oracle.probe_standard(o, half)
    dhalf = torch.cat([keys[: n // 2], probes[: n // 2]])
    for method in (1, 2):
        r = hg.probe_standard(t, dhalf, method=method)
        assert (r.match_count, r.key_comparisons) == (ro["match_count"], ro["key_comparisons"])
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    hg.probe_device(t, dhalf, res, method=2)
    assert [int(x) for x in res.cpu()] == [ro["match_count"], ro["key_comparisons"]]


@pytest.mark.parametrize("G,load,variant", [(4, 1.0, 2), (3, 1.5, 1), (8, 0.5, 2)])
def test_shard_route_and_local_builds(oracle, cuda, G, load, variant):
    """Single-GPU run of the sharded path's device kernels: hg_route groups
    keys by owner shard, every shard builds its vertex range with the global
    hash (vertex_base), and the concatenated shards equal the oracle table;
    routed probes summed over shards equal the oracle's totals."""
    torch = cuda
    from paper_1907_02900_b200.sharded import CudaEngine, shard_range
    n = 200_000
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    hg.generate(keys, kind=0, seed=21)
    hk = keys.cpu().numpy().view(np.uint32).astype(np.uint64)
    V = hg.derived_vertex_count(n, load)
    ref = oracle.build(hk, 1, load)
    eng = CudaEngine(variant)
    sk, sv, counts = eng.route(keys, None, 4, 1000, 0, 0, V, G)
    counts = counts.cpu().tolist()
    assert sum(counts) == n
    offs_all, k_all, v_all = [np.zeros(1, np.uint64)], [], []
    start = 0
    edge_base = 0
    for g in range(G):
        base, cnt = shard_range(V, G, g)
        kk, vv = sk[start:start + counts[g]], sv[start:start + counts[g]]
        start += counts[g]
        t = eng.build(kk, vv, V, base, max(cnt, 1), BuildConfig(load_factor=load,
                                                             mode=ExecMode.sequential), 0)
        assert t.num_vertices() == max(cnt, 1)
        offs_all.append(t.offsets()[1:] + edge_base)
        edge_base += t.num_edges()
        k_all.append(t.edge_keys())
        v_all.append(t.edge_index())
    offs = np.concatenate(offs_all)
    assert (offs == ref.offsets).all()
    # values carry global positions (val_base = 1000); sequential -> exact order
    assert (np.concatenate(k_all) == ref.keys).all()
    assert (np.concatenate(v_all) == ref.index + 1000).all()
    # probes: route, probe each shard, sum
    probes = torch.cat([keys[: n // 2], keys[: n // 4] ^ 0x5A5A5A5A])
    hp = probes.cpu().numpy().view(np.uint32).astype(np.uint64)
    pk, pv, pc = eng.route(probes, None, 4, 0, 0, 0, V, G)
    pc = pc.cpu().tolist()
    tot = np.zeros(2, np.int64)
    start = 0
    for g in range(G):
        base, cnt = shard_range(V, G, g)
        kk, vv = sk[sum(counts[:g]):sum(counts[:g + 1])], sv[sum(counts[:g]):sum(counts[:g + 1])]
        t = eng.build(kk, vv, V, base, max(cnt, 1), BuildConfig(load_factor=load), 0)
        tot += eng.probe_totals(t, pk[start:start + pc[g]]).cpu().numpy()
        start += pc[g]
    ro = oracle.probe_standard(ref, hp)
    assert tot.tolist() == [ro["match_count"], ro["key_comparisons"]]
