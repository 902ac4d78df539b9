"""GPU parity for the binned build at any vertex count (core.hpp:183-230 has no
limit on V) and for the shared-memory geometry edge cases.

* Sliced V2 build: when V needs more than 2^16 partitions of the tuned width
  (V > 2^28 at load 1), the keys are routed into power-of-two vertex-range
  slices and every slice is built into its range of the one table. Forced at
  small sizes with a narrow partition width so it is checked against the
  oracle (offsets bit-identical, segment multisets / sequential edge arrays),
  including partial last slices, heavy keys (K7b with the slice's entry base)
  and shard tables (vertex_base) that are themselves sliced.
* Full size: a 2^31-key single-GPU V2 build (V = 2^31) validated with its
  input keys on the device.
* Geometry caps: probe_new with inputs of very different sizes, V2 at load
  factor 0.05 and a requested 2^16-vertex partition (the partition width is
  capped so K7's shared memory fits one CTA); per-probe counts on u64 keys
  with twice as many probes as keys (the staged caps shrink to fit).
"""
import numpy as np
import pytest

import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import BuildConfig, ExecMode, ProbeOptions

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu(cuda):
    yield


def canon(offsets, keys, index):
    nv = len(offsets) - 1
    seg = np.repeat(np.arange(nv, dtype=np.uint64), np.diff(offsets).astype(np.int64))
    order = np.lexsort((index, keys, seg))
    return keys[order], index[order]


def same_table(t, o, exact):
    assert (t.offsets() == o.offsets).all(), "offsets differ"
    if exact:
        assert (t.edge_keys() == o.keys).all() and (t.edge_index() == o.index).all()
    else:
        a = canon(t.offsets(), t.edge_keys(), t.edge_index())
        b = canon(o.offsets, o.keys, o.index)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all(), "segment multisets differ"


@pytest.mark.parametrize("width,load,pv,heavy,mode", [
    (4, 1.0, 4, False, ExecMode.parallel),      # V = 2^20, 4 slices of 2^18
    (4, 1.5, 4, False, ExecMode.sequential),    # non-power-of-two V: partial last slice
    (8, 0.25, 16, False, ExecMode.parallel),    # u64 keys, V = 2^22: 4 slices of 2^20
    (4, 1.0, 4, True, ExecMode.parallel),       # heavy keys: oversized partitions (K7b)
    (8, 2.0, 2, True, ExecMode.sequential),
])
def test_sliced_v2_vs_oracle(oracle, width, load, pv, heavy, mode):
    rng = np.random.default_rng(int(load * 100) + pv + width)
    n = 1 << 20
    keys = rng.integers(0, 1 << (8 * width - 1), size=n, dtype=np.uint64)
    if heavy:
        keys[: n // 16] = 12345
        keys[n // 16: n // 8] = rng.integers(0, 64, size=n // 16, dtype=np.uint64)
    dt = np.uint32 if width == 4 else np.uint64
    t = hg.build_v2(keys.astype(dt), BuildConfig(load_factor=load, partition_vertices=pv, mode=mode))
    o = oracle.build(keys, variant=2, load=load)
    same_table(t, o, mode == ExecMode.sequential)
    assert hg.validate_csr(t, n, keys.astype(dt)) is None
    # probes answer like the oracle's (the table is an ordinary table)
    probes = np.concatenate([keys[: n // 2], rng.integers(0, 1 << 31, size=n // 2, dtype=np.uint64)])
    r = hg.probe_standard(t, probes.astype(dt))
    ro = oracle.probe_standard(o, probes)
    assert (r.match_count, r.key_comparisons) == (ro["match_count"], ro["key_comparisons"])


@pytest.mark.parametrize("G", [3, 4])
def test_sliced_shard_builds(oracle, cuda, G):
    """Shard tables (global hash, vertex_base) whose own range is sliced: the
    concatenated shards equal the oracle's table."""
    from paper_1907_02900_b200.sharded import CudaEngine, shard_range
    n = 1 << 20
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=5)
    hk = keys.cpu().numpy().view(np.uint32).astype(np.uint64)
    V = n
    ref = oracle.build(hk, 2, 1.0)
    eng = CudaEngine(2)
    sk, sv, counts = eng.route(keys, None, 4, 0, 0, 0, V, G)
    counts = counts.cpu().tolist()
    offs_all, start, edge_base = [np.zeros(1, np.uint64)], 0, 0
    k_all, v_all = [], []
    for g in range(G):
        base, cnt = shard_range(V, G, g)
        kk, vv = sk[start:start + counts[g]], sv[start:start + counts[g]]
        start += counts[g]
        t = eng.build(kk, vv, V, base, cnt, BuildConfig(partition_vertices=2,
                                                         mode=ExecMode.sequential), 0)
        offs_all.append(t.offsets()[1:] + edge_base)
        edge_base += t.num_edges()
        k_all.append(t.edge_keys())
        v_all.append(t.edge_index())
    assert (np.concatenate(offs_all) == ref.offsets).all()
    assert (np.concatenate(k_all) == ref.keys).all()
    assert (np.concatenate(v_all) == ref.index).all()


def test_v2_two_pow_31_keys_full_size(cuda):
    """a 2^31-key V2 build on one GPU (V = 2^31, 8 slices of
    2^28 vertices), validated on the device with its input keys (offsets
    monotone, offsets[V] = N, hash consistency, key == input[index],
    permutation); the sliced probe of 2^24 probes (half of them build keys)
    equals the direct-gather probe."""
    n = 1 << 31
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    t = hg.build_v2(keys)
    assert t.num_vertices() == n and t.num_edges() == n
    assert hg.validate_csr(t, n, keys) is None
    m = 1 << 24
    probes = cuda.cat([keys[: m // 2], keys[-m // 2:] ^ 0x5A5A5A5A])
    # auto = the sliced probe (V = 2^31 is too wide for one partitioned pass):
    # probes routed into 2^28-vertex slices, each probed partitioned; against
    # the direct-gather probe (method 1), totals and per-probe counts
    res, res1 = (cuda.zeros(2, dtype=cuda.int64, device="cuda") for _ in range(2))
    counts, counts1 = (cuda.zeros(m, dtype=cuda.int32, device="cuda") for _ in range(2))
    hg.probe_device(t, probes, res, counts=counts)
    hg.probe_device(t, probes, res1, counts=counts1, method=1)
    assert res.tolist() == res1.tolist()
    assert bool((counts == counts1).all()) and bool((counts[: m // 2] >= 1).all())
    res.zero_()
    hg.probe_device(t, probes, res)  # count-only: slices get keys only
    assert res.tolist() == res1.tolist()
    t.close()


def test_probe_new_lopsided_inputs(oracle):
    """the smaller side of probe_new is built over the
    larger side's V (join.hpp:171-174), i.e. at load ~0.01."""
    rng = np.random.default_rng(7)
    a = rng.integers(0, 1 << 32, size=1 << 20, dtype=np.uint64)
    b = np.concatenate([a[:5000], rng.integers(0, 1 << 32, size=5000, dtype=np.uint64)])
    for x, y in ((a, b), (b, a)):
        r = hg.probe_new(x.astype(np.uint32), y.astype(np.uint32), BuildConfig(),
                         ProbeOptions(materialize=True))
        ro = oracle.probe_new(x, y, materialize=True, cap=1 << 24)
        assert (r.match_count, r.key_comparisons) == (ro["match_count"], ro["key_comparisons"])


@pytest.mark.parametrize("load,pv", [(0.05, 0), (1.0, 1 << 16), (0.01, 0)])
def test_v2_wide_partitions(oracle, load, pv):
    """load factor <= 1/16 or a requested 2^16-vertex
    partition used to ask K7 for more than 227 KB of shared memory."""
    rng = np.random.default_rng(11)
    n = 1 << 18
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
    for dt in (np.uint32, np.uint64):
        t = hg.build_v2(keys.astype(dt), BuildConfig(load_factor=load, partition_vertices=pv))
        same_table(t, oracle.build(keys, variant=2, load=load), False)


def test_u64_probe_counts_many_probes(oracle, cuda):
    """per-probe counts on u64 keys, 2x more probes than
    keys, table > 96 MB -> partitioned probe with probe positions; the staged
    caps shrink so the layout fits one CTA."""
    n, m = 1 << 24, 1 << 25
    keys = cuda.empty(n, dtype=cuda.int64, device="cuda")
    hg.generate(keys, kind=0, seed=3)
    probes = cuda.cat([keys, keys.flip(0) ^ 1])
    t = hg.build_v2(keys)
    res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    counts = cuda.zeros(m, dtype=cuda.int32, device="cuda")
    hg.probe_device(t, probes, res, counts=counts, method=2)
    res0 = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    hg.probe_device(t, probes, res0, method=1)  # direct path as the cross-check
    assert res.tolist() == res0.tolist()
    assert int(counts.sum().item()) == int(res[0].item())
    assert bool((counts[:n] >= 1).all())
    sub = 1 << 20
    hk = keys.cpu().numpy().view(np.uint64)
    o = oracle.build(hk, variant=2)
    hp = probes[:sub].cpu().numpy().view(np.uint64)
    c2 = cuda.zeros(sub, dtype=cuda.int32, device="cuda")
    r2 = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    hg.probe_device(t, probes[:sub], r2, counts=c2)
    ro = oracle.probe_standard(o, hp)
    assert [int(x) for x in r2.tolist()] == [ro["match_count"], ro["key_comparisons"]]


@pytest.mark.parametrize("width", [4, 8])
def test_heavy_segments_deferred(oracle, cuda, width):
    """Segments longer than kHeavySeg (8192 entries: heavy keys of a skewed
    table) are queued by the partitioned probe and walked by the whole grid
    (k_heavy_walk): totals and per-probe counts equal the oracle's, including
    a queue item per 2^15 comparisons of a 300000-entry segment."""
    rng = np.random.default_rng(width)
    n = 1 << 22
    keys = rng.integers(0, 1 << 31, size=n, dtype=np.uint64)
    keys[:300000] = 777                      # one very heavy key
    keys[300000:340000] = rng.integers(1000, 1004, size=40000, dtype=np.uint64)  # 4 x ~10000
    dt = np.uint32 if width == 4 else np.uint64
    t = hg.build_v2(keys.astype(dt))
    m = 1 << 21
    probes = rng.integers(0, 1 << 31, size=m, dtype=np.uint64)
    probes[2::7] = keys[2::7][: len(probes[2::7])]
    probes[1::101] = 1001
    probes[::97] = 777
    dp = cuda.from_numpy(probes.astype(dt).view(np.int32 if width == 4 else np.int64)).cuda()
    o = oracle.build(keys, variant=2)
    ro = oracle.probe_standard(o, probes)
    res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    hg.probe_device(t, dp, res, method=2)
    assert [int(x) for x in res.tolist()] == [ro["match_count"], ro["key_comparisons"]]
    counts = cuda.zeros(m, dtype=cuda.int32, device="cuda")
    res.zero_()
    hg.probe_device(t, dp, res, counts=counts, method=2)
    assert [int(x) for x in res.tolist()] == [ro["match_count"], ro["key_comparisons"]]
    hc = counts.cpu().numpy()
    assert hc[::97].tolist() == [300000] * len(hc[::97])
    for j in (1, 102, 2, 9, 5):
        assert int(hc[j]) == oracle.count_instances(o, int(probes[j]))


@pytest.mark.parametrize("G,V", [(4, 1 << 20), (8, 1 << 21), (2, 1 << 20), (1, 1 << 20)])
def test_route_records_split_path(cuda, G, V):
    """Power-of-two spans route with the partition machinery (one TMA-staged
    split pass); the groups equal K11's (the SoA route) as (key, position)
    multisets, counts included, and keys-only routing returns the same keys."""
    from paper_1907_02900_b200.sharded import CudaEngine
    n = (1 << 20) + 77
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=17)
    eng = CudaEngine(2)
    sk, sv, c1 = eng.route(keys, None, 4, 5000, 0, 0, V, G)           # K11 (SoA with values)
    rec, c2 = eng.route_records(keys, 4, 5000, 0, 0, V, G)            # split path
    ko, _, c3 = eng.route(keys, None, 4, 0, 0, 0, V, G, keys_only=True)  # split path, keys only
    assert c1.tolist() == c2.tolist() == c3.tolist()
    rk, rv = eng.unpack_records(rec, 4, 4)
    start = 0
    for g, c in enumerate(c1.tolist()):
        a = np.stack([sk[start:start + c].cpu().numpy(), sv[start:start + c].cpu().numpy()], 1)
        b = np.stack([rk[start:start + c].cpu().numpy(), rv[start:start + c].cpu().numpy()], 1)
        assert (a[np.lexsort(a.T[::-1])] == b[np.lexsort(b.T[::-1])]).all(), f"group {g}"
        assert (np.sort(ko[start:start + c].cpu().numpy()) == np.sort(a[:, 0])).all()
        start += c


def test_c5_two_pow_32_keys_one_gpu(cuda):
    """C5's whole table on one GPU: 2^32 u32 keys (V = 2^32, u64 offsets, 16
    slices of 2^28 vertices) validated on the device with its input keys; a
    2^26-probe count-only sliced probe equals the direct-gather probe."""
    n = 1 << 32
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    t = hg.build_v2(keys)
    assert t.num_vertices() == n and t.num_edges() == n and t.off_width == 8
    assert hg.validate_csr(t, n, keys) is None
    m = 1 << 26
    probes = cuda.cat([keys[: m // 2], keys[n // 2: n // 2 + m // 2] ^ 0x3C3C3C3C])
    res, res1 = (cuda.zeros(2, dtype=cuda.int64, device="cuda") for _ in range(2))
    hg.probe_device(t, probes, res)
    hg.probe_device(t, probes, res1, method=1)
    assert res.tolist() == res1.tolist() and int(res[0]) >= m // 2
    t.close()
