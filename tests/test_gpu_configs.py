"""GPU parity on the BASELINE.json configurations,
through the C-ABI, against the oracle at sizes it finishes in seconds, and
through size-independent invariants at the full 2^28 / 2^29 sizes.

C1  2^20 splitmix u32 keys, load 1, simple build + probe_standard
C3  u64 keys ~ Zipf(s) over K ranks (key = mix64(r ^ 0x9E37...)), u64 values =
    input position, loads 0.5 / 1 / 1.5 / 2 / 4, both builds
C4  unique scramble31 build keys, probes at hit ratio 0.1 / 0.5 / 1.0 with
    pairs (every probe < 2^31 is a build key, every other probe misses)
Full-size invariant: key == input[index] for every entry, the
indices a permutation, every entry under the vertex its key hashes to and
offsets monotone with offsets[V] = N (hg_validate) pin the table to the
reference's up to intra-segment order."""
import numpy as np
import pytest

import paper_1907_02900_b200 as hg
from paper_1907_02900_b200 import BuildConfig, ProbeOptions

pytestmark = pytest.mark.gpu

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


@pytest.fixture(autouse=True)
def _need_gpu(cuda):
    yield


def mix64_np(x):
    """hash.hpp:12-19 on numpy u64 (wrapping)."""
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xFF51AFD7ED558CCD)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xC4CEB9FE1A85EC53)
        x ^= x >> np.uint64(33)
    return x


def zipf_keys_host(oracle, n, cdf, seed, start=0):
    """SURVEY.md Appendix B (C3) restated on the host."""
    u = (oracle.splitmix(seed, n, start=start, mask_u32=False) >> np.uint64(11)).astype(
        np.float64) * (1.0 / 9007199254740992.0)
    r = np.searchsorted(cdf, u, side="left").astype(np.uint64) + np.uint64(1)
    return mix64_np(r ^ np.uint64(0x9E3779B97F4A7C15))


def canon_equal(t, o):
    assert (t.offsets() == o.offsets).all(), "offsets differ"
    nv = len(o.offsets) - 1
    seg = np.repeat(np.arange(nv, dtype=np.uint64), np.diff(o.offsets).astype(np.int64))
    a = np.lexsort((t.edge_index(), t.edge_keys(), seg))
    b = np.lexsort((o.index, o.keys, seg))
    assert (t.edge_keys()[a] == o.keys[b]).all() and (t.edge_index()[a] == o.index[b]).all()


def test_c1_config(oracle, cuda):
    n = 1 << 20
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    host = keys.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert (host == oracle.splitmix(1, n)).all()
    probes = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(probes, kind=0, seed=2)
    hp = probes.cpu().numpy().view(np.uint32).astype(np.uint64)
    o = oracle.build(host, variant=1)
    for build in (hg.build_v1, hg.build_v2):
        t = build(keys)
        canon_equal(t, o)
        for pk, hpk in ((keys, host), (probes, hp)):
            r = hg.probe_standard(t, pk)
            ro = oracle.probe_standard(o, hpk)
            assert (r.match_count, r.key_comparisons) == (ro["match_count"], ro["key_comparisons"])


@pytest.mark.parametrize("s", [1.0, 1.2])
def test_c3_zipf_generator_and_builds(oracle, cuda, s):
    n, ranks = 1 << 20, 1 << 16
    cdf = hg.zipf_cdf(ranks, s)
    dcdf = cuda.tensor(cdf, dtype=cuda.float64, device="cuda")
    keys = cuda.empty(n, dtype=cuda.int64, device="cuda")
    hg.generate(keys, kind=3, seed=5, ref=dcdf)
    host = keys.cpu().numpy().view(np.uint64)
    assert (host == zipf_keys_host(oracle, n, cdf, 5)).all(), "device Zipf generator differs"
    vals = cuda.arange(n, dtype=cuda.int64, device="cuda")
    for load in (0.5, 1.0, 1.5, 2.0, 4.0):
        o = oracle.build(host, variant=1, load=load)
        for build in (hg.build_v1, hg.build_v2):
            t = build(keys, BuildConfig(load_factor=load), vals=vals)
            assert t.key_width == 8 and t.val_width == 8
            canon_equal(t, o)
            assert hg.validate_csr(t, n, keys) is None
    # skewed probes: heavy segments on the warp-cooperative path
    t = hg.build_v2(keys, vals=vals)
    o = oracle.build(host, variant=2)
    pr = host[: 1 << 12]
    r = hg.probe_standard(t, pr)
    ro = oracle.probe_standard(o, pr)
    assert (r.match_count, r.key_comparisons) == (ro["match_count"], ro["key_comparisons"])


@pytest.mark.parametrize("h", [0.1, 0.5, 1.0])
def test_c4_join_pairs(oracle, cuda, h):
    n, m = 1 << 20, 1 << 21
    build = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(build, kind=2)
    probes = cuda.empty(m, dtype=cuda.int32, device="cuda")
    hg.generate(probes, kind=1, seed=3, hit=h, ref=build)
    hb = build.cpu().numpy().view(np.uint32).astype(np.uint64)
    hp = probes.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert len(np.unique(hb)) == n and hb.max() < (1 << 31)
    t = hg.build_v2(build)
    o = oracle.build(hb, variant=2)
    ro = oracle.probe_standard(o, hp, materialize=True, cap=1 << 23)
    assert ro["match_count"] == int((hp < (1 << 31)).sum())
    for method in (1, 2):
        r = hg.probe_standard(t, probes, ProbeOptions(materialize=True, pair_cap=1 << 23),
                              method=method)
        assert (r.match_count, r.key_comparisons) == (ro["match_count"], ro["key_comparisons"])
        got = np.stack([r.pairs["left_index"], r.pairs["right_index"]], 1)
        exp = ro["pairs"]
        assert (got[np.lexsort((got[:, 0], got[:, 1]))] == exp[np.lexsort((exp[:, 0], exp[:, 1]))]).all()


def test_c3_full_size_invariants(cuda):
    """C3 at 2^27 u64 keys (s = 1.0 over 2^24 ranks), load 1, binned build:
    the device validator proves the table equals the reference's up to
    intra-segment order."""
    n = 1 << 27
    dcdf = cuda.tensor(hg.zipf_cdf(1 << 24, 1.0), dtype=cuda.float64, device="cuda")
    keys = cuda.empty(n, dtype=cuda.int64, device="cuda")
    hg.generate(keys, kind=3, seed=7, ref=dcdf)
    vals = cuda.arange(n, dtype=cuda.int64, device="cuda")
    for build in (hg.build_v2, hg.build_v1):
        t = build(keys, vals=vals)
        assert hg.validate_csr(t, n, keys) is None
        t.close()


def test_c4_full_size_invariants(cuda):
    """C4 at full size: 2^28 unique build keys, 2^29 probes at h = 0.5, pairs
    (u32 layout on the device). Every probe < 2^31 is a build key and every
    other probe misses, so match_count = #(probe < 2^31); each pair joins equal
    keys and no probe matches twice."""
    n, m = 1 << 28, 1 << 29
    build = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(build, kind=2)
    probes = cuda.empty(m, dtype=cuda.int32, device="cuda")
    hg.generate(probes, kind=1, seed=3, hit=0.5, ref=build)
    t = hg.build_v2(build)
    expect = int((probes >= 0).sum().item())  # int32 view: value < 2^31
    res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    pairs = cuda.empty((expect + 16, 2), dtype=cuda.int32, device="cuda")
    hg.probe_device(t, probes, res, pairs=pairs, pair_width=4, pair_cap=expect + 16)
    mc = int(res[0].item())
    assert mc == expect
    p = pairs[:mc].long()
    left, right = p[:, 0], p[:, 1]
    assert bool((build[left] == probes[right]).all())
    assert int(cuda.unique(right).numel()) == mc
    # count-only agrees
    res.zero_()
    hg.probe_device(t, probes, res)
    assert int(res[0].item()) == expect


def test_pipelined_host_probes(cuda):
    """Pinned host probes (>= 2^27, count-only) take the chunked H2D / probe
    pipeline of hg_probe; the results equal the device-resident probe."""
    n, m = 1 << 24, (1 << 27) + 12345
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    probes = cuda.empty(m, dtype=cuda.int32, device="cuda")
    hg.generate(probes, kind=0, seed=2)
    # mix in hits
    probes[: n // 2] = keys[: n // 2]
    t = hg.build_v2(keys)
    res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    dcounts = cuda.zeros(m, dtype=cuda.int32, device="cuda")
    hg.probe_device(t, probes, res, counts=dcounts)
    hp = probes.cpu().pin_memory()
    hcounts = np.zeros(m, np.uint32)
    r = hg.probe_standard(t, hp, counts=hcounts)
    assert (r.match_count, r.key_comparisons) == tuple(int(x) for x in res.cpu().tolist())
    assert (hcounts == dcounts.cpu().numpy().view(np.uint32)).all()
    r2 = hg.probe_standard(t, hp)
    assert (r2.match_count, r2.key_comparisons) == (r.match_count, r.key_comparisons)


def test_key_files_device(tmp_path, cuda):
    """HGKEYS01 straight to / from device memory (pinned staging chunks), then
    a build from the loaded keys equals the build from the originals."""
    n = (1 << 25) + 3
    keys = cuda.empty(n, dtype=cuda.int64, device="cuda")
    hg.generate(keys, kind=0, seed=4)
    path = str(tmp_path / "k.keys")
    hg.write_keys(path, keys)
    back = cuda.zeros(n, dtype=cuda.int64, device="cuda")
    hg.read_keys(path, out=back)
    assert bool((back == keys).all())
    small = cuda.zeros(n, dtype=cuda.int32, device="cuda")
    keys32 = (keys & 0x7FFFFFFF).to(cuda.int32)
    hg.write_keys(path, keys32)
    hg.read_keys(path, out=small)
    assert bool((small == keys32).all())
    t1, t2 = hg.build_v2(keys32), hg.build_v2(small)
    assert (t1.offsets() == t2.offsets()).all()


@pytest.mark.parametrize("tail", [4000, 2052, 100, 4092, 1540, 1541, 4096])
def test_partial_last_partition(oracle, cuda, tail):
    """V = 1023 * 4096 + tail: the last K7 partition is partial (vectorised
    scan for some threads, scalar for others; coalesced u32 offset stores)."""
    nv = 1023 * 4096 + tail
    rng = np.random.default_rng(tail)
    keys = rng.integers(0, 1 << 32, size=nv, dtype=np.uint64)
    t = hg.build_v2(keys.astype(np.uint32), vertex_count=nv)
    o = oracle.build(keys, variant=2, vertex_count=nv)
    canon_equal(t, o)


def test_sharded_engine_over_nccl_world1(cuda, oracle):
    """The N > 1 bench path end to end on one GPU: ShardedHashGraph over a
    world-1 NCCL group (hg_route_records, count all_gather, one
    all_to_all_single, hg_build_records with vertex_base, routed probe,
    all_reduce; pairs routed back by probe position) equals the unsharded
    build and probe; export_global rebases offsets like the reference."""
    import socket
    import torch.distributed as dist
    from paper_1907_02900_b200 import sharded
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=cuda.device("cuda", 0))
    try:
        n = 1 << 22
        keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
        probes = cuda.empty(n, dtype=cuda.int32, device="cuda")
        hg.generate(keys, kind=0, seed=1)
        hg.generate(probes, kind=0, seed=2)
        eng = sharded.ShardedHashGraph(1, 0, variant=2)
        st = eng.build(keys, 0, n)
        off, k, v = eng.export_global()
        o = oracle.build(keys.cpu().numpy().view(np.uint32).astype(np.uint64), variant=2)
        assert (off == o.offsets).all()
        tot = eng.probe_count(probes, 0)
        ref = hg.probe_standard(hg.build_v2(keys), probes)
        assert tuple(int(x) for x in tot.cpu().tolist()) == (ref.match_count, ref.key_comparisons)
        # pairs: routed as records {key, position}, probed, routed back by
        # probe position (hg_route_pairs) -- equal to the unsharded pair set
        mix = cuda.cat([keys[: n // 4], probes[: n // 4]])
        left, right, ptot = eng.probe_pairs(mix, 0, mix.numel())
        rp = hg.probe_standard(hg.build_v2(keys), mix,
                               hg.ProbeOptions(materialize=True, pair_cap=1 << 24))
        assert tuple(int(x) for x in ptot.cpu().tolist()) == (rp.match_count, rp.key_comparisons)
        got = np.stack([left.cpu().numpy(), right.cpu().numpy()], 1).astype(np.uint64)
        exp = np.stack([rp.pairs["left_index"], rp.pairs["right_index"]], 1).astype(np.uint64)
        assert len(got) == rp.match_count
        assert (got[np.lexsort((got[:, 1], got[:, 0]))] == exp[np.lexsort((exp[:, 1], exp[:, 0]))]).all()
        # records in, table out: hg_route_records + hg_build_records (V1 too)
        eng1 = sharded.ShardedHashGraph(1, 0, variant=1)
        eng1.build(keys, 0, n)
        off1, _, _ = eng1.export_global()
        assert (off1 == o.offsets).all()
        res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
        eng.build_and_probe(keys, probes, res)
        assert int(res[0]) == ref.match_count
        del st
    finally:
        dist.destroy_process_group()


def test_pipelined_host_probes_stream_order(cuda):
    """pinned host probes written by earlier work on the
    caller's stream (a pending device->host copy) are copied for the probe
    only after that work -- the chunked pipeline waits on the stream unless
    the caller passes host_ready (HG_PROBE_HOST_READY)."""
    n, m = 1 << 22, (1 << 27) + 4096
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    t = hg.build_v2(keys)
    probes = cuda.empty(m, dtype=cuda.int32, device="cuda")
    hg.generate(probes, kind=0, seed=2)
    probes[: n] = keys  # n hits at least
    ref = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    hg.probe_device(t, probes, ref)
    hp = cuda.zeros(m, dtype=cuda.int32).pin_memory()  # stale contents: all zero
    s = cuda.cuda.current_stream()
    cuda.cuda._sleep(50_000_000)                        # keep the stream busy a while
    hp.copy_(probes, non_blocking=True)                 # pending D2H on the stream
    r = hg.probe_standard(t, hp)                        # must see the copied probes
    assert (r.match_count, r.key_comparisons) == tuple(int(x) for x in ref.cpu().tolist())
    s.synchronize()
