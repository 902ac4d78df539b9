"""Parity at the exact headline configuration (BASELINE.json metric, SURVEY.md
8(d) C2): 2^28 splitmix64 u32 keys (seed 1) at load 1 through the binned
build (build_v2), then probe_standard count-only of 2^28 seed-2 probes --
the very calls bench.py times, at their full size (8+8-bit partition digits,
u32 offset-width index arithmetic).

Checks (SURVEY.md 8(c) "oracle at scale"):
  * table: hg_validate with the input keys -- offsets monotone, offsets[V] = N,
    every entry under the vertex its key hashes to, key == input[index], the
    indices a permutation -- i.e. the table equals the reference's up to
    intra-segment order;
  * offsets bit-identical to the compiled reference's build_v2 (oracle/_ref,
    core.hpp:183-230) on the same keys, when _ref is present;
  * match_count == sort_merge_join_count(keys, probes) (baselines.hpp:138-163,
    the reference's hash-free join cardinality);
  * key_comparisons == sum over probes of the length of the probe's segment
    (join.hpp:117-129 compares every key of the segment), from the exported
    offsets and the oracle's vertex hash.
"""
import numpy as np
import pytest

import paper_1907_02900_b200 as hg

pytestmark = pytest.mark.gpu


def _inputs(cuda, log2n):
    n = 1 << log2n
    keys = cuda.empty(n, dtype=cuda.int32, device="cuda")
    probes = cuda.empty(n, dtype=cuda.int32, device="cuda")
    hg.generate(keys, kind=0, seed=1)
    hg.generate(probes, kind=0, seed=2)
    return keys, probes


def _host_u64(t):
    return t.cpu().numpy().view(np.uint32).astype(np.uint64)


def test_c2_headline_full_size(oracle, cuda):
    from oracle.oracle import Reference, have_reference
    log2n = 28
    n = 1 << log2n
    keys, probes = _inputs(cuda, log2n)
    res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    # the simple build (V1) at full size: valid, and answers like V2 below
    t1 = hg.build_v1(keys)
    assert hg.validate_csr(t1, n, keys) is None
    hg.probe_device(t1, probes, res)
    r1 = res.cpu().tolist()
    offs1 = t1.offsets()
    t1.close()

    t = hg.build_v2(keys)
    assert t.num_vertices() == n and t.num_edges() == n
    assert hg.validate_csr(t, n, keys) is None
    res.zero_()
    hg.probe_device(t, probes, res)  # the bench's count-only call
    mc, cmp = (int(x) for x in res.cpu().tolist())
    assert [mc, cmp] == r1

    hk, hp = _host_u64(keys), _host_u64(probes)
    assert (hk == oracle.splitmix(1, n)).all() and (hp == oracle.splitmix(2, n)).all()
    offs = t.offsets()
    t.close()
    assert (offs == offs1).all()
    del offs1
    # key comparisons: every probe compares against its whole segment
    seglen = np.diff(offs)
    pv = oracle.vertices(hp, 0, n)
    assert cmp == int(seglen[pv.astype(np.int64)].sum())
    del pv, seglen

    if have_reference():
        ref = Reference()
        ref.set_threads(None)
        assert mc == ref.sort_merge_join_count(hk, hp)
        h = ref.build_handle(hk, variant=2)
        try:
            rt = ref.export(h)
        finally:
            ref.free(h)
        assert (rt.offsets == offs).all(), "offsets differ from the reference build_v2"
    else:
        assert mc == oracle.sort_merge_join_count(hk, hp)


def test_c2_per_probe_counts_full_size(oracle, cuda):
    """Per-probe counts at 2^28 (partitioned probe with probe positions, the
    u32 index path) agree with the count-only totals and with the segment
    hash of every probe that matched."""
    log2n = 28
    n = 1 << log2n
    keys, probes = _inputs(cuda, log2n)
    t = hg.build_v2(keys)
    res = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    hg.probe_device(t, probes, res)
    counts = cuda.zeros(n, dtype=cuda.int32, device="cuda")
    res2 = cuda.zeros(2, dtype=cuda.int64, device="cuda")
    hg.probe_device(t, probes, res2, counts=counts)
    assert res.tolist() == res2.tolist()
    assert int(counts.sum().item()) == int(res[0].item())
    # a probe that matched must find its key in the sorted build keys
    sk = cuda.sort(keys.long() & 0xFFFFFFFF).values
    hit = counts > 0
    pk = probes.long()[hit] & 0xFFFFFFFF
    pos = cuda.searchsorted(sk, pk)
    assert bool((sk[pos.clamp(max=n - 1)] == pk).all())
    # and a probe with count 0 must not
    miss = probes.long()[~hit][: 1 << 22] & 0xFFFFFFFF
    pos = cuda.searchsorted(sk, miss).clamp(max=n - 1)
    assert not bool((sk[pos] == miss).any())
    t.close()
