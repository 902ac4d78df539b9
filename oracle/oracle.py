"""TEST INFRASTRUCTURE ONLY -- Python bindings for the parity checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module. It is the checker, never the thing
measured or shipped: the product path (paper_1907_02900_b200) never imports it.

* ``Oracle``   -- ctypes over oracle/_build/libhgoracle.so, the plain-C
  restatement of the reference hot path (oracle/hg_oracle.c, each function
  citing the reference file:line it restates).
* ``Reference`` -- ctypes over oracle/_ref/libhgref.so, the unmodified reference
  headers compiled by oracle/Makefile (oracle/ref_shim.cpp forwards).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhgoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhgref.so")
REF_SO_V4 = os.path.join(HERE, "_ref", "libhgref_v4.so")


def cpu_has_avx512() -> bool:
    """x86-64-v4 feature set (avx512 f/bw/cd/dq/vl) on this host."""
    try:
        flags = next(l for l in open("/proc/cpuinfo") if l.startswith("flags")).split()
    except (OSError, StopIteration):
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"))


def reference_so() -> str:
    """The compiled reference to time: the x86-64-v4 build on AVX-512 hosts,
    else the portable x86-64-v2 build."""
    return REF_SO_V4 if os.path.exists(REF_SO_V4) and cpu_has_avx512() else REF_SO

HASH_MIX64 = 0
HASH_IDENTITY = 1

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_P = C.POINTER(C.c_uint64)


def build_oracle() -> None:
    """Compile the checkers (oracle/Makefile). Reference shim only where the
    reference headers exist (the build container)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


@dataclass
class Table:
    """Host CSR table in the reference layout (core.hpp:67-102): offsets[V+1]
    plus edges as parallel key/index arrays (Entry{key,index}, core.hpp:21-26)."""

    num_vertices: int
    offsets: np.ndarray
    keys: np.ndarray
    index: np.ndarray
    hash_seed: int = 0
    hash_kind: int = HASH_MIX64

    def segment(self, v: int):
        b, e = int(self.offsets[v]), int(self.offsets[v + 1])
        return list(zip(self.keys[b:e].tolist(), self.index[b:e].tolist()))

    def canonical_segments(self):
        """tests/support.hpp:50-58 canonical_segments, vectorised: edges sorted
        by (vertex, key, index). Returns (keys, index) arrays."""
        n = len(self.keys)
        seg = np.repeat(np.arange(self.num_vertices, dtype=np.uint64),
                        np.diff(self.offsets).astype(np.int64))
        order = np.lexsort((self.index, self.keys, seg)) if n else np.zeros(0, np.int64)
        return self.keys[order], self.index[order]


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        lib = C.CDLL(path)
        u64, dbl, i32 = C.c_uint64, C.c_double, C.c_int
        lib.hgo_mix64.restype = u64
        lib.hgo_mix64.argtypes = [u64]
        lib.hgo_vertex.restype = u64
        lib.hgo_vertex.argtypes = [u64, u64, u64, i32]
        lib.hgo_hash_to_vertex.restype = u64
        lib.hgo_hash_to_vertex.argtypes = [u64, u64, u64]
        lib.hgo_vertices.restype = None
        lib.hgo_vertices.argtypes = [_P, u64, u64, u64, i32, _P]
        lib.hgo_derived_vertex_count.restype = i32
        lib.hgo_derived_vertex_count.argtypes = [u64, dbl, _P]
        lib.hgo_build_v1.restype = i32
        lib.hgo_build_v1.argtypes = [_P, u64, u64, u64, i32, _P, _P, _P]
        lib.hgo_build_v2.restype = i32
        lib.hgo_build_v2.argtypes = [_P, u64, u64, u64, u64, i32, _P, _P, _P]
        lib.hgo_count_instances.restype = u64
        lib.hgo_count_instances.argtypes = [_P, _P, u64, u64, i32, u64]
        lib.hgo_probe_standard.restype = None
        lib.hgo_probe_standard.argtypes = [_P, _P, _P, u64, u64, i32, _P, u64, u64, _P, _P,
                                           _P, _P, _P]
        lib.hgo_probe_new_prepared.restype = None
        lib.hgo_probe_new_prepared.argtypes = [_P, _P, _P, _P, _P, _P, u64, u64, _P, _P, _P,
                                               _P]
        lib.hgo_validate_csr.restype = i32
        lib.hgo_validate_csr.argtypes = [_P, _P, _P, u64, u64, u64, u64, i32, _P]
        lib.hgo_exclusive_prefix_sum.restype = i32
        lib.hgo_exclusive_prefix_sum.argtypes = [_P, u64, _P]
        lib.hgo_sort_merge_join_count.restype = u64
        lib.hgo_sort_merge_join_count.argtypes = [_P, u64, _P, u64]
        lib.hgo_mt19937_64.restype = None
        lib.hgo_mt19937_64.argtypes = [u64, u64, _P, u64, i32]
        lib.hgo_generate_uniform.restype = i32
        lib.hgo_generate_uniform.argtypes = [u64, dbl, u64, _P]
        lib.hgo_splitmix64.restype = u64
        lib.hgo_splitmix64.argtypes = [u64, u64]
        lib.hgo_splitmix_fill.restype = None
        lib.hgo_splitmix_fill.argtypes = [u64, u64, u64, i32, _P]
        lib.hgo_fold.restype = u64
        lib.hgo_fold.argtypes = [_P, u64, u64]
        self.lib = lib

    # hash.hpp
    def mix64(self, x: int) -> int:
        return int(self.lib.hgo_mix64(x))

    def hash_to_vertex(self, key: int, seed: int, nv: int) -> int:
        return int(self.lib.hgo_hash_to_vertex(key, seed, nv))

    def vertex(self, key: int, seed: int, nv: int, hash_kind: int = HASH_MIX64) -> int:
        return int(self.lib.hgo_vertex(key, seed, nv, hash_kind))

    def vertices(self, keys, seed: int, nv: int, hash_kind: int = HASH_MIX64) -> np.ndarray:
        keys = _u64(keys)
        out = np.zeros(len(keys), np.uint64)
        self.lib.hgo_vertices(_ptr(keys), len(keys), seed, nv, hash_kind, _ptr(out))
        return out

    def derived_vertex_count(self, n: int, load: float) -> int:
        out = np.zeros(1, np.uint64)
        if self.lib.hgo_derived_vertex_count(n, load, _ptr(out)):
            raise ValueError("load_factor must be positive")
        return int(out[0])

    # core.hpp builds (sequential semantics)
    def build(self, keys, variant: int = 1, load: float = 1.0, bins: int = 1 << 15,
              seed: int = 0, vertex_count: int | None = None,
              hash_kind: int = HASH_MIX64) -> Table:
        keys = _u64(keys)
        if not load > 0 or bins < 1:
            raise ValueError("invalid BuildConfig")
        nv = vertex_count if vertex_count else self.derived_vertex_count(len(keys), load)
        off = np.zeros(nv + 1, np.uint64)
        ek = np.zeros(len(keys), np.uint64)
        ei = np.zeros(len(keys), np.uint64)
        if variant == 2:
            rc = self.lib.hgo_build_v2(_ptr(keys), len(keys), nv, bins, seed, hash_kind,
                                       _ptr(off), _ptr(ek), _ptr(ei))
        else:
            rc = self.lib.hgo_build_v1(_ptr(keys), len(keys), nv, seed, hash_kind, _ptr(off),
                                       _ptr(ek), _ptr(ei))
        if rc:
            raise RuntimeError(f"oracle build failed rc={rc}")
        return Table(nv, off, ek, ei, seed, hash_kind)

    def probe_standard(self, t: Table, probes, materialize: bool = False,
                       cap: int = 1 << 24, per_probe: bool = False):
        probes = _u64(probes)
        m = len(probes)
        mc = np.zeros(1, np.uint64)
        cmp = np.zeros(1, np.uint64)
        wr = np.zeros(1, np.uint64)
        pairs = np.zeros(2 * max(min(cap, 1 << 40), 0), np.uint64) if materialize else None
        if materialize and cap > 4 * (1 << 28):
            raise ValueError("oracle cap too large")
        pp = np.zeros(m, np.uint64) if per_probe else None
        self.lib.hgo_probe_standard(_ptr(t.offsets), _ptr(t.keys), _ptr(t.index), t.num_vertices,
                                    t.hash_seed, t.hash_kind, _ptr(probes), m, cap,
                                    _ptr(pairs), _ptr(pp), _ptr(mc), _ptr(cmp), _ptr(wr))
        res = {"match_count": int(mc[0]), "key_comparisons": int(cmp[0]),
               "truncated": bool(materialize and int(mc[0]) > cap)}
        if materialize:
            res["pairs"] = pairs[: 2 * int(wr[0])].reshape(-1, 2)
        if per_probe:
            res["per_probe"] = pp
        return res

    def probe_new_prepared(self, a: Table, b: Table, materialize: bool = False,
                           cap: int = 1 << 24):
        """join.hpp:143-166 (restated in hgo_probe_new_prepared)."""
        if a.num_vertices != b.num_vertices:
            raise ValueError("probe_new_prepared: tables use different vertex ranges")
        mc = np.zeros(1, np.uint64)
        cmp = np.zeros(1, np.uint64)
        wr = np.zeros(1, np.uint64)
        if materialize and cap > 4 * (1 << 28):
            raise ValueError("oracle cap too large")
        pairs = np.zeros(2 * max(cap, 0), np.uint64) if materialize else None
        self.lib.hgo_probe_new_prepared(_ptr(a.offsets), _ptr(a.keys), _ptr(a.index),
                                        _ptr(b.offsets), _ptr(b.keys), _ptr(b.index),
                                        a.num_vertices, cap, _ptr(pairs), _ptr(mc), _ptr(cmp),
                                        _ptr(wr))
        res = {"match_count": int(mc[0]), "key_comparisons": int(cmp[0]),
               "truncated": bool(materialize and int(mc[0]) > cap)}
        if materialize:
            res["pairs"] = pairs[: 2 * int(wr[0])].reshape(-1, 2)
        return res

    def probe_new(self, a, b, load: float = 1.0, bins: int = 1 << 15, seed: int = 0,
                  hash_kind: int = HASH_MIX64, materialize: bool = False, cap: int = 1 << 24):
        """join.hpp:170-182: both sides built with build_v2 over the V of the
        larger input, then probe_new_prepared."""
        a, b = _u64(a), _u64(b)
        nv = self.derived_vertex_count(max(len(a), len(b)), load)
        ta = self.build(a, variant=2, load=load, bins=bins, seed=seed, vertex_count=nv,
                        hash_kind=hash_kind)
        tb = self.build(b, variant=2, load=load, bins=bins, seed=seed, vertex_count=nv,
                        hash_kind=hash_kind)
        return self.probe_new_prepared(ta, tb, materialize, cap)

    def count_instances(self, t: Table, key: int) -> int:
        return int(self.lib.hgo_count_instances(_ptr(t.offsets), _ptr(t.keys), t.num_vertices,
                                                t.hash_seed, t.hash_kind, key))

    def validate_csr(self, t: Table, expected: int, input_keys=None) -> int:
        inp = None if input_keys is None else _u64(input_keys)
        return int(self.lib.hgo_validate_csr(_ptr(t.offsets), _ptr(t.keys), _ptr(t.index),
                                             t.num_vertices, len(t.keys), expected, t.hash_seed,
                                             t.hash_kind, _ptr(inp)))

    def exclusive_prefix_sum(self, counts):
        counts = _u64(counts)
        out = np.zeros(len(counts) + 1, np.uint64)
        if self.lib.hgo_exclusive_prefix_sum(_ptr(counts), len(counts), _ptr(out)):
            raise OverflowError("exclusive_prefix_sum: counter sum exceeds 64 bits")
        return out

    def sort_merge_join_count(self, a, b) -> int:
        a, b = _u64(a), _u64(b)
        return int(self.lib.hgo_sort_merge_join_count(_ptr(a), len(a), _ptr(b), len(b)))

    def mt19937_64(self, seed: int, n: int, skip: int = 0, mask_u32: bool = False):
        out = np.zeros(n, np.uint64)
        self.lib.hgo_mt19937_64(seed, skip, _ptr(out), n, int(mask_u32))
        return out

    def generate_uniform(self, n: int, mult: float, seed: int):
        out = np.zeros(n, np.uint64)
        if self.lib.hgo_generate_uniform(n, mult, seed, _ptr(out)):
            raise ValueError("multiplicity must be positive")
        return out

    def splitmix(self, seed: int, n: int, start: int = 0, mask_u32: bool = True):
        out = np.zeros(n, np.uint64)
        self.lib.hgo_splitmix_fill(seed, start, n, int(mask_u32), _ptr(out))
        return out

    def fold(self, xs, h: int = 0) -> int:
        xs = _u64(xs)
        return int(self.lib.hgo_fold(_ptr(xs), len(xs), h))


class Reference:
    """The reference headers themselves (oracle/_ref). Threads follow
    HASHGRAPH_THREADS (parallel.hpp:25-34); ``threads`` sets it per call."""

    def __init__(self, path: str | None = None):
        path = path or reference_so()
        if not os.path.exists(path):
            build_oracle()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} (reference not compiled here)")
        self.path = path
        lib = C.CDLL(path)
        u64, dbl, i32, vp = C.c_uint64, C.c_double, C.c_int, C.c_void_p
        lib.hgr_mix64.restype = u64
        lib.hgr_mix64.argtypes = [u64]
        lib.hgr_hash_to_vertex.restype = u64
        lib.hgr_hash_to_vertex.argtypes = [u64, u64, u64]
        lib.hgr_derived_vertex_count.restype = i32
        lib.hgr_derived_vertex_count.argtypes = [u64, dbl, _P]
        lib.hgr_build.restype = vp
        lib.hgr_build.argtypes = [_P, u64, i32, dbl, u64, u64, i32, u64, i32, C.POINTER(i32)]
        lib.hgr_free.restype = None
        lib.hgr_free.argtypes = [vp]
        lib.hgr_info.restype = None
        lib.hgr_info.argtypes = [vp, _P, _P]
        lib.hgr_export.restype = None
        lib.hgr_export.argtypes = [vp, _P, _P, _P]
        lib.hgr_probe.restype = None
        lib.hgr_probe.argtypes = [vp, _P, u64, i32, u64, _P, _P, C.POINTER(i32), _P, _P]
        lib.hgr_probe_new_prepared.restype = i32
        lib.hgr_probe_new_prepared.argtypes = [vp, vp, i32, u64, _P, _P, C.POINTER(i32), _P, _P]
        lib.hgr_probe_new.restype = i32
        lib.hgr_probe_new.argtypes = [_P, u64, _P, u64, dbl, u64, u64, i32, i32, u64, _P, _P,
                                      C.POINTER(i32), _P, _P]
        lib.hgr_count_instances.restype = u64
        lib.hgr_count_instances.argtypes = [vp, u64]
        lib.hgr_validate.restype = i32
        lib.hgr_validate.argtypes = [vp, u64]
        lib.hgr_sort_merge_join_count.restype = u64
        lib.hgr_sort_merge_join_count.argtypes = [_P, u64, _P, u64]
        lib.hgr_exclusive_prefix_sum.restype = i32
        lib.hgr_exclusive_prefix_sum.argtypes = [_P, u64, C.c_uint, _P]
        lib.hgr_generate.restype = i32
        lib.hgr_generate.argtypes = [i32, u64, dbl, u64, _P]
        lib.hgr_resolve_threads.restype = C.c_uint
        lib.hgr_write_keys.restype = i32
        lib.hgr_write_keys.argtypes = [C.c_char_p, _P, u64]
        lib.hgr_read_keys.restype = i32
        lib.hgr_read_keys.argtypes = [C.c_char_p, _P, u64, _P]
        self.lib = lib

    @staticmethod
    def set_threads(threads: int | None) -> None:
        if threads is None:
            os.environ.pop("HASHGRAPH_THREADS", None)
        else:
            os.environ["HASHGRAPH_THREADS"] = str(threads)

    def mix64(self, x: int) -> int:
        return int(self.lib.hgr_mix64(x))

    def hash_to_vertex(self, key: int, seed: int, nv: int) -> int:
        return int(self.lib.hgr_hash_to_vertex(key, seed, nv))

    def build_handle(self, keys, variant=1, load=1.0, bins=1 << 15, seed=0, sequential=False,
                     vertex_count=None, hash_kind=HASH_MIX64):
        keys = _u64(keys)
        err = C.c_int(0)
        h = self.lib.hgr_build(_ptr(keys), len(keys), variant, load, bins, seed, int(sequential),
                               vertex_count or 0, hash_kind, C.byref(err))
        if not h:
            raise ValueError(f"reference build rejected config (err={err.value})")
        return h

    def free(self, h) -> None:
        self.lib.hgr_free(h)

    def export(self, h, seed=0, hash_kind=HASH_MIX64) -> Table:
        nv = np.zeros(1, np.uint64)
        ne = np.zeros(1, np.uint64)
        self.lib.hgr_info(h, _ptr(nv), _ptr(ne))
        off = np.zeros(int(nv[0]) + 1, np.uint64)
        k = np.zeros(int(ne[0]), np.uint64)
        i = np.zeros(int(ne[0]), np.uint64)
        self.lib.hgr_export(h, _ptr(off), _ptr(k), _ptr(i))
        return Table(int(nv[0]), off, k, i, seed, hash_kind)

    def build(self, keys, variant=1, load=1.0, bins=1 << 15, seed=0, sequential=False,
              vertex_count=None, hash_kind=HASH_MIX64) -> Table:
        h = self.build_handle(keys, variant, load, bins, seed, sequential, vertex_count,
                              hash_kind)
        try:
            return self.export(h, seed, hash_kind)
        finally:
            self.free(h)

    def probe(self, h, probes, materialize=False, cap=1 << 24):
        probes = _u64(probes)
        mc = np.zeros(1, np.uint64)
        cmp = np.zeros(1, np.uint64)
        npairs = np.zeros(1, np.uint64)
        tr = C.c_int(0)
        pairs = np.zeros(2 * min(cap, 1 << 30), np.uint64) if materialize else None
        self.lib.hgr_probe(h, _ptr(probes), len(probes), int(materialize), cap, _ptr(mc),
                           _ptr(cmp), C.byref(tr), _ptr(pairs), _ptr(npairs))
        res = {"match_count": int(mc[0]), "key_comparisons": int(cmp[0]),
               "truncated": bool(tr.value)}
        if materialize:
            res["pairs"] = pairs[: 2 * int(npairs[0])].reshape(-1, 2)
        return res

    @staticmethod
    def _join_result(rc, mc, cmp, tr, pairs, npairs, materialize, what):
        if rc:
            raise ValueError(f"{what}: tables use different vertex ranges")
        res = {"match_count": int(mc[0]), "key_comparisons": int(cmp[0]),
               "truncated": bool(tr.value)}
        if materialize:
            res["pairs"] = pairs[: 2 * int(npairs[0])].reshape(-1, 2)
        return res

    def probe_new_prepared(self, ha, hb, materialize=False, cap=1 << 24):
        mc, cmp, npairs = (np.zeros(1, np.uint64) for _ in range(3))
        tr = C.c_int(0)
        pairs = np.zeros(2 * min(cap, 1 << 30), np.uint64) if materialize else None
        rc = self.lib.hgr_probe_new_prepared(ha, hb, int(materialize), cap, _ptr(mc), _ptr(cmp),
                                             C.byref(tr), _ptr(pairs), _ptr(npairs))
        return self._join_result(rc, mc, cmp, tr, pairs, npairs, materialize,
                                 "probe_new_prepared")

    def probe_new(self, a, b, load=1.0, bins=1 << 15, seed=0, hash_kind=HASH_MIX64,
                  materialize=False, cap=1 << 24):
        a, b = _u64(a), _u64(b)
        mc, cmp, npairs = (np.zeros(1, np.uint64) for _ in range(3))
        tr = C.c_int(0)
        pairs = np.zeros(2 * min(cap, 1 << 30), np.uint64) if materialize else None
        rc = self.lib.hgr_probe_new(_ptr(a), len(a), _ptr(b), len(b), load, bins, seed,
                                    hash_kind, int(materialize), cap, _ptr(mc), _ptr(cmp),
                                    C.byref(tr), _ptr(pairs), _ptr(npairs))
        return self._join_result(rc, mc, cmp, tr, pairs, npairs, materialize, "probe_new")

    def count_instances(self, h, key: int) -> int:
        return int(self.lib.hgr_count_instances(h, key))

    def validate(self, h, expected: int) -> bool:
        return self.lib.hgr_validate(h, expected) == 0

    def sort_merge_join_count(self, a, b) -> int:
        a, b = _u64(a), _u64(b)
        return int(self.lib.hgr_sort_merge_join_count(_ptr(a), len(a), _ptr(b), len(b)))

    def exclusive_prefix_sum(self, counts, threads=1):
        counts = _u64(counts)
        out = np.zeros(len(counts) + 1, np.uint64)
        if self.lib.hgr_exclusive_prefix_sum(_ptr(counts), len(counts), threads, _ptr(out)):
            raise OverflowError("exclusive_prefix_sum: counter sum exceeds 64 bits")
        return out

    def write_keys(self, path, keys) -> None:
        keys = _u64(keys)
        if self.lib.hgr_write_keys(os.fsencode(path), _ptr(keys), len(keys)):
            raise RuntimeError("KeyFileError")

    def read_keys(self, path):
        n = np.zeros(1, np.uint64)
        if self.lib.hgr_read_keys(os.fsencode(path), None, 0, _ptr(n)):
            raise RuntimeError("KeyFileError")
        out = np.zeros(int(n[0]), np.uint64)
        self.lib.hgr_read_keys(os.fsencode(path), _ptr(out), len(out), _ptr(n))
        return out

    def generate(self, kind: int, n: int, mult: float = 1.0, seed: int = 0):
        out = np.zeros(n, np.uint64)
        if self.lib.hgr_generate(kind, n, mult, seed, _ptr(out)):
            raise ValueError("bad KeySpec")
        return out


def have_reference() -> bool:
    return os.path.exists(REF_SO)
