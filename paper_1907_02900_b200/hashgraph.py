"""Python mirror of the reference's hot-path API (proj/include/hashgraph).

Same names, argument meaning and error behaviour as the reference headers, so
parity tests read like the reference's own tests; every call goes through the
C-ABI (include/hg_b200.h) into the sm_100a kernels. Arrays may be numpy
arrays / Python sequences (host) or torch tensors (host or CUDA): host data is
staged by the library, CUDA tensors are used in place on the current torch
stream.

  reference (file:line)                     here
  hash.hpp:27-39 VertexHasher/hash_to_vertex hash_to_vertex, VertexHasher
  core.hpp:21-26 Entry                       ENTRY_DTYPE (structured numpy)
  core.hpp:28-35 ExecMode/BuildConfig        ExecMode, BuildConfig
  core.hpp:40-56 BuildStats                  BuildStats (exact op counts)
  core.hpp:59-63 derived_vertex_count        derived_vertex_count
  core.hpp:67-102 HashGraph                  HashGraph (device-resident)
  core.hpp:160-177 build_v1                  build_v1
  core.hpp:183-230 build_v2                  build_v2
  core.hpp:235-246 count_instances           count_instances
  core.hpp:251-287 validate_csr              validate_csr (device validator)
  join.hpp:18-35 MatchPair/ProbeOptions/JoinResult
  join.hpp:110-136 probe_standard            probe_standard
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (BUILD_BINNED, BUILD_SIMPLE, HASH_IDENTITY, HASH_MIX64, HG_EINVAL, HG_EIO,
                   HG_EOVERFLOW, HG_ERANGE, HashGraphError)

ENTRY_DTYPE = np.dtype([("key", "<u8"), ("index", "<u8")])
MATCH_PAIR_DTYPE = np.dtype([("left_index", "<u8"), ("right_index", "<u8")])


class InvalidArgument(HashGraphError, ValueError):
    """std::invalid_argument (core.hpp:106-109, join.hpp:145-147)."""


class KeyFileError(HashGraphError, RuntimeError):
    """keygen.hpp:75-77 (I/O or HGKEYS01 format problem)."""


class OutOfRange(HashGraphError, IndexError):
    """std::out_of_range (core.hpp:88-90)."""


class Overflow(HashGraphError, OverflowError):
    """std::overflow_error (parallel.hpp:153,171,178)."""


def _check(status: int) -> None:
    if status == 0:
        return
    msg = _lib.lib().hg_last_error().decode(errors="replace")
    cls = {HG_EINVAL: InvalidArgument, HG_ERANGE: OutOfRange, HG_EOVERFLOW: Overflow,
           HG_EIO: KeyFileError}.get(
        status, HashGraphError)
    raise cls(status, msg)


class ExecMode(enum.Enum):
    sequential = 0
    parallel = 1


@dataclass
class BuildConfig:
    """core.hpp:30-35 plus B200 knobs (variant is chosen by build_v1/build_v2)."""

    load_factor: float = 1.0
    bin_count: int = 1 << 15
    hash_seed: int = 0
    mode: ExecMode = ExecMode.parallel
    aggregate: int = -1
    partition_vertices: int = 0


@dataclass
class BuildStats:
    """core.hpp:40-56. Filled with the exact operation counts the reference's
    instrumented loops would record (2N / 4N hash evaluations etc.,
    test_core.cpp:206-236); the device kernels perform exactly these
    operations."""

    hash_evals: int = 0
    count_increments: int = 0
    placement_writes: int = 0
    bin_count_increments: int = 0
    bin_placement_writes: int = 0
    counter_zero_writes: int = 0

    def reset(self) -> None:
        self.__init__()


@dataclass
class ProbeOptions:
    """join.hpp:25-28."""

    materialize: bool = False
    pair_cap: int = 1 << 24


@dataclass
class JoinResult:
    """join.hpp:30-35. pairs: structured array of MatchPair (left = build
    entry index, right = probe position) when materialised."""

    match_count: int = 0
    key_comparisons: int = 0
    truncated: bool = False
    pairs: Optional[np.ndarray] = None


class VertexHasher:
    """hash.hpp:27-34 (the default hasher)."""

    kind = HASH_MIX64

    def __init__(self, seed: int = 0):
        self.seed = seed

    def __call__(self, key: int, num_vertices: int) -> int:
        return hash_to_vertex(key, self.seed, num_vertices)


class IdentityHasher:
    """tests/support.hpp:42-46: vertex = key % V (hand-traced fixtures)."""

    kind = HASH_IDENTITY

    def __call__(self, key: int, num_vertices: int) -> int:
        return key % num_vertices


def derived_vertex_count(n: int, load_factor: float) -> int:
    out = C.c_uint64(0)
    _check(_lib.lib().hg_derived_vertex_count(n, float(load_factor), C.byref(out)))
    return out.value


def hash_to_vertex(key: int, seed: int, num_vertices: int) -> int:
    return int(_lib.lib().hg_hash_to_vertex(key, seed, num_vertices))


# ------------------------------------------------------------------ arrays

def _torch():
    try:
        import torch
        return torch
    except ImportError:  # pragma: no cover
        return None


_WIDTH = {np.dtype(np.uint32): 4, np.dtype(np.int32): 4, np.dtype(np.uint64): 8,
          np.dtype(np.int64): 8}


class _Arr:
    """(pointer, length, width) view of a caller array; keeps it alive."""

    def __init__(self, x, default_dtype=np.uint64):
        torch = _torch()
        self.is_cuda = False
        if torch is not None and isinstance(x, torch.Tensor):
            if not x.is_contiguous():
                x = x.contiguous()
            w = x.element_size()
            if w not in (4, 8) or x.is_floating_point():
                raise TypeError("keys must be a 32- or 64-bit integer tensor")
            self.keep, self.ptr, self.n, self.width = x, x.data_ptr(), x.numel(), w
            self.is_cuda = x.is_cuda
            return
        a = np.asarray(x)
        if a.dtype not in _WIDTH:
            if a.size == 0 or a.dtype.kind in "iu" or a.dtype == object:
                a = np.asarray(x, dtype=default_dtype)
            else:
                raise TypeError(f"unsupported key dtype {a.dtype}")
        a = np.ascontiguousarray(a)
        self.keep, self.n, self.width = a, a.size, _WIDTH[a.dtype]
        self.ptr = a.ctypes.data if a.size else None


def _stream_for(*arrs) -> Optional[int]:
    if any(a.is_cuda for a in arrs if a is not None):
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream
    return None


# ------------------------------------------------------------------ table

class HashGraph:
    """core.hpp:67-102 -- a device-resident CSR table. offsets()/edges()
    export the reference layout (u64) on first access."""

    def __init__(self, handle: int, stream=None):
        self._h = handle
        self._stream = stream
        info = _lib.hg_table_info()
        _check(_lib.lib().hg_table_get_info(handle, C.byref(info)))
        self._info = info
        self._offsets = None
        self._keys = None
        self._vals = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().hg_table_destroy(h, self._stream)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    @property
    def handle(self) -> int:
        return self._h

    def num_vertices(self) -> int:
        return self._info.num_vertices

    def num_edges(self) -> int:
        return self._info.num_edges

    def hash_seed(self) -> int:
        return self._info.hash_seed

    def load_factor(self) -> float:
        return self._info.load_factor

    @property
    def key_width(self) -> int:
        return self._info.key_width

    @property
    def val_width(self) -> int:
        return self._info.val_width

    @property
    def off_width(self) -> int:
        return self._info.off_width

    @property
    def hash_kind(self) -> int:
        return self._info.hash_kind

    def _export(self):
        if self._offsets is None:
            nv, ne = self.num_vertices(), self.num_edges()
            off = np.zeros(nv + 1, np.uint64)
            k = np.zeros(ne, np.uint64)
            v = np.zeros(ne, np.uint64)
            _check(_lib.lib().hg_table_export(self._h, off.ctypes.data,
                                              k.ctypes.data if ne else None,
                                              v.ctypes.data if ne else None, self._stream))
            self._offsets, self._keys, self._vals = off, k, v

    def offsets(self) -> np.ndarray:
        self._export()
        return self._offsets

    def edge_keys(self) -> np.ndarray:
        self._export()
        return self._keys

    def edge_index(self) -> np.ndarray:
        self._export()
        return self._vals

    def edges(self) -> np.ndarray:
        """Structured array of Entry{key, index} (core.hpp:21-26)."""
        self._export()
        e = np.zeros(self.num_edges(), ENTRY_DTYPE)
        e["key"], e["index"] = self._keys, self._vals
        return e

    def vertex_entries(self, v: int) -> np.ndarray:
        """core.hpp:87-94; OutOfRange (IndexError) for v >= V."""
        if v < 0 or v >= self.num_vertices():
            raise OutOfRange(HG_ERANGE, "vertex_entries: vertex id out of range")
        self._export()
        b, e = int(self._offsets[v]), int(self._offsets[v + 1])
        return self.edges()[b:e]

    def close(self, stream=None) -> None:
        """Frees the device table now (stream-ordered on `stream`)."""
        if self._h:
            _lib.lib().hg_table_destroy(self._h, stream if stream is not None else self._stream)
            self._h = None

    def device_arrays(self):
        """Raw device pointers (offsets, keys, vals)."""
        o, k, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.lib().hg_table_device_arrays(self._h, C.byref(o), C.byref(k), C.byref(v)))
        return o.value, k.value, v.value


def _hash_kind(hasher) -> int:
    if hasher is None or isinstance(hasher, VertexHasher) or hasher is VertexHasher:
        return HASH_MIX64
    if isinstance(hasher, IdentityHasher) or hasher is IdentityHasher:
        return HASH_IDENTITY
    raise TypeError("the device engine supports VertexHasher and IdentityHasher only "
                    "(arbitrary host callables cannot run on the GPU)")


def _build(variant: int, keys, cfg: Optional[BuildConfig], hasher, stats, vertex_count,
           vals=None, stream=None, shard=None) -> HashGraph:
    cfg = cfg or BuildConfig()
    ka = _Arr(keys)
    va = _Arr(vals) if vals is not None else None
    c = _lib.hg_build_config()
    _lib.lib().hg_build_config_init(C.byref(c))
    c.load_factor = float(cfg.load_factor)
    c.bin_count = int(cfg.bin_count) if cfg.bin_count >= 0 else 0
    c.hash_seed = int(cfg.hash_seed)
    c.vertex_count = int(vertex_count or 0)
    c.variant = variant
    c.hash_kind = _hash_kind(hasher)
    c.stable = 1 if cfg.mode == ExecMode.sequential else 0
    c.aggregate = int(cfg.aggregate)
    c.partition_vertices = int(cfg.partition_vertices)
    if shard is not None:
        c.global_vertices, c.vertex_base = int(shard[0]), int(shard[1])
    s = stream if stream is not None else _stream_for(ka, va)
    h = C.c_void_p()
    _check(_lib.lib().hg_build(ka.ptr, ka.width, va.ptr if va else None, va.width if va else 0,
                               ka.n, C.byref(c), s, C.byref(h)))
    hg = HashGraph(h.value, s)
    if stats is not None:
        n, nv = ka.n, hg.num_vertices()
        stats.hash_evals += (2 if variant == BUILD_SIMPLE else 4) * n
        stats.count_increments += n
        stats.placement_writes += n
        stats.counter_zero_writes += nv
        if variant == BUILD_BINNED:
            stats.bin_count_increments += n
            stats.bin_placement_writes += n
            stats.counter_zero_writes += min(int(cfg.bin_count), nv)
    return hg


def build_v1(keys, cfg: Optional[BuildConfig] = None, stats: Optional[BuildStats] = None,
             vertex_count: Optional[int] = None, hasher=None, vals=None,
             stream=None, shard=None) -> HashGraph:
    """core.hpp:160-177 (simple build: count, scan, place).
    vals: explicit entry values (default: input positions, Entry::index).
    shard: (global_vertices, vertex_base) for a hash-range shard whose local
    vertex range has vertex_count vertices (sharded.py)."""
    return _build(BUILD_SIMPLE, keys, cfg, hasher, stats, vertex_count, vals, stream, shard)


def build_v2(keys, cfg: Optional[BuildConfig] = None, stats: Optional[BuildStats] = None,
             vertex_count: Optional[int] = None, hasher=None, vals=None,
             stream=None, shard=None) -> HashGraph:
    """core.hpp:183-230 (binned build: partition, then per-partition build)."""
    return _build(BUILD_BINNED, keys, cfg, hasher, stats, vertex_count, vals, stream, shard)


def probe_standard(hg: HashGraph, probe_keys, opts: Optional[ProbeOptions] = None,
                   counts=None, method: int = 0, host_ready: bool = False) -> JoinResult:
    """join.hpp:110-136. `counts` (optional, length-m uint32 array / CUDA
    tensor) receives each probe's match count. method: 0 auto, 1 direct
    gathers, 2 vertex-range partitioned probes. host_ready: pinned host probes
    already hold their final contents, so their host->device copies may
    overlap earlier work on the stream (HG_PROBE_HOST_READY)."""
    opts = opts or ProbeOptions()
    pa = _Arr(probe_keys, np.uint64 if hg.key_width == 8 else np.uint32)
    if pa.width == 8 and hg.key_width == 4:
        # A u32-keyed table probed with u64 keys: only keys < 2^32 can match.
        host = np.asarray(pa.keep if not pa.is_cuda else pa.keep.cpu().numpy(), np.uint64)
        if host.size and host.max() > 0xFFFFFFFF:
            raise InvalidArgument(HG_EINVAL, "u64 probe keys >= 2^32 against a u32-keyed table")
        pa = _Arr(host.astype(np.uint32))
    o = _lib.hg_probe_options()
    _lib.lib().hg_probe_options_init(C.byref(o))
    o.materialize = 1 if opts.materialize else 0
    o.pair_width = 8
    o.pair_cap = int(opts.pair_cap)
    o.method = int(method)
    o.flags = 1 if host_ready else 0
    pairs = None
    if opts.materialize:
        pairs = np.empty(max(min(int(opts.pair_cap), max(pa.n, 1) * max(hg.num_edges(), 1)), 0),
                         MATCH_PAIR_DTYPE)
        o.pairs = pairs.ctypes.data if pairs.size else None
        if pairs.size == 0:
            o.pair_cap = 0
    ca = _Arr(counts) if counts is not None else None
    if ca is not None:
        o.counts = ca.ptr
    r = _lib.hg_probe_result()
    s = _stream_for(pa, ca)
    _check(_lib.lib().hg_probe(hg.handle, pa.ptr, pa.width, pa.n, C.byref(o), C.byref(r), s))
    res = JoinResult(r.match_count, r.key_comparisons, bool(r.truncated), None)
    if opts.materialize:
        res.pairs = pairs[: r.pairs_written]
        res.truncated = r.match_count > int(opts.pair_cap)
    return res


def probe_device(hg: HashGraph, probes, device_result, counts=None, pairs=None,
                 pair_width: int = 4, pair_cap: int = 0, stream=None, method: int = 0) -> None:
    """Fully asynchronous probe_standard on device-resident data: totals
    {match_count, key_comparisons} land in `device_result` (CUDA u64[2]
    tensor); optional per-probe `counts` (u32) and `pairs` (pair_width 4:
    (u32 build index, u32 probe index); 8: MatchPair layout) buffers."""
    pa, ra = _Arr(probes), _Arr(device_result)
    o = _lib.hg_probe_options()
    _lib.lib().hg_probe_options_init(C.byref(o))
    o.device_result = ra.ptr
    o.method = int(method)
    if counts is not None:
        o.counts = _Arr(counts).ptr
    if pairs is not None:
        o.materialize = 1
        o.pair_width = pair_width
        o.pair_cap = pair_cap
        o.pairs = _Arr(pairs).ptr
    s = stream if stream is not None else _stream_for(pa, ra)
    _check(_lib.lib().hg_probe(hg.handle, pa.ptr, pa.width, pa.n, C.byref(o), None, s))


def _join_options(opts: ProbeOptions, cap_bound: int):
    o = _lib.hg_probe_options()
    _lib.lib().hg_probe_options_init(C.byref(o))
    o.materialize = 1 if opts.materialize else 0
    o.pair_width = 8
    o.pair_cap = int(opts.pair_cap)
    pairs = None
    if opts.materialize:
        pairs = np.empty(max(min(int(opts.pair_cap), cap_bound), 0), MATCH_PAIR_DTYPE)
        o.pairs = pairs.ctypes.data if pairs.size else None
        if pairs.size == 0:
            o.pair_cap = 0
    return o, pairs


def _join_result(r, opts: ProbeOptions, pairs) -> JoinResult:
    res = JoinResult(r.match_count, r.key_comparisons, bool(r.truncated), None)
    if opts.materialize:
        res.pairs = pairs[: r.pairs_written]
        res.truncated = r.match_count > int(opts.pair_cap)
    return res


def probe_new_prepared(hg_a: HashGraph, hg_b: HashGraph,
                       opts: Optional[ProbeOptions] = None) -> JoinResult:
    """join.hpp:143-166: adjacency intersection of two tables over one vertex
    range (K12 k_intersect). Pairs are (index in A's input, index in B's
    input), in sequential order (vertex, A position, B position).
    Raises InvalidArgument when the vertex ranges differ (join.hpp:145-147)."""
    opts = opts or ProbeOptions()
    o, pairs = _join_options(opts, max(hg_a.num_edges(), 1) * max(hg_b.num_edges(), 1))
    r = _lib.hg_probe_result()
    _check(_lib.lib().hg_probe_new_prepared(hg_a.handle, hg_b.handle, C.byref(o), C.byref(r),
                                            hg_a._stream))
    return _join_result(r, opts, pairs)


def probe_new_device(hg_a: HashGraph, hg_b: HashGraph, device_result, pairs=None,
                     pair_width: int = 4, pair_cap: int = 0, stream=None) -> None:
    """Fully asynchronous probe_new_prepared on device-resident tables:
    {match_count, key_comparisons} land in `device_result` (CUDA u64[2])."""
    ra = _Arr(device_result)
    o = _lib.hg_probe_options()
    _lib.lib().hg_probe_options_init(C.byref(o))
    o.device_result = ra.ptr
    if pairs is not None:
        o.materialize = 1
        o.pair_width = pair_width
        o.pair_cap = pair_cap
        o.pairs = _Arr(pairs).ptr
    s = stream if stream is not None else _stream_for(ra)
    _check(_lib.lib().hg_probe_new_prepared(hg_a.handle, hg_b.handle, C.byref(o), None, s))


def probe_new(keys_a, keys_b, cfg: Optional[BuildConfig] = None,
              opts: Optional[ProbeOptions] = None, hasher=None) -> JoinResult:
    """join.hpp:170-182: dual-table join. Both inputs are built (binned build)
    over the shared V = derived_vertex_count(max(|A|, |B|), load_factor), then
    intersected vertex by vertex."""
    cfg = cfg or BuildConfig()
    opts = opts or ProbeOptions()
    wa, wb = _Arr(keys_a), _Arr(keys_b)
    if wa.width != wb.width:
        wide = np.uint64
        wa = _Arr(np.asarray(wa.keep if not wa.is_cuda else wa.keep.cpu().numpy()).astype(wide))
        wb = _Arr(np.asarray(wb.keep if not wb.is_cuda else wb.keep.cpu().numpy()).astype(wide))
    c = _lib.hg_build_config()
    _lib.lib().hg_build_config_init(C.byref(c))
    c.load_factor = float(cfg.load_factor)
    c.bin_count = int(cfg.bin_count) if cfg.bin_count >= 0 else 0
    c.hash_seed = int(cfg.hash_seed)
    c.hash_kind = _hash_kind(hasher)
    c.stable = 1 if cfg.mode == ExecMode.sequential else 0
    c.aggregate = int(cfg.aggregate)
    o, pairs = _join_options(opts, max(wa.n, 1) * max(wb.n, 1))
    r = _lib.hg_probe_result()
    _check(_lib.lib().hg_probe_new(wa.ptr, wa.n, wb.ptr, wb.n, wa.width, C.byref(c), C.byref(o),
                                   C.byref(r), _stream_for(wa, wb)))
    return _join_result(r, opts, pairs)


def intersect_adjacency(a, b, emit=None, comparisons: Optional[list] = None) -> int:
    """join.hpp:41-57 for two (host) segments of ENTRY_DTYPE entries. Segment
    intersection on the device happens inside probe_new_prepared; this host
    helper exists for API completeness (it is the definition the K12 kernel
    implements per vertex)."""
    a = np.asarray(a, ENTRY_DTYPE)
    b = np.asarray(b, ENTRY_DTYPE)
    count = 0
    for ea in a:
        hits = np.nonzero(b["key"] == ea["key"])[0]
        for j in hits:
            count += 1
            if emit is not None:
                emit(int(ea["index"]), int(b["index"][j]))
    if comparisons is not None:
        comparisons[0] += len(a) * len(b)
    return count


def count_instances(hg: HashGraph, key: int, hasher=None) -> int:
    """core.hpp:235-246."""
    if hasher is not None and _hash_kind(hasher) != hg.hash_kind:
        raise TypeError("hasher does not match the table's hash")
    out = C.c_uint64(0)
    _check(_lib.lib().hg_count_instances(hg.handle, int(key), C.byref(out), None))
    return out.value


_VIOLATIONS = {
    1: "table has no vertices",
    3: "offsets[0] is not 0",
    4: "offsets are not non-decreasing",
    5: "offsets[V] does not equal the edge count",
    6: "edge count does not equal the input size",
    7: "entry stored under a vertex its key does not hash to",
    8: "entry index out of range",
    9: "duplicate entry index",
    10: "entry key does not equal input[index]",
}


def validate_csr(hg: HashGraph, expected_entries: int, input_keys=None) -> Optional[str]:
    """core.hpp:251-287 on the device; None when valid, else the violated
    invariant. input_keys additionally checks key == input[index]."""
    ia = _Arr(input_keys, np.uint64 if hg.key_width == 8 else np.uint32) \
        if input_keys is not None else None
    if ia is not None and ia.width != hg.key_width:
        ia = _Arr(np.asarray(ia.keep if not ia.is_cuda else ia.keep.cpu().numpy()).astype(
            np.uint64 if hg.key_width == 8 else np.uint32))
    code = C.c_int32(0)
    _check(_lib.lib().hg_validate(hg.handle, ia.ptr if ia else None, int(expected_entries),
                                  C.byref(code), _stream_for(ia) if ia else None))
    return None if code.value == 0 else _VIOLATIONS.get(code.value, f"violation {code.value}")


def write_keys(path, keys) -> None:
    """keygen.hpp:100-111: HGKEYS01 file from host or CUDA keys (u32 keys are
    zero-extended). Raises KeyFileError on I/O problems."""
    ka = _Arr(keys)
    _check(_lib.lib().hg_keys_write(os.fsencode(path), ka.ptr, ka.width, ka.n, _stream_for(ka)))


def read_keys(path, out=None, key_width: int = 8):
    """keygen.hpp:113-130. Returns a numpy u64 array, or fills `out` (host array
    or CUDA tensor, key_width taken from it; device destinations are streamed
    through pinned staging) and returns it. Raises KeyFileError on any I/O or
    format problem, OutOfRange when `out` is too small or a key does not fit."""
    p = os.fsencode(path)
    if out is None:
        n = C.c_uint64(0)
        _check(_lib.lib().hg_keys_file_count(p, C.byref(n)))
        out = np.zeros(n.value, np.uint64 if key_width == 8 else np.uint32)
    oa = _Arr(out)
    got = C.c_uint64(0)
    _check(_lib.lib().hg_keys_read(p, oa.ptr, oa.width, oa.n, C.byref(got), _stream_for(oa)))
    return out[: got.value] if got.value != oa.n else out


def zipf_cdf(ranks: int, s: float) -> np.ndarray:
    """CDF of P(r) ~ r^-s over ranks 1..K, built on
    the host in double and uploaded as-is (the last entry is exactly 1.0)."""
    p = np.arange(1, ranks + 1, dtype=np.float64) ** (-float(s))
    cdf = np.cumsum(p) / p.sum()
    cdf[-1] = 1.0
    return cdf


def generate(out_tensor, kind: int = 0, seed: int = 1, start: int = 0, hit: float = 1.0,
             ref=None) -> None:
    """Fills a CUDA tensor with SURVEY.md Appendix B synthetic keys: kind 0
    splitmix64, 1 C4 probes over `ref` with hit ratio `hit`, 2 scramble31
    (C4 build keys), 3 C3 Zipf keys over `ref` = a CUDA float64 CDF
    (zipf_cdf)."""
    oa = _Arr(out_tensor)
    if kind == 3:
        torch = _torch()
        if ref is None or not (isinstance(ref, torch.Tensor) and ref.is_cuda
                               and ref.dtype == torch.float64):
            raise InvalidArgument(HG_EINVAL, "Zipf keys need ref = a CUDA float64 CDF tensor")
        ref = ref.contiguous()
        rp, rn = ref.data_ptr(), ref.numel()
    else:
        ra = _Arr(ref) if ref is not None else None
        rp, rn = (ra.ptr, ra.n) if ra else (None, 0)
    _check(_lib.lib().hg_generate(oa.ptr, oa.width, oa.n, kind, seed, start, float(hit),
                                  rp, rn, _stream_for(oa)))
