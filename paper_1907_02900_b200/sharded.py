"""Hash-range sharded HashGraph across GPUs (one process per GPU).

SURVEY.md 8(e): the reference's bin formula (core.hpp:192-197,
bin = v / ceil(V / bins)) at bins = G picks the owner GPU of vertex v, so the
global table is the concatenation of G local tables over contiguous vertex
ranges. Per rank:

  build   route   keys -> owner-grouped AoS records {key, global index} in
                  one buffer (K11, hg_route_records)
          counts  all_to_all_single of the G send counts (device), one D2H
                  of (send, recv) counts -- NCCL needs host-known split sizes
          all2all ONE all_to_all_single of the records over NCCL / NVLink
          build   local V1/V2 build over [base, base + S) with the global hash,
                  straight from the received records (hg_build_records: the
                  binned build's first pass reads them, no unpack)
  probe   count-only: route probe keys (hg_route), one all_to_all of the keys,
          local probe_standard, all_reduce of (match_count, key_comparisons);
          pairs: route probes as records {key, global probe position}, local
          probe with pairs, then the REVERSE route (hg_route_pairs, owner =
          probe position / probes per rank) and all_to_all return every pair
          to the rank that holds its probe.

The result equals the reference's single table: offsets of shard g are its
local offsets + the number of entries on shards < g, and per-vertex entry
multisets are identical (SURVEY.md 8(c) invariant proof).

The collective plumbing is shared between the product engine (CudaEngine:
the C-ABI kernels on CUDA tensors, NCCL) and any engine with the same
interface -- the CPU tests run this exact host logic over the gloo backend
with the oracle as the engine (tests/test_sharded_gloo.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from . import _lib
from .hashgraph import (BuildConfig, ExecMode, HashGraph, _Arr, _check, build_v1, build_v2,
                        derived_vertex_count, probe_device)


def shard_range(global_vertices: int, shards: int, shard: int) -> tuple[int, int]:
    """(vertex_base, vertex_count) of `shard` (hg_shard_range)."""
    span = (global_vertices + shards - 1) // shards
    b = min(global_vertices, shard * span)
    e = min(global_vertices, b + span)
    return b, e - b


class CudaEngine:
    """Product engine: the sm_100a kernels through the C-ABI, CUDA tensors."""

    def __init__(self, variant: int = 2):
        import torch
        self.torch = torch
        self.variant = variant

    def empty(self, n: int, width: int):
        t = self.torch
        return t.empty(n, dtype=t.int32 if width == 4 else t.int64, device="cuda")

    def route(self, keys, vals, val_width: int, val_base: int, seed: int, hash_kind: int,
              global_vertices: int, shards: int, keys_only: bool = False):
        t = self.torch
        ka = _Arr(keys)
        n = ka.n
        out_k = self.empty(n, ka.width)
        out_v = None if keys_only else self.empty(n, val_width)
        counts = t.zeros(shards, dtype=t.int64, device="cuda")
        va = _Arr(vals) if vals is not None else None
        s = t.cuda.current_stream().cuda_stream
        _check(_lib.lib().hg_route(ka.ptr, ka.width, va.ptr if va else None, val_width, n,
                                   val_base, seed, hash_kind, global_vertices, shards,
                                   out_k.data_ptr(), out_v.data_ptr() if out_v is not None else None,
                                   counts.data_ptr(), s))
        return out_k, out_v, counts

    def build(self, keys, vals, global_vertices: int, base: int, count: int, cfg: BuildConfig,
              hash_kind: int):
        from .hashgraph import IdentityHasher
        fn = build_v2 if self.variant == 2 else build_v1
        hasher = IdentityHasher() if hash_kind == 1 else None
        if count == 0:  # this rank owns no vertex (V < G): an empty unsharded table
            return fn(keys, cfg, vertex_count=1, hasher=hasher, vals=vals)
        return fn(keys, cfg, vertex_count=count, hasher=hasher, vals=vals,
                  shard=(global_vertices, base))

    @staticmethod
    def record_words(key_width: int, val_width: int) -> int:
        """int64 words per AoS record (8-byte records for 4 + 4, else 16)."""
        return 1 if key_width == 4 and val_width == 4 else 2

    def route_records(self, keys, val_width: int, val_base: int, seed: int, hash_kind: int,
                      global_vertices: int, shards: int):
        """Owner-grouped AoS records {key, global index} (hg_route_records) as an
        int64 tensor of n * record_words elements, plus device counts."""
        t = self.torch
        ka = _Arr(keys)
        w = self.record_words(ka.width, val_width)
        out = t.empty(max(ka.n, 1) * w, dtype=t.int64, device="cuda")
        counts = t.zeros(shards, dtype=t.int64, device="cuda")
        s = t.cuda.current_stream().cuda_stream
        _check(_lib.lib().hg_route_records(ka.ptr, ka.width, None, val_width, ka.n, val_base,
                                           seed, hash_kind, global_vertices, shards,
                                           out.data_ptr(), counts.data_ptr(), s))
        return out[: ka.n * w], counts

    def build_records(self, records, key_width: int, val_width: int, global_vertices: int,
                      base: int, count: int, cfg: BuildConfig, hash_kind: int) -> HashGraph:
        """Local build straight from received records (hg_build_records)."""
        from .hashgraph import BUILD_BINNED, BUILD_SIMPLE, ExecMode
        t = self.torch
        w = self.record_words(key_width, val_width)
        n = records.numel() // w
        c = _lib.hg_build_config()
        _lib.lib().hg_build_config_init(C.byref(c))
        c.load_factor = float(cfg.load_factor)
        c.hash_seed = int(cfg.hash_seed)
        c.variant = BUILD_BINNED if self.variant == 2 else BUILD_SIMPLE
        c.hash_kind = int(hash_kind)
        c.stable = 1 if cfg.mode == ExecMode.sequential else 0
        c.partition_vertices = int(cfg.partition_vertices)
        if count:
            c.vertex_count = int(count)
            c.global_vertices, c.vertex_base = int(global_vertices), int(base)
        else:  # this rank owns no vertex: an empty unsharded table
            c.vertex_count = 1
        s = t.cuda.current_stream().cuda_stream
        h = C.c_void_p()
        _check(_lib.lib().hg_build_records(records.data_ptr() if n else None, key_width,
                                           val_width, n, C.byref(c), s, C.byref(h)))
        return HashGraph(h.value, s)

    def unpack_records(self, records, key_width: int, val_width: int):
        """(keys, values) views of received records, contiguous for the C-ABI."""
        t = self.torch
        if self.record_words(key_width, val_width) == 1:
            kv = records.view(t.int32).view(-1, 2)
            return kv[:, 0].contiguous(), kv[:, 1].contiguous()
        kv = records.view(-1, 2)
        keys = kv[:, 0].contiguous()
        if key_width == 4:
            keys = keys.to(t.int32)
        vals = kv[:, 1].contiguous()
        return keys, (vals.to(t.int32) if val_width == 4 else vals)

    def route_pairs(self, left, right, span: int, shards: int):
        """Pairs grouped by the rank holding their probe (owner = right / span),
        AoS records {left, right} (hg_route_pairs) + device counts."""
        t = self.torch
        la, ra = _Arr(left), _Arr(right)
        n = la.n
        out = t.empty(max(n, 1) * 2, dtype=left.dtype, device="cuda")
        counts = t.zeros(shards, dtype=t.int64, device="cuda")
        s = t.cuda.current_stream().cuda_stream
        _check(_lib.lib().hg_route_pairs(la.ptr, ra.ptr, la.width, n, span, shards,
                                         out.data_ptr(), counts.data_ptr(), s))
        return out[: 2 * n], counts

    def probe_totals(self, table: HashGraph, probes):
        t = self.torch
        res = t.zeros(2, dtype=t.int64, device="cuda")
        probe_device(table, probes, res)
        return res

    def probe_pairs(self, table: HashGraph, probes, probe_idx):
        """Pairs (build global index, probe global index) as two tensors."""
        t = self.torch
        n = probes.numel()
        res = t.zeros(2, dtype=t.int64, device="cuda")
        probe_device(table, probes, res)  # count-only pass sizes the pair buffer
        total = int(res[0].item())
        pw = 8 if table.val_width == 8 or n > (1 << 32) else 4
        pairs = t.empty(max(total, 1) * 2, dtype=t.int32 if pw == 4 else t.int64, device="cuda")
        res2 = t.zeros(2, dtype=t.int64, device="cuda")
        probe_device(table, probes, res2, pairs=pairs, pair_width=pw, pair_cap=total)
        pairs = pairs[: 2 * total].view(total, 2)
        left = pairs[:, 0].to(t.int64) & 0xFFFFFFFF if pw == 4 else pairs[:, 0]
        right_local = pairs[:, 1].to(t.int64) & 0xFFFFFFFF if pw == 4 else pairs[:, 1]
        pidx = probe_idx.to(t.int64) & (0xFFFFFFFF if probe_idx.element_size() == 4 else -1)
        return left, pidx[right_local], res


@dataclass
class ShardedTable:
    table: HashGraph
    global_vertices: int
    vertex_base: int
    vertex_count: int
    edge_base: int        # entries on shards < rank (global offsets = local + edge_base)
    local_n: int


class ShardedHashGraph:
    """Hash-range sharded build + probe across the ranks of `group`."""

    def __init__(self, world: int, rank: int, variant: int = 2, engine=None, group=None,
                 hash_seed: int = 0, hash_kind: int = 0):
        import torch.distributed as dist
        self.dist = dist
        self.world, self.rank, self.group = world, rank, group
        self.engine = engine or CudaEngine(variant)
        self.hash_seed, self.hash_kind = hash_seed, hash_kind
        self.table: Optional[ShardedTable] = None
        self.last_local_n = self.last_local_m = self.last_local_c = 0
        self.local_vertices = 0
        self.last_build_bytes = self.last_probe_bytes = 0
        self.exchange_events = None  # a list -> time every all_to_all (bench)

    # -------------------------------------------------------------- plumbing
    def _count_matrix(self, counts):
        """G x G send-count matrix M[g][p] (rank g -> rank p) from every rank's
        device counts: one all_gather, one D2H (NCCL's all-to-all takes host
        split sizes, and the local build sizes its scratch from its count)."""
        import torch
        G = self.world
        cnt = counts.to(torch.int64)
        gathered = [torch.zeros_like(cnt) for _ in range(G)]
        self.dist.all_gather(gathered, cnt, group=self.group)
        flat = torch.stack(gathered).cpu().tolist()
        return [[int(x) for x in row] for row in flat]

    def _alltoall(self, send, M, words: int = 1):
        """ONE all_to_all_single of an owner-grouped buffer (`words` elements
        per item) by the count matrix M; returns the received buffer."""
        r = self.rank
        send_splits = [c * words for c in M[r]]
        recv_splits = [M[g][r] * words for g in range(self.world)]
        recv = send.new_empty(sum(recv_splits))
        ev = None
        if self.exchange_events is not None and send.is_cuda:
            import torch
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        self.dist.all_to_all_single(recv, send, recv_splits, send_splits, group=self.group)
        if ev is not None:
            ev[1].record()
            self.exchange_events.append(ev)
        return recv

    def exchange_ms(self) -> float:
        """Device time of the all-to-alls recorded since exchange_events was
        set to [] (CUDA events on the current stream around each exchange)."""
        ms = sum(a.elapsed_time(b) for a, b in self.exchange_events or [])
        self.exchange_events = None
        return ms

    def _allreduce_sum(self, x):
        self.dist.all_reduce(x, group=self.group)
        return x

    # -------------------------------------------------------------- build
    def build(self, keys, global_offset: int, global_n: int, load_factor: float = 1.0,
              vertex_count: Optional[int] = None, mode: ExecMode = ExecMode.parallel,
              partition_vertices: int = 0) -> ShardedTable:
        """keys: this rank's slice of the global input, whose first element is
        global position `global_offset`; global_n = total keys on all ranks."""
        V = vertex_count or derived_vertex_count(global_n, load_factor)
        base, count = shard_range(V, self.world, self.rank)
        kw = keys.element_size()
        vw = 4 if global_n <= (1 << 32) else 8
        w = self.engine.record_words(kw, vw)
        rec, counts = self.engine.route_records(keys, vw, global_offset, self.hash_seed,
                                                self.hash_kind, V, self.world)
        M = self._count_matrix(counts)
        recv = self._alltoall(rec, M, w)
        cfg = BuildConfig(load_factor=load_factor, hash_seed=self.hash_seed, mode=mode,
                          partition_vertices=partition_vertices)
        table = self.engine.build_records(recv, kw, vw, V, base, count, cfg, self.hash_kind)
        n_of = [sum(M[g][p] for g in range(self.world)) for p in range(self.world)]
        edge_base = sum(n_of[: self.rank])
        local_n = n_of[self.rank]
        self.table = ShardedTable(table, V, base, count, edge_base, local_n)
        self.last_local_n = local_n
        self.local_vertices = count
        self.last_build_bytes = self._nvlink_bytes(M, w * 8)
        return self.table

    def _nvlink_bytes(self, M, item_bytes: int) -> int:
        """Bytes this rank sends to OTHER ranks (its NVLink egress) in one
        exchange with count matrix M."""
        r = self.rank
        return sum(c for p, c in enumerate(M[r]) if p != r) * item_bytes

    # -------------------------------------------------------------- probe
    def probe_count(self, probes, global_offset: int = 0):
        """probe_standard match_count / key_comparisons over all ranks'
        probes (device tensor [2] after the all_reduce). Only the probe keys
        travel (count-only needs no positions)."""
        st = self.table
        send_k, _, counts = self.engine.route(probes, None, 4, global_offset, self.hash_seed,
                                              self.hash_kind, st.global_vertices, self.world,
                                              keys_only=True)
        M = self._count_matrix(counts)
        recv_k = self._alltoall(send_k, M)
        self.last_local_m = int(recv_k.numel())
        self.last_probe_bytes = self._nvlink_bytes(M, probes.element_size())
        tot = self.engine.probe_totals(st.table, recv_k)
        self.last_local_c = int(tot[1].item())
        return self._allreduce_sum(tot)

    def probe_pairs(self, probes, global_offset: int, global_m: int):
        """probe_standard with pairs: returns, on the rank that holds the
        probes, the pairs (build global index, probe global index) of ITS
        probes -- routed to the table owner as records {key, global probe
        position}, probed there, and routed back by probe position
        (hg_route_pairs) -- plus the all-reduced (match_count,
        key_comparisons). Ranks hold equal probe slices: rank r's probes have
        global positions [r * m, (r + 1) * m)."""
        st = self.table
        m = probes.numel()
        if global_offset != self.rank * m:
            raise ValueError("probe_pairs expects equal probe slices (global_offset = rank * m)")
        kw = probes.element_size()
        pw = 4 if global_m <= (1 << 32) else 8
        w = self.engine.record_words(kw, pw)
        rec, counts = self.engine.route_records(probes, pw, global_offset, self.hash_seed,
                                                self.hash_kind, st.global_vertices, self.world)
        M = self._count_matrix(counts)
        recv = self._alltoall(rec, M, w)
        keys, pos = self.engine.unpack_records(recv, kw, pw)
        left, right, tot = self.engine.probe_pairs(st.table, keys, pos)
        # reverse route: every pair back to the rank holding its probe
        prec, pcounts = self.engine.route_pairs(left, right, max(m, 1), self.world)
        M2 = self._count_matrix(pcounts)
        back = self._alltoall(prec, M2, 2).view(-1, 2)
        return back[:, 0], back[:, 1], self._allreduce_sum(tot)

    # -------------------------------------------------------------- step
    def build_and_probe(self, keys, probes, result, n_per_rank: Optional[int] = None):
        """One bench step: sharded build of every rank's keys + count-only
        probe of every rank's probes; result (device int64[2]) receives the
        global (match_count, key_comparisons)."""
        n = keys.numel()
        g_n = n * self.world if n_per_rank is None else n_per_rank * self.world
        self.build(keys, self.rank * n, g_n)
        tot = self.probe_count(probes, self.rank * probes.numel())
        result.copy_(tot)
        self.table.table.close()

    def export_global(self):
        """Rank-local view rebased to global offsets: (offsets[count+1] with
        global values, keys, vals) as host numpy arrays."""
        st = self.table
        off = st.table.offsets().copy() + st.edge_base
        return off, st.table.edge_keys(), st.table.edge_index()
