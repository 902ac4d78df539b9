"""Hash-range sharded HashGraph across GPUs (one process per GPU).

SURVEY.md 8(e): the reference's bin formula (core.hpp:192-197,
bin = v / ceil(V / bins)) at bins = G picks the owner GPU of vertex v, so the
global table is the concatenation of G local tables over contiguous vertex
ranges. Per rank:

  build   route   keys -> owner-grouped (key, global index) send buffers
                  (K11, hg_route; one pass of the partition machinery)
          counts  all_gather of the G x G send-count matrix
          all2all torch.distributed all_to_all_single over NCCL / NVLink
          build   local V1/V2 build over [base, base + S) with the global hash
                  (hg_build with global_vertices / vertex_base)
  probe   route probes the same way (value = global probe position), local
          probe_standard, all_reduce of (match_count, key_comparisons);
          pairs stay on the owner (or are gathered for parity checks).

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
              global_vertices: int, shards: int):
        t = self.torch
        ka = _Arr(keys)
        n = ka.n
        out_k = self.empty(n, ka.width)
        out_v = self.empty(n, val_width)
        counts = t.zeros(shards, dtype=t.int64, device="cuda")
        va = _Arr(vals) if vals is not None else None
        s = t.cuda.current_stream().cuda_stream
        _check(_lib.lib().hg_route(ka.ptr, ka.width, va.ptr if va else None, val_width, n,
                                   val_base, seed, hash_kind, global_vertices, shards,
                                   out_k.data_ptr(), out_v.data_ptr(), counts.data_ptr(), s))
        return out_k, out_v, counts

    def build(self, keys, vals, global_vertices: int, base: int, count: int, cfg: BuildConfig,
              hash_kind: int):
        from .hashgraph import IdentityHasher
        fn = build_v2 if self.variant == 2 else build_v1
        hasher = IdentityHasher() if hash_kind == 1 else None
        return fn(keys, cfg, vertex_count=count, hasher=hasher, vals=vals,
                  shard=(global_vertices, base))

    def probe_totals(self, table: HashGraph, probes):
        t = self.torch
        res = t.zeros(2, dtype=t.int64, device="cuda")
        probe_device(table, probes, res)
        return res

    def probe_pairs(self, table: HashGraph, probes, probe_idx):
        """Pairs (build global index, probe global index) as two tensors."""
        t = self.torch
        n = probes.numel()
        counts = t.zeros(n, dtype=t.int32, device="cuda")
        res = t.zeros(2, dtype=t.int64, device="cuda")
        probe_device(table, probes, res, counts=counts)
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

    # -------------------------------------------------------------- plumbing
    def _exchange(self, send_k, send_v, counts):
        """All-to-all of owner-grouped SoA buffers; returns received (k, v)."""
        import torch
        dist = self.dist
        G = self.world
        cnt = counts.to(torch.int64)
        gathered = [torch.zeros_like(cnt) for _ in range(G)]
        dist.all_gather(gathered, cnt, group=self.group)
        send_splits = [int(x) for x in cnt.cpu().tolist()]
        recv_splits = [int(g[self.rank].item()) for g in gathered]
        nrecv = sum(recv_splits)
        recv_k = send_k.new_empty(nrecv)
        recv_v = send_v.new_empty(nrecv)
        dist.all_to_all_single(recv_k, send_k, recv_splits, send_splits, group=self.group)
        dist.all_to_all_single(recv_v, send_v, recv_splits, send_splits, group=self.group)
        return recv_k, recv_v

    def _allreduce_sum(self, x):
        self.dist.all_reduce(x, group=self.group)
        return x

    # -------------------------------------------------------------- build
    def build(self, keys, global_offset: int, global_n: int, load_factor: float = 1.0,
              vertex_count: Optional[int] = None, mode: ExecMode = ExecMode.parallel,
              partition_vertices: int = 0) -> ShardedTable:
        """keys: this rank's slice of the global input, whose first element is
        global position `global_offset`; global_n = total keys on all ranks."""
        import torch
        V = vertex_count or derived_vertex_count(global_n, load_factor)
        base, count = shard_range(V, self.world, self.rank)
        val_width = 4 if global_n <= (1 << 32) else 8
        send_k, send_v, counts = self.engine.route(keys, None, val_width, global_offset,
                                                   self.hash_seed, self.hash_kind, V, self.world)
        recv_k, recv_v = self._exchange(send_k, send_v, counts)
        cfg = BuildConfig(load_factor=load_factor, hash_seed=self.hash_seed, mode=mode,
                          partition_vertices=partition_vertices)
        table = self.engine.build(recv_k, recv_v, V, base, max(count, 1), cfg, self.hash_kind)
        n_local = torch.tensor([recv_k.numel()], dtype=torch.int64, device=recv_k.device)
        all_n = [torch.zeros_like(n_local) for _ in range(self.world)]
        self.dist.all_gather(all_n, n_local, group=self.group)
        edge_base = sum(int(x.item()) for x in all_n[: self.rank])
        self.table = ShardedTable(table, V, base, count, edge_base, int(recv_k.numel()))
        self.last_local_n = int(recv_k.numel())
        self.local_vertices = count
        return self.table

    # -------------------------------------------------------------- probe
    def probe_count(self, probes, global_offset: int = 0):
        """probe_standard match_count / key_comparisons over all ranks'
        probes (device tensor [2] after the all_reduce)."""
        st = self.table
        width = 4 if probes.element_size() == 4 else 8
        send_k, send_v, counts = self.engine.route(probes, None, 4, global_offset, self.hash_seed,
                                                   self.hash_kind, st.global_vertices, self.world)
        recv_k, _ = self._exchange(send_k, send_v, counts)
        self.last_local_m = int(recv_k.numel())
        tot = self.engine.probe_totals(st.table, recv_k)
        self.last_local_c = int(tot[1].item()) if self.world > 0 else 0
        return self._allreduce_sum(tot)

    def probe_pairs(self, probes, global_offset: int, global_m: int):
        """Match pairs (build global index, probe global index) owned by this
        rank, plus the all-reduced (match_count, key_comparisons)."""
        st = self.table
        pw = 4 if global_m <= (1 << 32) else 8
        send_k, send_v, counts = self.engine.route(probes, None, pw, global_offset,
                                                   self.hash_seed, self.hash_kind,
                                                   st.global_vertices, self.world)
        recv_k, recv_v = self._exchange(send_k, send_v, counts)
        left, right, tot = self.engine.probe_pairs(st.table, recv_k, recv_v)
        return left, right, self._allreduce_sum(tot)

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
