"""CPU, world_size 2 over gloo: the sharded build/probe host logic of
paper_1907_02900_b200/sharded.py (routing splits, count exchange,
all_to_all, shard vertex ranges, global offset rebasing, result reduction)
with a numpy engine standing in for the CUDA kernels. The concatenated shard
tables must equal the oracle's single table."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class NumpyEngine:
    """Same interface as sharded.CudaEngine; CPU tensors; hashing by the oracle."""

    def __init__(self):
        from oracle.oracle import Oracle
        self.o = Oracle()

    def route(self, keys, vals, val_width, val_base, seed, hash_kind, V, G, keys_only=False):
        k = keys.numpy().astype(np.uint64) if keys.dtype == torch.int64 else \
            keys.numpy().view(np.uint32).astype(np.uint64)
        v = self.o.vertices(k, seed, V, hash_kind)
        span = (V + G - 1) // G
        owner = (v // np.uint64(span)).astype(np.int64)
        order = np.argsort(owner, kind="stable")
        idx = np.arange(val_base, val_base + len(k), dtype=np.int64)
        counts = np.bincount(owner, minlength=G).astype(np.int64)
        return (keys[torch.from_numpy(order)].contiguous(),
                torch.from_numpy(idx[order].copy()), torch.from_numpy(counts))

    @staticmethod
    def record_words(key_width, val_width):
        return 1 if key_width == 4 and val_width == 4 else 2

    def route_records(self, keys, val_width, val_base, seed, hash_kind, V, G):
        """hg_route_records' layout: 8-byte records (key | value << 32) for
        4 + 4, else two int64 words per record."""
        k, v, counts = self.route(keys, None, val_width, val_base, seed, hash_kind, V, G)
        ku = (k.numpy().view(np.uint32).astype(np.uint64) if k.dtype == torch.int32
              else k.numpy().view(np.uint64))
        vu = v.numpy().astype(np.uint64)
        if self.record_words(keys.element_size(), val_width) == 1:
            rec = (ku | (vu << np.uint64(32))).view(np.int64)
        else:
            rec = np.stack([ku, vu], 1).reshape(-1).view(np.int64)
        return torch.from_numpy(rec.copy()), counts

    def unpack_records(self, rec, key_width, val_width):
        r = rec.numpy().view(np.uint64)
        if self.record_words(key_width, val_width) == 1:
            ku, vu = r & np.uint64(0xFFFFFFFF), r >> np.uint64(32)
        else:
            ku, vu = r[0::2], r[1::2]
        k = torch.from_numpy(ku.astype(np.uint32).view(np.int32)) if key_width == 4 else \
            torch.from_numpy(ku.view(np.int64).copy())
        return k, torch.from_numpy(vu.astype(np.int64))

    def build_records(self, rec, key_width, val_width, V, base, count, cfg, hash_kind):
        k, v = self.unpack_records(rec, key_width, val_width)
        return self.build(k, v, V, base, count, cfg, hash_kind)

    def probe_pairs(self, t, probes, pos):
        """(build global index, probe global position) of every match."""
        p = probes.numpy().view(np.uint32).astype(np.uint64) if probes.dtype == torch.int32 else \
            probes.numpy().view(np.uint64)
        lv = self.o.vertices(p, t["seed"], t["V"], t["hk"]).astype(np.int64) - t["base"]
        left, right = [], []
        m = c = 0
        for j, key in enumerate(p):
            b, e = int(t["offsets"][lv[j]]), int(t["offsets"][lv[j] + 1])
            c += e - b
            hit = np.nonzero(t["keys"][b:e] == key)[0]
            m += len(hit)
            left.extend(int(t["vals"][b + h]) for h in hit)
            right.extend([int(pos[j])] * len(hit))
        return (torch.tensor(left, dtype=torch.int64), torch.tensor(right, dtype=torch.int64),
                torch.tensor([m, c], dtype=torch.int64))

    def route_pairs(self, left, right, span, G):
        owner = (right.numpy() // span).astype(np.int64)
        order = np.argsort(owner, kind="stable")
        rec = np.stack([left.numpy()[order], right.numpy()[order]], 1).reshape(-1)
        return torch.from_numpy(rec.copy()), torch.from_numpy(
            np.bincount(owner, minlength=G).astype(np.int64))

    def build(self, keys, vals, V, base, count, cfg, hash_kind):
        k = keys.numpy().astype(np.uint64) if keys.dtype == torch.int64 else \
            keys.numpy().view(np.uint32).astype(np.uint64)
        lv = self.o.vertices(k, cfg.hash_seed, V, hash_kind).astype(np.int64) - base
        assert (lv >= 0).all() and (lv < count).all(), "key routed to the wrong shard"
        order = np.argsort(lv, kind="stable")
        offs = np.zeros(count + 1, np.uint64)
        offs[1:] = np.cumsum(np.bincount(lv, minlength=count))
        return {"offsets": offs, "keys": k[order], "vals": vals.numpy()[order].astype(np.uint64),
                "V": V, "base": base, "count": count, "seed": cfg.hash_seed, "hk": hash_kind}

    def probe_totals(self, t, probes):
        p = probes.numpy().astype(np.uint64) if probes.dtype == torch.int64 else \
            probes.numpy().view(np.uint32).astype(np.uint64)
        lv = self.o.vertices(p, t["seed"], t["V"], t["hk"]).astype(np.int64) - t["base"]
        m = c = 0
        for j, key in enumerate(p):
            b, e = int(t["offsets"][lv[j]]), int(t["offsets"][lv[j] + 1])
            c += e - b
            m += int((t["keys"][b:e] == key).sum())
        return torch.tensor([m, c], dtype=torch.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1907_02900_b200.sharded import ShardedHashGraph
    from oracle.oracle import Oracle
    o = Oracle()
    n, m = 3000, 2000
    keys_all = o.splitmix(7, n * world, mask_u32=True)
    probes_all = np.concatenate([keys_all[: m * world // 2], o.splitmix(8, m * world // 2)])
    probes_all &= np.uint64(0xFFFFFFFF)
    sl = slice(rank * n, (rank + 1) * n)
    keys = torch.from_numpy(keys_all[sl].astype(np.uint32).view(np.int32))
    probes = torch.from_numpy(probes_all[rank * m:(rank + 1) * m].astype(np.uint32).view(np.int32))
    eng = ShardedHashGraph(world, rank, engine=NumpyEngine())
    for load in (1.0, 1.5):
        st = eng.build(keys, rank * n, n * world, load_factor=load)
        t = st.table
        np.savez(os.path.join(out_dir, f"shard{rank}_{load}.npz"), offsets=t["offsets"] + st.edge_base,
                 keys=t["keys"], vals=t["vals"], base=st.vertex_base, count=st.vertex_count)
        tot = eng.probe_count(probes, rank * m)
        np.save(os.path.join(out_dir, f"tot{rank}_{load}.npy"), tot.numpy())
        # pairs come back to the rank that holds the probe
        left, right, ptot = eng.probe_pairs(probes, rank * m, m * world)
        np.savez(os.path.join(out_dir, f"pairs{rank}_{load}.npz"), left=left.numpy(),
                 right=right.numpy(), tot=ptot.numpy())
    # V = 1 < world: rank 1 owns no vertex (an empty shard) and still builds
    st = eng.build(keys, rank * n, n * world, vertex_count=1)
    tot = eng.probe_count(probes, rank * m)
    np.save(os.path.join(out_dir, f"tot{rank}_v1.npy"), tot.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_build_probe_gloo(oracle, tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    n, m = 3000, 2000
    keys_all = oracle.splitmix(7, n * world, mask_u32=True)
    probes_all = np.concatenate([keys_all[: m * world // 2], oracle.splitmix(8, m * world // 2)])
    probes_all &= np.uint64(0xFFFFFFFF)
    for load in (1.0, 1.5):
        ref = oracle.build(keys_all, 1, load)
        parts = [np.load(tmp_path / f"shard{r}_{load}.npz") for r in range(world)]
        # contiguous vertex ranges, concatenated offsets == reference offsets
        assert parts[0]["base"] == 0
        offs = np.concatenate([parts[0]["offsets"][:1]] + [p["offsets"][1:] for p in parts])
        assert (offs == ref.offsets).all()
        keys = np.concatenate([p["keys"] for p in parts])
        vals = np.concatenate([p["vals"] for p in parts])
        # sequential per-shard builds keep input order -> exact equality
        assert (keys == ref.keys).all() and (vals == ref.index).all()
        r = oracle.probe_standard(ref, probes_all, materialize=True, cap=1 << 24)
        for rank in range(world):
            tot = np.load(tmp_path / f"tot{rank}_{load}.npy")
            assert tot.tolist() == [r["match_count"], r["key_comparisons"]]
        # pairs: each rank holds exactly the pairs of its own probes; together
        # they are the reference's pair set (left = build index, right = probe)
        got = []
        for rank in range(world):
            pz = np.load(tmp_path / f"pairs{rank}_{load}.npz")
            assert pz["tot"].tolist() == [r["match_count"], r["key_comparisons"]]
            assert ((pz["right"] >= rank * m) & (pz["right"] < (rank + 1) * m)).all()
            got.append(np.stack([pz["left"], pz["right"]], 1))
        got = np.concatenate(got).astype(np.uint64)
        exp = r["pairs"]
        assert len(got) == r["match_count"]
        assert (got[np.lexsort((got[:, 1], got[:, 0]))] ==
                exp[np.lexsort((exp[:, 1], exp[:, 0]))]).all()
    ref1 = oracle.build(keys_all, 1, vertex_count=1)
    r1 = oracle.probe_standard(ref1, probes_all)
    for rank in range(world):
        assert np.load(tmp_path / f"tot{rank}_v1.npy").tolist() == [r1["match_count"],
                                                                    r1["key_comparisons"]]
