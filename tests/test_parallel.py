"""Host-side multi-GPU logic on CPU: residue-balanced sharding and the
gather/merge exchange step, with world_size-2 gloo process groups (the GPU
kernels are replaced by the oracle here; the NCCL path runs the same code)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import sw_inputs as si
from paper_1702_07195_b200.parallel import (assemble_scores, gather_to_root, merge_topk_host, pad_to,
                                            shard_arrays, shard_database)


def test_shard_partition_and_balance():
    w = si.config1(scale=0.05)
    L = w.db.lengths()
    for n in (1, 2, 3, 4, 8):
        sh = shard_database(L, n)
        allidx = np.concatenate(sh)
        assert np.array_equal(np.sort(allidx), np.arange(L.size))      # exact partition
        res = np.array([L[s].sum() for s in sh])
        assert res.max() - res.min() <= L.max()                       # within one sequence
        cnt = np.array([s.size for s in sh])
        assert cnt.max() - cnt.min() <= 1
        for s in sh:
            assert np.all(np.diff(s) > 0)                              # ascending original order


def test_shard_arrays_roundtrip():
    w = si.config0(scale=0.05)
    sh = shard_database(w.db.lengths(), 3)
    for idx in sh:
        res, offs = shard_arrays(w.db.residues, w.db.offsets, idx)
        for k in (0, len(idx) // 2, len(idx) - 1):
            assert np.array_equal(res[offs[k]:offs[k + 1]], w.db.seq(int(idx[k])))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = si.config0(scale=0.1)
    q = w.queries[0]
    shards = shard_database(w.db.lengths(), world)
    idx = shards[rank]
    res, offs = shard_arrays(w.db.residues, w.db.offsets, idx)
    local = oracle.batch(q, res, offs, w.matrix, w.gap_open, w.gap_extend).astype(np.int32)
    # local top-k in global indices (what sw_topk_dev produces on each GPU)
    li, ls = merge_topk_host([local], [idx], k)
    nmax = max(s.size for s in shards)
    t_sc = torch.from_numpy(pad_to(local, nmax))
    t_ti = torch.from_numpy(pad_to(li.astype(np.int64), k))
    t_ts = torch.from_numpy(pad_to(ls.astype(np.int32), k))
    g_sc = gather_to_root(t_sc, world, rank, dist)
    g_ti = gather_to_root(t_ti, world, rank, dist)
    g_ts = gather_to_root(t_ts, world, rank, dist)
    if rank == 0:
        full = assemble_scores([x.numpy() for x in g_sc], shards, w.db.count)
        mi, ms = merge_topk_host([x.numpy() for x in g_ts], [x.numpy() for x in g_ti], k)
        np.savez(result_path, full=full, mi=mi, ms=ms)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_merge_matches_single_process(tmp_path, world):
    k = 10
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), k, path), nprocs=world, join=True)
    r = np.load(path)
    w = si.config0(scale=0.1)
    exp = oracle.batch(w.queries[0], w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend)
    assert np.array_equal(r["full"], exp)
    ei, es = oracle.topk(exp, k)
    assert np.array_equal(r["mi"], ei) and np.array_equal(r["ms"], es)


# ---------------------------------------------------------------------------
# The bench's own multi-GPU step (bench.Work + parallel.ShardedSearch) on CPU
# tensors with gloo, world size 2: per-rank shard generation, the gather of
# padded score vectors and top-k candidates, the rank-0 assembly in original
# order and the merged top-k.  The library calls are replaced by a stub
# backend (oracle scores, host top-k and scatter with the kernels' documented
# semantics); the NCCL/GPU path runs the same ShardedSearch code.
# ---------------------------------------------------------------------------
class OracleBackend:
    def __init__(self, db):
        self.db = db

    def search(self, queries, M, go, ge, d_out, stream):
        n = self.db.count
        for k, q in enumerate(queries):
            sc = oracle.batch(q, self.db.residues, self.db.offsets, M, go, ge).astype(np.int32)
            d_out[k * n:(k + 1) * n] = torch.from_numpy(sc)
        return len(queries)

    def topk(self, d_scores, d_index, n, k, d_idx_out, d_score_out, stream):
        s = d_scores[:n].numpy().astype(np.int64)
        idx = d_index[:n].numpy() if d_index is not None else np.arange(n)
        order = np.lexsort((idx, -s))[:k]
        d_idx_out[:k] = torch.from_numpy(idx[order].astype(np.int64))
        d_score_out[:k] = torch.from_numpy(s[order].astype(np.int32))
        return k

    def scatter(self, d_src, d_index, n, d_dst, dst_count, stream):
        src, idx = d_src[:n].numpy(), d_index[:n].numpy()
        keep = (idx >= 0) & (idx < dst_count)
        d_dst.numpy()[idx[keep]] = src[keep]


def _bench_worker(rank, world, port, cfg, scale, nq, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1702_07195_b200.parallel import ShardedSearch
    w = bench.Work(cfg, scale, world, rank)
    queries = w.queries[:nq]
    ss = ShardedSearch(OracleBackend(w.db), w.gidx, w.count_global, len(queries), 10, torch.device("cpu"),
                       dist=dist, world=world, rank=rank)
    ss.step(queries, w.matrix, w.gap_open, w.gap_extend, None)
    if rank == 0:
        full, ti, ts = ss.result()
        np.savez(result_path, full=full.numpy(), ti=ti.numpy(), ts=ts.numpy(),
                 ng=w.count_global, res=w.residues_global)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,scale,nq", [(0, 0.05, 1), (2, 0.0005, 2)])
def test_bench_sharded_step_gloo_world2_matches_oracle(tmp_path, cfg, scale, nq):
    """cfg0 is weak-scaled (database = configs[0] x 2), cfg2 strong (its
    database split over 2 ranks); cfg2 runs two queries through the batched
    layout [query][sequence]."""
    world = 2
    path = str(tmp_path / "res.npz")
    mp.spawn(_bench_worker, args=(world, _free_port(), cfg, scale, nq, path), nprocs=world, join=True)
    r = np.load(path)
    gscale = scale * (world if cfg in (0, 1) else 1)
    wfull = si.make_config(cfg, scale=gscale)
    qs = si.config_queries(cfg)[:nq]
    assert int(r["ng"]) == wfull.db.count and int(r["res"]) == wfull.db.total_residues
    for k, q in enumerate(qs):
        exp = oracle.batch(q, wfull.db.residues, wfull.db.offsets, wfull.matrix, wfull.gap_open, wfull.gap_extend)
        assert np.array_equal(r["full"][k], exp)
        ei, es = oracle.topk(exp, 10)
        assert np.array_equal(r["ti"][k], ei) and np.array_equal(r["ts"][k], es)


def test_host_topk_matches_oracle_sort():
    import bench
    rng = np.random.default_rng(3)
    for n, k in [(1, 10), (5, 10), (1000, 10), (1000, 1000), (50_000, 7)]:
        x = rng.integers(0, 20, n).astype(np.int32)     # many ties
        ei, _ = oracle.topk(x, k)
        assert np.array_equal(bench.host_topk(x, k), ei)
