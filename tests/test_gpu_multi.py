"""GPU: the multi-GPU assembly and ordering pieces of the path, on one GPU.

* sw_scatter_dev (rank 0's reassembly of the gathered shard scores in
  original order) against its documented semantics;
* parallel.ShardedSearch with the library backend at world size 1 (the same
  step bench.py times at N ranks), single query and query batch, against the
  oracle;
* searches enqueued on different streams without synchronisation (the
  library orders each search after the previous one);
* the >= 255-pass path (flag byte saturated at 255, re-scored from row 0);
* bench.py on BASELINE configs[2] as strong scaling with the NCCL gather at
  world size 1 (--dist), and the launch counter.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import sw_inputs as si
from sw_inputs import BLOSUM62, encode

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

sw = pytest.importorskip("paper_1702_07195_b200")
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield
    sw.sw_set_tile(0)


def test_scatter_dev_semantics():
    rng = np.random.default_rng(9)
    for n, dst_count, off in [(1, 1, 0), (7, 20, 0), (4096 + 3, 5000, 0), (100_003, 120_000, 1), (12, 4, 0)]:
        perm = rng.permutation(dst_count)[:min(n, dst_count)]
        idx = np.full(n, -1, np.int64)
        pos = rng.choice(n, perm.size, replace=False)
        idx[pos] = perm
        if n > 8:
            idx[rng.choice(n, 3, replace=False)] = dst_count + 5   # out of range: skipped
            idx[idx == dst_count + 5] = -7
        src = rng.integers(-2**31, 2**31 - 1, n).astype(np.int32)
        exp = np.full(dst_count, 12345, np.int32)
        keep = (idx >= 0) & (idx < dst_count)
        exp[idx[keep]] = src[keep]
        # off = 1: misaligned device pointers (the kernel's scalar path)
        d_src = torch.from_numpy(np.concatenate([[0] * off, src]).astype(np.int32)).cuda()[off:]
        d_idx = torch.from_numpy(np.concatenate([[0] * off, idx]).astype(np.int64)).cuda()[off:]
        d_dst = torch.full((dst_count,), 12345, dtype=torch.int32, device="cuda")
        sw.sw_scatter_dev(d_src, d_idx, n, d_dst, dst_count)
        torch.cuda.synchronize()
        assert np.array_equal(d_dst.cpu().numpy(), exp), (n, dst_count, off)
    with pytest.raises(sw.SWError):
        sw.sw_scatter_dev(None, None, 5, None, 5)


@pytest.mark.parametrize("nq", [1, 3])
def test_sharded_search_world1_lib_backend(nq):
    from paper_1702_07195_b200.parallel import LibBackend, ShardedSearch
    w = si.config2(scale=0.002)
    rng = np.random.default_rng(31)
    qs = [si.rr_residues(rng, L) for L in (464, 1000, 144)[:nq]]
    sw.sw_db_load(w.db.residues, w.db.offsets)
    st = torch.cuda.Stream()
    ss = ShardedSearch(LibBackend(sw), np.arange(w.db.count), w.db.count, nq, 10, torch.device("cuda"))
    ss.step(qs, w.matrix, w.gap_open, w.gap_extend, st)
    st.synchronize()
    full, ti, ts = ss.result()
    for k, q in enumerate(qs):
        exp = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend)
        assert np.array_equal(full[k].cpu().numpy(), exp), k
        ei, es = oracle.topk(exp, 10)
        assert np.array_equal(ti[k].cpu().numpy(), ei) and np.array_equal(ts[k].cpu().numpy(), es), k


def test_searches_on_different_streams_need_no_sync():
    """sw_search_dev on a side stream followed at once by
    sw_search / sw_search_dev on other streams must not clobber the shared
    per-search scratch of the first search."""
    rng = np.random.default_rng(77)
    w = si.config1(scale=0.02)
    qa, qb, qc = si.rr_residues(rng, 1500), si.rr_residues(rng, 300), si.rr_residues(rng, 900)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    ea = oracle.batch(qa, w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
    eb = oracle.batch(qb, w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
    ec = oracle.batch(qc, w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        da = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
        dc = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
        sw.sw_search_dev(qa, BLOSUM62, 10, 2, da, s1)          # multi-pass, side stream
        gb = sw.sw_search(qb, BLOSUM62, 10, 2)                  # library stream, immediately
        sw.sw_search_dev(qc, BLOSUM62, 10, 2, dc, s2)          # a third stream
        sw.sw_search_dev(qa, BLOSUM62, 10, 2, da, None)         # legacy default stream
        torch.cuda.synchronize()
        assert np.array_equal(gb, eb)
        assert np.array_equal(dc.cpu().numpy(), ec)
        assert np.array_equal(da.cpu().numpy(), ea)


def test_255_or_more_query_passes():
    """queries of >= 255 passes (8x8 tile: 64 rows per pass).  The
    flag byte saturates at 255; sequences first flagged in pass >= 254 are
    re-scored from row 0 at the end, earlier ones from their pass boundary."""
    rng = np.random.default_rng(255)
    m_rand = 13_300
    q = np.concatenate([encode("W" * 3100), si.rr_residues(rng, m_rand), encode("W" * 3000)])   # 302 passes
    seqs = [encode("W" * 3000),                       # flags early (rows < 3100)
            encode("W" * 3050),
            si.rr_residues(rng, 900),
            encode("A" * 5 + "W" * 2990),
            si.rr_residues(rng, 40)]
    db = si.database_from_list(seqs)
    exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
    assert exp.max() >= 32_757
    try:
        sw.sw_set_tile(8, 8)
        sw.sw_db_load(db.residues, db.offsets)
        got = sw.sw_search(q, BLOSUM62, 10, 2)
        st = sw.sw_last_stats()
        assert st["passes"] >= 255 and st["flagged"] >= 3
        assert np.array_equal(got, exp), (got, exp)
        # the W run at the end of the query: a sequence that saturates only in pass >= 254
        db2 = si.database_from_list([encode("G" * 30 + "W" * 2990), si.rr_residues(rng, 700)])
        sw.sw_db_load(db2.residues, db2.offsets)
        q2 = np.concatenate([si.rr_residues(rng, 16_320), encode("W" * 3000)])
        got2 = sw.sw_search(q2, BLOSUM62, 10, 2)
        exp2 = oracle.batch(q2, db2.residues, db2.offsets, BLOSUM62, 10, 2)
        assert sw.sw_last_stats()["flagged"] >= 1
        assert np.array_equal(got2, exp2), (got2, exp2)
    finally:
        sw.sw_set_tile(0)


def test_launch_counter_counts_library_kernels():
    w = si.config0(scale=0.05)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    n0 = sw.sw_launch_count()
    sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
    n1 = sw.sw_launch_count()
    st = sw.sw_last_stats()
    # 144 x 11 < the flag threshold: no score can flag, so the search is the
    # profile (with the per-search zeroing), pass and update launches only
    # (no detect, no 32-bit kernel)
    assert st["passes"] == 1 and n1 - n0 == 3
    sw.sw_topk(10)
    assert sw.sw_launch_count() - n1 == 3
    # a query whose scores can reach the threshold: the profile, then per
    # pass the pass, detect, update and 32-bit launches (plus item skipping)
    db = si.database_from_list([encode("W" * 3000), encode("A" * 40)])
    sw.sw_db_load(db.residues, db.offsets)
    try:
        sw.sw_set_wave(-1)     # per-pass launches (two items would pick the wavefront)
        n2 = sw.sw_launch_count()
        got = sw.sw_search(encode("W" * 3100), BLOSUM62, 10, 2)
        st = sw.sw_last_stats()
        assert int(got[0]) == 33000 and st["flagged"] >= 1 and st["wave"] == 0
        assert sw.sw_launch_count() - n2 >= 1 + 4 * st["passes"]
        # the wavefront: profile, one pass launch, detect + update, flag
        # compaction + 32-bit kernel at the end
        sw.sw_set_wave(1)
        n3 = sw.sw_launch_count()
        got = sw.sw_search(encode("W" * 3100), BLOSUM62, 10, 2)
        assert int(got[0]) == 33000 and sw.sw_last_stats()["wave"] == 1
        assert sw.sw_launch_count() - n3 == 6
    finally:
        sw.sw_set_wave(0)


def _run(args, env=None):
    r = subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_config2_strong_scaling_nccl_world1():
    d = _run(["bench.py", "--dist", "--config", "2", "--scale", "0.02", "--steps", "3", "--warmup", "3",
              "--no-cpu-baseline"])
    assert d["scaling"] == "strong" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["assembly_check"] is True and d["gpu_launches"] > 0
    assert d["config"]["db_sequences"] == 130_000


def test_bench_gpus_flag_single_gpu():
    d = _run(["bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3", "--scale", "0.02", "--no-cpu-baseline"])
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["config"]["assembly_check"] is True


@pytest.mark.parametrize("k", [33, 100, 1000, 4096, 4097, 10_000])
def test_topk_radix_select_matches_oracle(k):
    """Sorting stage for k > 32 (radix select of the k-th key + sort of k):
    scores with many ties, positions as indices and a sparse index map."""
    rng = np.random.default_rng(k)
    n = 600_000
    x = rng.integers(0, 60, n).astype(np.int32)            # heavy ties
    x[rng.choice(n, 50, replace=False)] = rng.integers(-5, 3000, 50)
    d = torch.from_numpy(x).cuda()
    ti = torch.empty(k, dtype=torch.int64, device="cuda")
    ts = torch.empty(k, dtype=torch.int32, device="cuda")
    assert sw.sw_topk_dev(d, None, n, k, ti, ts) == k
    ei, es = oracle.topk(x, k)
    assert np.array_equal(ti.cpu().numpy(), ei) and np.array_equal(ts.cpu().numpy(), es)
    # with an index map (global indices of a shard, as the multi-GPU merge uses)
    gidx = np.sort(rng.choice(8 * n, n, replace=False)).astype(np.int64)
    sw.sw_topk_dev(d, torch.from_numpy(gidx).cuda(), n, k, ti, ts)
    order = np.lexsort((gidx, -x.astype(np.int64)))[:k]
    assert np.array_equal(ti.cpu().numpy(), gidx[order]) and np.array_equal(ts.cpu().numpy(), x[order])


def test_topk_on_config2_scores():
    w = si.config2(scale=0.05)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    got = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
    for k in (10, 33, 100, 10_000):
        idx, sc = sw.sw_topk(k)
        ei, es = oracle.topk(got, k)
        assert np.array_equal(idx, ei) and np.array_equal(sc, es), k


@pytest.mark.parametrize("n", [2, 5, 100, 195, 1000, 2047, 2048, 5000])
def test_topk_full_sort_small_n(n):
    """The sorting stage's full bitonic path (k > n/4) for every size class:
    n < 2048 runs only global step kernels (a regression of round 2: the
    launch counter had put a step launch outside its loop)."""
    rng = np.random.default_rng(n)
    x = rng.integers(-3, 40, n).astype(np.int32)
    d = torch.from_numpy(x).cuda()
    for k in sorted({min(n, 33), n // 2 + 1, n}):
        ti = torch.empty(k, dtype=torch.int64, device="cuda")
        ts = torch.empty(k, dtype=torch.int32, device="cuda")
        assert sw.sw_topk_dev(d, None, n, k, ti, ts) == k
        ei, es = oracle.topk(x, k)
        assert np.array_equal(ti.cpu().numpy(), ei) and np.array_equal(ts.cpu().numpy(), es), (n, k)


def test_topk_dev_is_stream_ordered_and_serialised():
    """sw_topk_dev returns once enqueued (swdb.h): several calls on two side
    streams, back to back with no synchronisation in between, each read only
    after its own stream; the shared key scratch is ordered by the library."""
    rng = np.random.default_rng(7)
    n = 300_000
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    xs = [rng.integers(0, 500, n).astype(np.int32) for _ in range(4)]
    ds = [torch.from_numpy(x).cuda() for x in xs]
    torch.cuda.synchronize()
    outs = []
    for i, (x, d) in enumerate(zip(xs, ds)):
        st = s1 if i % 2 == 0 else s2
        k = (10, 33, 100, 32)[i]
        ti = torch.empty(k, dtype=torch.int64, device="cuda")
        ts = torch.empty(k, dtype=torch.int32, device="cuda")
        assert sw.sw_topk_dev(d, None, n, k, ti, ts, st) == k
        outs.append((x, k, ti, ts, st))
    for x, k, ti, ts, st in outs:
        st.synchronize()
        ei, es = oracle.topk(x, k)
        assert np.array_equal(ti.cpu().numpy(), ei) and np.array_equal(ts.cpu().numpy(), es), k


def test_timing_history_matches_last_timing():
    """sw_timing_history: the pass-kernel time of each of the last searches,
    oldest first, from the events sw_last_timing reads for the last one."""
    w = si.config0()
    sw.sw_db_load(w.db.residues, w.db.offsets)
    d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    qs = [w.queries[0], si.rr_residues(si.rng_for(0, 99), 300), si.rr_residues(si.rng_for(0, 98), 700)]
    for q in qs:
        sw.sw_search_dev(q, BLOSUM62, 10, 2, d, st)
    h = sw.sw_timing_history(3)
    last = sw.sw_last_timing()["pass_kernels_ms"]
    assert len(h) == 3 and all(x > 0 for x in h)
    assert abs(h[-1] - last) < 1e-6
    assert len(sw.sw_timing_history(1000)) <= 64
    assert (d.cpu().numpy() == oracle.batch(qs[-1], w.db.residues, w.db.offsets, BLOSUM62, 10, 2)).all()


# ---------------------------------------------------------------------------
# The bench's sharded step at world size 2 with the real kernels: two ranks
# (gloo process group, both on cuda:0, each with its own library state) build
# their shards with bench.Work, run the search and the shard top-k in
# libswdb.so, and rank 0 assembles every score in original order and merges
# the top-k with the library's scatter / top-k kernels.  gloo gathers only CPU
# tensors, so ShardedSearch runs on CPU buffers and the backend stages each
# call's operands through device copies; the ranks' kernels never wait on one
# another (no device-side exchange), so one GPU is a faithful stand-in for
# the data each rank computes.  Expected: the oracle over the whole database.
# ---------------------------------------------------------------------------
class _StagedLibBackend:
    def __init__(self):
        from paper_1702_07195_b200.parallel import LibBackend
        self.lib = LibBackend(sw)

    def search(self, queries, M, go, ge, d_out, stream):
        d = torch.zeros(d_out.numel(), dtype=torch.int32, device="cuda")
        n = self.lib.search(queries, M, go, ge, d, None)
        torch.cuda.synchronize()
        d_out.copy_(d.cpu())
        return n

    def topk(self, d_scores, d_index, n, k, d_idx_out, d_score_out, stream):
        s = d_scores[:n].cuda()
        i = d_index[:n].cuda() if d_index is not None else None
        oi = torch.empty(k, dtype=torch.int64, device="cuda")
        os_ = torch.empty(k, dtype=torch.int32, device="cuda")
        r = self.lib.topk(s, i, n, k, oi, os_, None)
        torch.cuda.synchronize()
        d_idx_out[:k].copy_(oi.cpu())
        d_score_out[:k].copy_(os_.cpu())
        return r

    def scatter(self, d_src, d_index, n, d_dst, dst_count, stream):
        dst = d_dst.cuda()
        self.lib.scatter(d_src[:n].cuda(), d_index[:n].cuda(), n, dst, dst_count, None)
        torch.cuda.synchronize()
        d_dst.copy_(dst.cpu())


def _world2_worker(rank, world, port, cfg, scale, nq, result_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1702_07195_b200.parallel import ShardedSearch
    w = bench.Work(cfg, scale, world, rank)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    queries = w.queries[:nq]
    ss = ShardedSearch(_StagedLibBackend(), w.gidx, w.count_global, len(queries), 10, torch.device("cpu"),
                       dist=dist, world=world, rank=rank)
    for _ in range(2):    # a second step over the same buffers: the assembly is repeatable
        ss.step(queries, w.matrix, w.gap_open, w.gap_extend, None)
    if rank == 0:
        full, ti, ts = ss.result()
        np.savez(result_path, full=full.numpy(), ti=ti.numpy(), ts=ts.numpy(), ng=w.count_global,
                 res=w.residues_global, mine=w.db.count)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,scale,nq", [(2, 0.003, 1), (3, 0.002, 3), (4, 0.01, 1), (0, 0.2, 1)])
def test_bench_sharded_step_world2_real_kernels(tmp_path, cfg, scale, nq):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "res.npz")
    mp.spawn(_world2_worker, args=(2, port, cfg, scale, nq, path), nprocs=2, join=True)
    r = np.load(path)
    gscale = scale * (2 if cfg in (0, 1) else 1)
    wfull = si.make_config(cfg, scale=gscale)
    assert int(r["ng"]) == wfull.db.count and int(r["res"]) == wfull.db.total_residues
    assert 0 < int(r["mine"]) < wfull.db.count          # rank 0 held a proper shard
    qs = wfull.queries[:nq]
    for k, q in enumerate(qs):
        exp = oracle.batch(q, wfull.db.residues, wfull.db.offsets, wfull.matrix, wfull.gap_open,
                           wfull.gap_extend)
        assert np.array_equal(r["full"][k], exp), (cfg, k, int(np.sum(r["full"][k] != exp)))
        ei, es = oracle.topk(exp, 10)
        assert np.array_equal(r["ti"][k], ei) and np.array_equal(r["ts"][k], es)
