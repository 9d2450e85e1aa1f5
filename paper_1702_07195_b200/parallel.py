"""Multi-GPU plumbing: residue-balanced database sharding and the one exchange
step of the path (BASELINE.json north_star (f)).

One process per GPU; each process loads only its shard with sw_db_load.  The
alignments are independent, so the only collective is the gather of results
to rank 0 (NCCL through torch.distributed):

  every rank   sw_search_dev / sw_search_batch_dev on its shard  -> local scores
               sw_topk_dev per query, indices mapped to the global database
  gather       the padded local score vectors and the top-k candidates
  rank 0       sw_scatter_dev: all scores back to original database order,
               sw_topk_dev over the candidates: the global top-k per query
               (score descending, index ascending, R5)

Every step of the path runs in the library's kernels (the backend); this
module only sizes buffers, builds the static index maps and calls the
collectives.  ``ShardedSearch`` takes the backend as an argument so that the
same orchestration runs on CPU tensors with gloo in the tests (with a stub
backend there) and on the GPU with NCCL and libswdb.so in bench.py.
"""
from __future__ import annotations

import numpy as np


def shard_database(lengths: np.ndarray, nranks: int) -> list[np.ndarray]:
    """Residue-balanced, length-stratified partition of sequence indices.

    Sequences are sorted by length (descending, ties by index) and dealt in
    serpentine order 0,1,..,N-1,N-1,..,0,0,1,.. so every rank receives the
    same length histogram and (to within one longest sequence) the same
    residue count.  Each rank's list is returned in ascending original order.
    """
    lengths = np.asarray(lengths, dtype=np.int64)
    n = lengths.size
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    order = np.lexsort((np.arange(n), -lengths))
    pos = np.arange(n)
    rnd = pos // nranks
    within = pos % nranks
    rank_of = np.where(rnd % 2 == 0, within, nranks - 1 - within)
    shards = []
    for r in range(nranks):
        shards.append(np.sort(order[rank_of == r]))
    return shards


def shard_arrays(residues: np.ndarray, offsets: np.ndarray, idx: np.ndarray):
    """(residues, offsets) of the sub-database idx (kept in idx order)."""
    idx = np.asarray(idx, dtype=np.int64)
    starts = offsets[idx]
    lens = offsets[idx + 1] - starts
    offs = np.zeros(idx.size + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    if idx.size == 0:
        return np.zeros(0, np.uint8), offs
    # vectorised gather of the residue ranges
    rep = np.repeat(starts - offs[:-1], lens)
    res = residues[np.arange(int(offs[-1]), dtype=np.int64) + rep]
    return res, offs


def merge_topk_host(scores_list, index_list, k: int):
    """Reference merge (host): global top-k by (score desc, index asc)."""
    s = np.concatenate([np.asarray(x, np.int64) for x in scores_list])
    i = np.concatenate([np.asarray(x, np.int64) for x in index_list])
    order = np.lexsort((i, -s))[:k]
    return i[order], s[order]


def gather_to_root(t, world: int, rank: int, dist, out=None):
    """Gather equal-shape tensors to rank 0 (returns list on rank 0, else None).
    With a process group (dist given) the collective runs even at world size 1.
    out: optional list of `world` preallocated receive tensors (rank 0)."""
    if dist is None:
        return [t]
    if rank == 0:
        if out is None:
            out = [t.new_empty(t.shape) for _ in range(world)]
        dist.gather(t, gather_list=out, dst=0)
        return out
    dist.gather(t, dst=0)
    return None


def assemble_scores(gathered, shards, total: int) -> np.ndarray:
    """Host reference of the rank-0 assembly: scatter the gathered (padded)
    per-rank score vectors back to the original database order."""
    out = np.empty(total, dtype=np.int32)
    for sc, idx in zip(gathered, shards):
        sc = np.asarray(sc)
        out[idx] = sc[: idx.size]
    return out


def pad_to(a, n: int):
    """Pad a 1-D numpy array or torch tensor to length n with zeros (equal-count gather)."""
    if hasattr(a, "new_zeros"):
        out = a.new_zeros(n)
        out[: a.numel()] = a
        return out
    out = np.zeros(n, dtype=a.dtype)
    out[: a.size] = a
    return out


class LibBackend:
    """The product backend: the C-ABI calls of libswdb.so on device tensors."""

    def __init__(self, sw):
        self.sw = sw

    def search(self, queries, matrix, gap_open, gap_extend, d_out, stream):
        """Scores of every query against the loaded shard into d_out (flat,
        [nq][count])."""
        if len(queries) == 1:
            self.sw.sw_search_dev(queries[0], matrix, gap_open, gap_extend, d_out, stream)
            return 1
        self.sw.sw_search_batch_dev(queries, matrix, gap_open, gap_extend, d_out, stream)
        return len(queries)

    def topk(self, d_scores, d_index, n, k, d_idx_out, d_score_out, stream):
        return self.sw.sw_topk_dev(d_scores, d_index, n, k, d_idx_out, d_score_out, stream)

    def scatter(self, d_src, d_index, n, d_dst, dst_count, stream):
        self.sw.sw_scatter_dev(d_src, d_index, n, d_dst, dst_count, stream)


class ShardedSearch:
    """One rank's part of the sharded search step.

    gidx: this rank's sequences as global database indices (ascending), in
    the order they were loaded into the backend.  count_global: sequences of
    the whole database.  nq: queries per step.  All buffers are torch tensors
    on `device`; with `dist` None the rank is alone (world 1, no collective).

    Static state (built once): every rank's local -> global index map, padded
    to the largest shard with -1 and gathered to rank 0, in the flat layout of
    the gathered score buffer: entry (rank r, query k, local i) at
    r*nq*nmax + k*count_r + i maps to k*count_global + gidx_r[i].
    """

    def __init__(self, backend, gidx, count_global: int, nq: int, topk: int, device, dist=None,
                 world: int = 1, rank: int = 0):
        import torch
        self.torch = torch
        self.backend, self.dist, self.world, self.rank = backend, dist, world, rank
        self.nq, self.k, self.count_global = int(nq), int(topk), int(count_global)
        gidx = np.asarray(gidx, dtype=np.int64)
        self.count = int(gidx.size)
        nmax = self.count
        if dist is not None:
            t = torch.tensor([self.count], dtype=torch.int64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            nmax = int(t.item())
        self.nmax = nmax
        span = self.nq * nmax
        self.d_gidx = torch.from_numpy(gidx).to(device)
        # local scores [nq][count], padded to nq*nmax for the equal-count gather
        self.d_scores = torch.zeros(span, dtype=torch.int32, device=device)
        self.tk_i = torch.empty(self.nq * self.k, dtype=torch.int64, device=device)
        self.tk_s = torch.empty(self.nq * self.k, dtype=torch.int32, device=device)
        flat = np.full(span, -1, dtype=np.int64)
        for q in range(self.nq):
            flat[q * self.count:(q + 1) * self.count] = q * self.count_global + gidx
        d_flat = torch.from_numpy(flat).to(device)
        self.kk = min(self.k, self.count_global)
        # a single process holding the whole database in original order: the
        # assembly is the identity and the merged top-k is the local one
        self.identity = (dist is None and world == 1 and self.count == self.count_global
                         and bool(np.array_equal(gidx, np.arange(self.count, dtype=np.int64))))
        if self.identity:
            self.full = self.d_scores[:self.nq * self.count]
            self.top_i = self.tk_i.view(self.nq, self.k)
            self.top_s = self.tk_s.view(self.nq, self.k)
            self.kl = min(self.k, self.count)
            return
        if rank == 0:
            self.g_scores = torch.empty(world * span, dtype=torch.int32, device=device)
            self.g_tk_i = torch.empty(world * self.nq * self.k, dtype=torch.int64, device=device)
            self.g_tk_s = torch.empty(world * self.nq * self.k, dtype=torch.int32, device=device)
            self.full = torch.zeros(self.nq * self.count_global, dtype=torch.int32, device=device)
            self.top_i = torch.empty((self.nq, self.k), dtype=torch.int64, device=device)
            self.top_s = torch.empty((self.nq, self.k), dtype=torch.int32, device=device)
            self.g_index = torch.empty(world * span, dtype=torch.int64, device=device)
        else:
            self.g_scores = self.g_tk_i = self.g_tk_s = self.full = self.top_i = self.top_s = None
            self.g_index = None
        # the static index maps, gathered once
        if dist is not None:
            gather_to_root(d_flat, world, rank, dist, out=self._views(self.g_index, world, span))
        elif rank == 0:
            self.g_index.copy_(d_flat)
        # per-rank top-k valid count (a shard smaller than k yields fewer); the
        # rest of each candidate list is padding that the merge never selects
        # (score below any real one; kk <= the real candidates of all ranks)
        self.kl = min(self.k, self.count)
        if self.kl < self.k:
            for q in range(self.nq):
                self.tk_i[q * self.k + self.kl:(q + 1) * self.k].fill_(-1)
                self.tk_s[q * self.k + self.kl:(q + 1) * self.k].fill_(-(1 << 31))

    @staticmethod
    def _views(buf, world, n):
        if buf is None:
            return None
        return [buf[r * n:(r + 1) * n] for r in range(world)]

    def step(self, queries, matrix, gap_open, gap_extend, stream) -> int:
        """One search of every query on every rank, then the gather and, on
        rank 0, the assembly of all scores in original order and the merged
        top-k.  Returns the number of library launches this rank issued."""
        nq, k, span = self.nq, self.k, self.nq * self.nmax
        launches = 0
        ctx = self.torch.cuda.stream(stream) if stream is not None else _null()
        with ctx:   # torch-side copies and the collectives follow the search stream
            if self.count > 0:
                launches += self.backend.search(queries, matrix, gap_open, gap_extend, self.d_scores, stream)
                for q in range(nq):
                    self.backend.topk(self.d_scores[q * self.count:], self.d_gidx, self.count, self.kl,
                                      self.tk_i[q * k:], self.tk_s[q * k:], stream)
                    launches += 3
            if self.identity:
                return launches
            if self.dist is not None:
                gather_to_root(self.d_scores, self.world, self.rank, self.dist,
                               out=self._views(self.g_scores, self.world, span))
                gather_to_root(self.tk_i, self.world, self.rank, self.dist,
                               out=self._views(self.g_tk_i, self.world, nq * k))
                gather_to_root(self.tk_s, self.world, self.rank, self.dist,
                               out=self._views(self.g_tk_s, self.world, nq * k))
            elif self.rank == 0:
                self.g_scores.copy_(self.d_scores)
                self.g_tk_i.copy_(self.tk_i)
                self.g_tk_s.copy_(self.tk_s)
            if self.rank != 0:
                return launches
            self.backend.scatter(self.g_scores, self.g_index, self.world * span, self.full,
                                 nq * self.count_global, stream)
            launches += 1
            # merge: the candidates of query q are the k entries at (r*nq + q)*k of every rank r
            ci, cs = self.g_tk_i, self.g_tk_s
            if nq > 1:
                ci = ci.view(self.world, nq, k).transpose(0, 1).contiguous()
                cs = cs.view(self.world, nq, k).transpose(0, 1).contiguous()
            ci = ci.view(nq, self.world * k)
            cs = cs.view(nq, self.world * k)
            for q in range(nq):
                self.backend.topk(cs[q], ci[q], self.world * k, self.kk, self.top_i[q], self.top_s[q], stream)
                launches += 3
        return launches

    def result(self):
        """Rank 0: (scores [nq, count_global], top-k indices [nq, kk], scores [nq, kk])."""
        if self.rank != 0:
            return None
        return (self.full.view(self.nq, self.count_global), self.top_i[:, :self.kk], self.top_s[:, :self.kk])


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
