"""Multi-GPU plumbing: residue-balanced database sharding and the one exchange
step of the path (BASELINE.json north_star (f)): gathering per-GPU scores and
top-k candidates to rank 0 with NCCL (torch.distributed) and merging them
with the library's device top-k (sw_topk_dev).

One process per GPU; each process loads only its shard with sw_db_load.
The alignments are independent, so the only collective is the gather of
results.  Host-side logic here is covered by
world_size-2 gloo tests on CPU (tests/test_parallel.py).
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


def gather_to_root(t, world: int, rank: int, dist):
    """Gather equal-shape tensors to rank 0 (returns list on rank 0, else None).
    With a process group (dist given) the collective runs even at world size 1."""
    if dist is None:
        return [t]
    if rank == 0:
        out = [t.new_empty(t.shape) for _ in range(world)]
        dist.gather(t, gather_list=out, dst=0)
        return out
    dist.gather(t, dst=0)
    return None


def assemble_scores(gathered, shards, total: int) -> np.ndarray:
    """Rank 0: scatter the gathered (padded) per-rank score vectors back to the
    original database order using the static shard index maps."""
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
