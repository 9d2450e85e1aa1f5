"""Thin Python binding of libswdb.so (include/swdb.h) -- argument marshalling
only.  Every step of the search runs in the native library's CUDA kernels;
there is no Python or CPU fallback: if the library is missing or fails to
load, every call raises.

Names follow the C-ABI: sw_db_load, sw_search, sw_search_dev, sw_topk,
sw_topk_dev, sw_db_free, sw_last_error.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB

SW_OK, SW_EINVAL, SW_ENOMEM, SW_ECUDA, SW_ENODB, SW_ESTATE = 0, -1, -2, -3, -4, -5
_NAMES = {SW_EINVAL: "SW_EINVAL", SW_ENOMEM: "SW_ENOMEM", SW_ECUDA: "SW_ECUDA",
          SW_ENODB: "SW_ENODB", SW_ESTATE: "SW_ESTATE"}

EXPORTS = ["sw_db_load", "sw_db_load_streamed", "sw_db_chunks", "sw_db_head_columns", "sw_db_free", "sw_db_count", "sw_db_residues", "sw_search",
           "sw_search_dev", "sw_search_batch", "sw_search_batch_dev", "sw_topk", "sw_topk_dev", "sw_scatter_dev", "sw_last_stats", "sw_last_timing", "sw_timing_history", "sw_set_tile",
           "sw_tile_supported", "sw_set_wave", "sw_set_latency_mode", "sw_set_profile", "sw_set_rows_mode", "sw_last_error", "sw_version", "sw_launch_count"]


class SWError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def library_path() -> str:
    return LIB


def load_library():
    """Load libswdb.so (raises if it is missing: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise RuntimeError(f"native library {LIB} is missing; build it with "
                           "`python -m paper_1702_07195_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB)
    p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "sw_db_load": (ctypes.c_int, [p, p, i64]),
        "sw_db_load_streamed": (ctypes.c_int, [p, p, i64, i64]),
        "sw_db_chunks": (i64, []),
        "sw_db_head_columns": (i64, []),
        "sw_db_free": (None, []),
        "sw_db_count": (i64, []),
        "sw_db_residues": (i64, []),
        "sw_search": (ctypes.c_int, [p, i32, p, i32, i32, p]),
        "sw_search_dev": (ctypes.c_int, [p, i32, p, i32, i32, p, p]),
        "sw_search_batch": (ctypes.c_int, [p, p, i32, p, i32, i32, p]),
        "sw_search_batch_dev": (ctypes.c_int, [p, p, i32, p, i32, i32, p, p]),
        "sw_topk": (i64, [i64, p, p]),
        "sw_topk_dev": (i64, [p, p, i64, i64, p, p, p]),
        "sw_scatter_dev": (ctypes.c_int, [p, p, i64, p, i64, p]),
        "sw_last_stats": (ctypes.c_int, [p, ctypes.c_int]),
        "sw_last_timing": (ctypes.c_int, [p, ctypes.c_int]),
        "sw_timing_history": (ctypes.c_int, [p, ctypes.c_int]),
        "sw_set_tile": (ctypes.c_int, [i32, i32]),
        "sw_tile_supported": (ctypes.c_int, [i32, i32]),
        "sw_set_wave": (ctypes.c_int, [i32]),
        "sw_set_latency_mode": (ctypes.c_int, [i32]),
        "sw_set_profile": (ctypes.c_int, [i32]),
        "sw_set_rows_mode": (ctypes.c_int, [i32]),
        "sw_last_error": (ctypes.c_char_p, []),
        "sw_version": (ctypes.c_char_p, []),
        "sw_launch_count": (i64, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(rc: int) -> int:
    if rc < 0:
        raise SWError(int(rc), sw_last_error())
    return rc


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _matrix(m) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(m, dtype=np.int8))
    if m.shape != (24, 24):
        raise ValueError("matrix must be 24x24 int8")
    return m


def _dev_ptr(x) -> int:
    if x is None:
        return 0
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    return int(x)


def _stream_ptr(stream) -> int:
    if stream is None:
        return 0
    if hasattr(stream, "cuda_stream"):
        return int(stream.cuda_stream)
    return int(stream)


def sw_last_error() -> str:
    return load_library().sw_last_error().decode()


def sw_launch_count() -> int:
    """Kernels launched by the library since it was loaded."""
    return int(load_library().sw_launch_count())


def sw_version() -> str:
    return load_library().sw_version().decode()


def sw_db_load(residues, offsets) -> None:
    res = _u8(residues)
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    count = int(offs.size - 1)
    _check(load_library().sw_db_load(_ptr(res) if res.size else None, _ptr(offs), count))


def sw_db_load_streamed(residues, offsets, chunk_bytes: int) -> None:
    """Out-of-core database: the image stays in pinned host memory and is
    streamed to the device in chunks of <= chunk_bytes during each search."""
    res = _u8(residues)
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    _check(load_library().sw_db_load_streamed(_ptr(res) if res.size else None, _ptr(offs), int(offs.size - 1),
                                              int(chunk_bytes)))


def sw_db_chunks() -> int:
    return int(load_library().sw_db_chunks())


def sw_db_head_columns() -> int:
    """Columns of a streamed database's resident head, 0 if none (swdb.h)."""
    return int(load_library().sw_db_head_columns())


def sw_db_free() -> None:
    load_library().sw_db_free()


def sw_db_count() -> int:
    return int(load_library().sw_db_count())


def sw_db_residues() -> int:
    return int(load_library().sw_db_residues())


def sw_search(query, matrix, gap_open: int, gap_extend: int, out: np.ndarray | None = None) -> np.ndarray:
    q = _u8(query)
    m = _matrix(matrix)
    n = sw_db_count()
    if out is None:
        out = np.empty(n, dtype=np.int32)
    assert out.dtype == np.int32 and out.flags.c_contiguous and out.size >= n
    _check(load_library().sw_search(_ptr(q), int(q.size), _ptr(m), int(gap_open), int(gap_extend), _ptr(out)))
    return out


def sw_search_dev(query, matrix, gap_open: int, gap_extend: int, d_scores, stream=None) -> None:
    q = _u8(query)
    m = _matrix(matrix)
    _check(load_library().sw_search_dev(_ptr(q), int(q.size), _ptr(m), int(gap_open), int(gap_extend),
                                        _dev_ptr(d_scores), _stream_ptr(stream)))


def _pack_queries(queries):
    qs = [_u8(q) for q in queries]
    offs = np.zeros(len(qs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([q.size for q in qs])
    cat = np.ascontiguousarray(np.concatenate(qs) if qs else np.zeros(0, np.uint8))
    return cat, offs


def sw_search_batch(queries, matrix, gap_open: int, gap_extend: int) -> np.ndarray:
    """Scores of every query (list of uint8 arrays) -> int32[nq, count]."""
    cat, offs = _pack_queries(queries)
    m = _matrix(matrix)
    n = sw_db_count()
    out = np.empty((len(queries), n), dtype=np.int32)
    _check(load_library().sw_search_batch(_ptr(cat), _ptr(offs), len(queries), _ptr(m), int(gap_open),
                                          int(gap_extend), _ptr(out)))
    return out


def sw_search_batch_dev(queries, matrix, gap_open: int, gap_extend: int, d_scores, stream=None) -> None:
    cat, offs = _pack_queries(queries)
    m = _matrix(matrix)
    _check(load_library().sw_search_batch_dev(_ptr(cat), _ptr(offs), len(queries), _ptr(m), int(gap_open),
                                              int(gap_extend), _dev_ptr(d_scores), _stream_ptr(stream)))


def sw_topk(k: int):
    n = max(0, min(int(k), sw_db_count()))
    idx = np.empty(max(n, 1), dtype=np.int64)
    sc = np.empty(max(n, 1), dtype=np.int32)
    r = _check(load_library().sw_topk(int(k), _ptr(idx), _ptr(sc)))
    return idx[:r], sc[:r]


def sw_topk_dev(d_scores, d_index, n: int, k: int, d_idx_out, d_score_out, stream=None) -> int:
    return int(_check(load_library().sw_topk_dev(_dev_ptr(d_scores), _dev_ptr(d_index), int(n), int(k),
                                                 _dev_ptr(d_idx_out), _dev_ptr(d_score_out),
                                                 _stream_ptr(stream))))


def sw_scatter_dev(d_src, d_index, n: int, d_dst, dst_count: int, stream=None) -> None:
    """d_dst[d_index[i]] = d_src[i] on the device (negative index = padding)."""
    _check(load_library().sw_scatter_dev(_dev_ptr(d_src), _dev_ptr(d_index), int(n), _dev_ptr(d_dst),
                                         int(dst_count), _stream_ptr(stream)))


def sw_last_stats() -> dict:
    a = np.zeros(14, dtype=np.int64)
    _check(load_library().sw_last_stats(_ptr(a), 14))
    keys = ["rows_per_pass", "passes", "G", "R", "flagged", "cells32", "pair_columns", "items",
            "flag_threshold", "arith", "wave", "lat", "profile", "rows_pairs"]
    return {k: int(v) for k, v in zip(keys, a)}


def sw_last_timing() -> dict:
    a = np.zeros(2, dtype=np.float32)
    _check(load_library().sw_last_timing(_ptr(a), 2))
    return {"pass_kernels_ms": float(a[0]), "search_ms": float(a[1])}


def sw_timing_history(n: int) -> list:
    """Pass-kernel ms of each of the last n searches, oldest first (swdb.h)."""
    a = np.zeros(max(int(n), 1), dtype=np.float32)
    k = _check(load_library().sw_timing_history(_ptr(a), int(n)))
    return [float(x) for x in a[:k]]


def sw_set_tile(G: int, R: int = 0) -> None:
    _check(load_library().sw_set_tile(int(G), int(R)))


def sw_set_wave(mode: int) -> None:
    """Cross-pass wavefront: 0 auto (default), 1 always, -1 never (swdb.h)."""
    _check(load_library().sw_set_wave(int(mode)))


def sw_set_latency_mode(mode: int) -> None:
    """Low-latency (LAT) tiles: 0 auto (default), 1 always, -1 never (swdb.h)."""
    _check(load_library().sw_set_latency_mode(int(mode)))


def sw_set_rows_mode(mode: int) -> None:
    """Rows mode for the long sequences: 0 auto (default), 1 whenever possible, -1 never (swdb.h)."""
    _check(load_library().sw_set_rows_mode(int(mode)))


def sw_set_profile(mode: int) -> None:
    """Substitution scores: 0 auto (default), 1 query profile, 2 score profile (swdb.h)."""
    _check(load_library().sw_set_profile(int(mode)))


def sw_tile_supported(G: int, R: int, lat: bool = False, sp: bool = False) -> bool:
    """Whether (G, R) is a compiled throughput tile, latency tile (lat=True) or
    score-profile tile (sp=True)."""
    return bool(load_library().sw_tile_supported(int(G), int(R)) & (4 if sp else (2 if lat else 1)))
