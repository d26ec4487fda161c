"""Seeded synthetic CSR inputs shared by the CUDA path's tests/bench and the oracle.

This module holds none of the method's arithmetic: it only builds graphs (C++,
``graphgen.cpp``) and picks sources.  The five BASELINE.json workloads are
``CONFIGS``; DESIGN.md "Input recipe" states each recipe and the readings it takes.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "graphgen.cpp")
_LIB = os.path.join(_HERE, "libgraphgen.so")
_lib = None
_P32 = ctypes.POINTER(ctypes.c_int32)

RMAT_ABC = (0.57, 0.19, 0.19)  # d = 0.05 (BASELINE.json configs[2..4])


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        vp = ctypes.c_void_p
        lib.gg_last_error.restype = ctypes.c_char_p
        lib.gg_n.argtypes = [vp]; lib.gg_n.restype = ctypes.c_int32
        lib.gg_nnz.argtypes = [vp]; lib.gg_nnz.restype = ctypes.c_int64
        lib.gg_meta.argtypes = [vp, ctypes.c_int]; lib.gg_meta.restype = ctypes.c_int64
        lib.gg_copy.argtypes = [vp, ctypes.c_void_p, ctypes.c_void_p]; lib.gg_copy.restype = None
        lib.gg_free.argtypes = [vp]; lib.gg_free.restype = None
        lib.gg_from_edges.argtypes = [ctypes.c_int32, ctypes.c_int64, _P32, _P32, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int]
        lib.gg_from_edges.restype = vp
        lib.gg_er.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int]
        lib.gg_er.restype = vp
        lib.gg_grid.argtypes = [ctypes.c_int32, ctypes.c_int32]; lib.gg_grid.restype = vp
        lib.gg_rmat.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                ctypes.c_double, ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        lib.gg_rmat.restype = vp
        lib.gg_rmat_tail.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_uint64, ctypes.c_double,
                                     ctypes.c_int32, ctypes.c_int]
        lib.gg_rmat_tail.restype = vp
        lib.gg_pick_sources.argtypes = [ctypes.c_int32, _P32, _P32, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_uint64, _P32]
        lib.gg_pick_sources.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclasses.dataclass
class Graph:
    """int32 CSR out-adjacency.  ``meta`` carries generator facts (e.g. the tail's far end)."""
    name: str
    row_offsets: np.ndarray
    col_indices: np.ndarray
    meta: dict
    sources: list

    @property
    def n(self) -> int:
        return int(self.row_offsets.size - 1)

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)


def _take(ptr, name: str, out_ro=None, out_col=None) -> Graph:
    lib = _load()
    if not ptr:
        raise RuntimeError(f"graphgen {name}: {lib.gg_last_error().decode()}")
    try:
        n, nnz = lib.gg_n(ptr), lib.gg_nnz(ptr)
        ro = out_ro if out_ro is not None else np.empty(n + 1, np.int32)
        col = out_col if out_col is not None else np.empty(nnz, np.int32)
        lib.gg_copy(ptr, ro.ctypes.data, col.ctypes.data)
        meta = {k: int(lib.gg_meta(ptr, i)) for i, k in
                enumerate(["m0", "m1", "m2", "m3", "m4", "m5", "m6", "m7"])}
    finally:
        lib.gg_free(ptr)
    return Graph(name, ro, col, meta, [])


def from_edges(n: int, edges, symmetrize: bool = True, dedup: bool = False,
               drop_self_loops: bool = False, name: str = "edges") -> Graph:
    """CSR from an explicit edge list (multigraph kept unless dedup)."""
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    u = np.ascontiguousarray(e[:, 0]) if e.size else np.zeros(1, np.int32)
    v = np.ascontiguousarray(e[:, 1]) if e.size else np.zeros(1, np.int32)
    ptr = _load().gg_from_edges(int(n), int(e.shape[0]), u.ctypes.data_as(_P32),
                                v.ctypes.data_as(_P32), int(symmetrize), int(dedup),
                                int(drop_self_loops))
    return _take(ptr, name)


def er(n: int = 1 << 16, m: int = 1 << 19, seed: int = 1, threads: int = 0) -> Graph:
    return _take(_load().gg_er(n, m, seed, threads), "er")


def grid(rows: int = 1024, cols: int = 1024) -> Graph:
    return _take(_load().gg_grid(rows, cols), "grid")


def rmat(scale: int, ef: int = 16, seed: int = 2, abc=RMAT_ABC, permute: bool = True,
         threads: int = 0) -> Graph:
    a, b, c = abc
    return _take(_load().gg_rmat(scale, ef, a, b, c, seed, int(permute), threads), f"rmat{scale}")


def rmat_tail(scale: int = 22, ef: int = 16, seed: int = 4, abc=RMAT_ABC, extra_frac: float = 0.01,
              path_len: int = 20000, threads: int = 0) -> Graph:
    a, b, c = abc
    g = _take(_load().gg_rmat_tail(scale, ef, a, b, c, seed, extra_frac, path_len, threads), "tail")
    g.meta = {"anchor": g.meta["m0"], "path_first": g.meta["m1"], "far_end": g.meta["m2"],
              "giant_rmat": g.meta["m3"]}
    return g


def pick_sources(g: Graph, count: int, seed: int, mode: str = "nonisolated") -> list:
    """Distinct seeded sources: 'nonisolated' (deg > 0) or 'largest_cc'."""
    out = np.empty(max(count, 1), np.int32)
    got = _load().gg_pick_sources(g.n, g.row_offsets.ctypes.data_as(_P32),
                                  g.col_indices.ctypes.data_as(_P32) if g.nnz else _P32(),
                                  {"nonisolated": 0, "largest_cc": 1}[mode], count, seed,
                                  out.ctypes.data_as(_P32))
    if got < 0:
        raise RuntimeError(_load().gg_last_error().decode())
    return [int(x) for x in out[:got]]


# --- the five BASELINE.json workloads -------------------------
SOURCE_SEED = 7  # seed of the source-selection stream (separate from every edge stream)


def make_config(name: str, threads: int = 0) -> Graph:
    if name == "er":          # configs[0]
        g = er(1 << 16, 1 << 19, seed=1, threads=threads)
        g.sources = pick_sources(g, 8, SOURCE_SEED, "largest_cc")
    elif name == "grid":      # configs[1]
        g = grid(1024, 1024)
        g.sources = [0, 512 * 1024 + 512]
    elif name == "rmat20":    # configs[2]
        g = rmat(20, 16, seed=2, threads=threads)
        g.sources = pick_sources(g, 16, SOURCE_SEED, "nonisolated")
    elif name == "rmat24":    # configs[3]
        g = rmat(24, 16, seed=3, threads=threads)
        g.sources = pick_sources(g, 16, SOURCE_SEED, "nonisolated")
    elif name == "tail":      # configs[4]
        g = rmat_tail(22, 16, seed=4, threads=threads)
        g.sources = [g.meta["far_end"]] + pick_sources(g, 8, SOURCE_SEED, "largest_cc")
    else:
        raise KeyError(name)
    g.name = name
    return g


CONFIG_NAMES = ("er", "grid", "rmat20", "rmat24", "tail")
