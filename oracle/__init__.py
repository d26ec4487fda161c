"""CPU oracle for the S3BFS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2209_08764_b200``) never imports it and shares no code with it.

The arithmetic lives in ``s3bfs_oracle.c`` (plain serial C, each function citing the
PAPER.md passage it follows); this module only marshals numpy arrays through ctypes.
Every function is pinned by ``tests/test_oracle_pins.py`` against brute force, closed
forms, SPEC worked examples or mutation tests -- never against itself.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "s3bfs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_P32 = ctypes.POINTER(ctypes.c_int32)
_P64 = ctypes.POINTER(ctypes.c_int64)


_NATIVE_LIB = os.path.join(_HERE, "liboracle_native.so")
_use_native = False


def build(force: bool = False, native: bool = False) -> str:
    """Compile liboracle.so (gcc -O3; portable, built wherever the tests run).  With native,
    liboracle_native.so with -O3 -march=native (SURVEY 8(d) D7's flags for the timed CPU
    baseline), built on the machine that runs it.  Building the checker is not using it."""
    lib = _NATIVE_LIB if native else _LIB
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
        tmp = lib + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", *(["-march=native"] if native else []), "-std=c11",
                               "-shared", "-fPIC", "-Wall", "-Wextra", "-o", tmp, _SRC])
        os.replace(tmp, lib)
    return lib


def use_native() -> str:
    """Switch this process to the -march=native build (bench.py's CPU baseline legs only).
    Returns the compiler flags in use."""
    global _use_native, _lib
    build(force=True, native=True)
    _use_native, _lib = True, None
    return "gcc -O3 -march=native -std=c11"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _load():
    global _lib
    if _lib is None:
        path = build(native=_use_native)
        lib = ctypes.CDLL(path)
        lib.oracle_bfs.argtypes = [ctypes.c_int32, _P32, _P32, ctypes.c_int32, _P32, _P32]
        lib.oracle_inclusive_scan.argtypes = [_P32, ctypes.c_int64, _P32]
        lib.oracle_exclusive_scan.argtypes = [_P32, ctypes.c_int64, _P32]
        lib.oracle_find_start_points.argtypes = [_P32, ctypes.c_int32, ctypes.c_int64,
                                                 ctypes.c_int32, _P32, _P32]
        lib.oracle_dedup_linearize.argtypes = [ctypes.c_int32, _P64, _P32, _P32, _P32, _P32, _P64]
        lib.oracle_s3bfs_fig1.argtypes = [ctypes.c_int32, _P32, _P32, ctypes.c_int32,
                                          ctypes.c_int32, _P32, ctypes.c_int32, _P64, _P64,
                                          _P64, _P32]
        lib.oracle_level_profile.argtypes = [ctypes.c_int32, _P32, _P32, ctypes.c_int32, _P64,
                                             _P64, _P32, _P64, _P64]
        lib.oracle_check_bfs.argtypes = [ctypes.c_int32, _P32, _P32, ctypes.c_int32, _P32, _P32,
                                         _P64]
        for f in ("oracle_bfs", "oracle_inclusive_scan", "oracle_exclusive_scan",
                  "oracle_find_start_points", "oracle_dedup_linearize", "oracle_s3bfs_fig1",
                  "oracle_level_profile", "oracle_check_bfs"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _p32(a: np.ndarray):
    return a.ctypes.data_as(_P32)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(_P64)


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise OracleError(f"{what} failed with code {rc}")


def bfs(row_offsets, col_indices, source: int):
    """Serial FIFO BFS. Returns (level, parent) int32 arrays, -1 = unreached."""
    ro, col = _i32(row_offsets), _i32(col_indices)
    n = ro.size - 1
    level = np.empty(n, np.int32)
    parent = np.empty(n, np.int32)
    col_p = _p32(col) if col.size else _P32()
    _check(_load().oracle_bfs(n, _p32(ro), col_p, int(source), _p32(level), _p32(parent)),
           "oracle_bfs")
    return level, parent


def inclusive_scan(values) -> np.ndarray:
    """Parallel-Prefix-Sum of Fig.1 L14 (inclusive)."""
    a = _i32(values)
    out = np.empty(a.size, np.int32)
    if a.size:
        _check(_load().oracle_inclusive_scan(_p32(a), a.size, _p32(out)), "inclusive_scan")
    return out


def exclusive_scan(values) -> np.ndarray:
    """Exclusive scan with total appended: n+1 entries, out[n] = e_l (R5)."""
    a = _i32(values)
    out = np.empty(a.size + 1, np.int32)
    inp = _p32(a) if a.size else _P32()
    _check(_load().oracle_exclusive_scan(inp, a.size, _p32(out)), "exclusive_scan")
    return out


def find_start_points(edge_sum_inclusive, chunk: int, p_l: int):
    """Find-StartExpPoint (Fig.1 L17) by the range rule of P:43-45.
    Returns (u, off) arrays of length p_l (-1 where no start exists)."""
    es = _i32(edge_sum_inclusive)
    u = np.empty(max(p_l, 1), np.int32)
    off = np.empty(max(p_l, 1), np.int32)
    es_p = _p32(es) if es.size else _P32()
    _check(_load().oracle_find_start_points(es_p, es.size, int(chunk), int(p_l), _p32(u),
                                            _p32(off)), "find_start_points")
    return u[:p_l], off[:p_l]


def dedup_linearize(queues, owner):
    """Fig.1 L19-L29: queues = list of lists; owner = array.  Returns (Sizes inclusive, frontier)."""
    p_l = len(queues)
    q_begin = np.zeros(p_l + 1, np.int64)
    for i, q in enumerate(queues):
        q_begin[i + 1] = q_begin[i] + len(q)
    items = _i32([v for q in queues for v in q] or [0])
    own = _i32(owner)
    sizes = np.empty(max(p_l, 1), np.int32)
    frontier = np.empty(max(int(q_begin[-1]), 1), np.int32)
    count = np.zeros(1, np.int64)
    _check(_load().oracle_dedup_linearize(p_l, _p64(q_begin), _p32(items), _p32(own),
                                          _p32(sizes), _p32(frontier), _p64(count)),
           "dedup_linearize")
    return sizes[:p_l], frontier[: int(count[0])]


def s3bfs_fig1(row_offsets, col_indices, source: int, P: int, max_levels: int | None = None):
    """Figure 1 end to end with P simulated workers.
    Returns (level, n_l, e_l, P_l) -- per-level arrays over the levels with n_l > 0."""
    ro, col = _i32(row_offsets), _i32(col_indices)
    n = ro.size - 1
    cap = max_levels if max_levels is not None else n + 1
    level = np.empty(n, np.int32)
    nl = np.zeros(cap, np.int64)
    el = np.zeros(cap, np.int64)
    pl = np.zeros(cap, np.int64)
    num = np.zeros(1, np.int32)
    col_p = _p32(col) if col.size else _P32()
    _check(_load().oracle_s3bfs_fig1(n, _p32(ro), col_p, int(source), int(P), _p32(level), cap,
                                     _p64(nl), _p64(el), _p64(pl), _p32(num)), "s3bfs_fig1")
    k = int(num[0])
    return level, nl[:k], el[:k], pl[:k]


def level_profile(row_offsets, level):
    """Per-level n_l, e_l (int64 arrays), and m_c, n_c."""
    ro, lv = _i32(row_offsets), _i32(level)
    n = ro.size - 1
    L = int(lv.max()) + 1 if lv.size else 0
    nl = np.zeros(max(L, 1), np.int64)
    el = np.zeros(max(L, 1), np.int64)
    num = np.zeros(1, np.int32)
    mc = np.zeros(1, np.int64)
    nc = np.zeros(1, np.int64)
    _check(_load().oracle_level_profile(n, _p32(ro), _p32(lv), max(L, 1), _p64(nl), _p64(el),
                                        _p32(num), _p64(mc), _p64(nc)), "level_profile")
    return nl[:L], el[:L], int(mc[0]), int(nc[0])


CHECK_CODES = {
    0: "ok",
    1: "source entry wrong",
    2: "parent out of range",
    3: "parent level is not level-1",
    4: "(parent, v) is not an arc",
    5: "arc (u,v) violates level[v] <= level[u]+1 / reachability",
    6: "unreached vertex has a parent or an invalid level",
}


def check_bfs(row_offsets, col_indices, source: int, level, parent):
    """Certificate.  Returns (code, bad_vertex); code 0 = valid."""
    ro, col = _i32(row_offsets), _i32(col_indices)
    lv, pa = _i32(level), _i32(parent)
    bad = np.zeros(1, np.int64)
    col_p = _p32(col) if col.size else _P32()
    rc = _load().oracle_check_bfs(ro.size - 1, _p32(ro), col_p, int(source), _p32(lv), _p32(pa),
                                  _p64(bad))
    if rc < 0:
        raise OracleError("check_bfs: invalid arguments")
    return int(rc), int(bad[0])
