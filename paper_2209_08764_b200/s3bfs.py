"""Thin ctypes binding over libs3bfs.so (include/s3bfs.h) -- argument marshalling only.

Every step of the traversal runs in the CUDA kernels of ``csrc/``; this module converts
torch tensors to device pointers and torch streams to ``cudaStream_t``.  There is no CPU
fallback: if the library is missing or fails to load, every call raises.
Names follow the C ABI (``s3bfs_create`` / ``s3bfs_run`` / ``s3bfs_destroy`` ...).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

# S3BFS_LIB selects another build of the same sources (the bounds-checked build of
# tests/check_suite.py); the default is the in-tree libs3bfs.so
LIB_PATH = os.environ.get("S3BFS_LIB", _build.LIB)
_lib = None

S3BFS_OK = 0
STATUS_NAMES = {0: "ok", 1: "invalid argument", 2: "unsupported", 3: "out of memory",
                4: "CUDA error", 5: "invalid CSR graph"}

EXPORTED = ("s3bfs_create", "s3bfs_clone", "s3bfs_run", "s3bfs_destroy", "s3bfs_status_string",
            "s3bfs_last_error", "s3bfs_get_level_stats", "s3bfs_get_info", "s3bfs_get_kernel_times",
            "s3bfs_debug_exclusive_scan", "s3bfs_debug_find_start_points", "s3bfs_debug_timeline",
            "s3bfs_dist_export", "s3bfs_dist_connect", "s3bfs_dist_begin", "s3bfs_dist_explore",
            "s3bfs_dist_dedup", "s3bfs_dist_advance", "s3bfs_dist_advance_flag", "s3bfs_dist_status",
            "s3bfs_dist_end")


class S3BFSError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}"
                         + (f" -- {detail}" if detail else ""))


class Options(ctypes.Structure):
    """s3bfs_options (zero = defaults)."""
    _fields_ = [("edges_per_cta", ctypes.c_int32), ("tier0_max_edges", ctypes.c_int32),
                ("loop_mode", ctypes.c_int32), ("collect_stats", ctypes.c_int32),
                ("validate_csr", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("max_ctas", ctypes.c_int32), ("debug_poison", ctypes.c_int32),
                ("time_kernels", ctypes.c_int32), ("reorder", ctypes.c_int32),
                ("direction", ctypes.c_int32), ("do_alpha", ctypes.c_int32),
                ("do_beta", ctypes.c_int32), ("dist_size", ctypes.c_int32),
                ("dist_rank", ctypes.c_int32), ("cluster_max_edges", ctypes.c_int32),
                ("hub_vertices", ctypes.c_int32), ("tag_mode_pct", ctypes.c_int32),
                ("split_min_edges", ctypes.c_int32), ("split_first_pct", ctypes.c_int32),
                ("split_passes", ctypes.c_int32)]


class DistPeer(ctypes.Structure):
    """s3bfs_dist_peer: a rank's exchange record (addresses + CUDA IPC handle)."""
    _fields_ = [("base", ctypes.c_uint64), ("recv", ctypes.c_uint64), ("rcnt", ctypes.c_uint64),
                ("rmeta", ctypes.c_uint64), ("rtot", ctypes.c_uint64), ("bm", ctypes.c_uint64),
                ("vinfo", ctypes.c_uint64),
                ("ipc", ctypes.c_uint8 * 64), ("ipc_valid", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("size", ctypes.c_int32), ("pad", ctypes.c_int32)]


class LevelStat(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("n_l", ctypes.c_int32), ("e_l", ctypes.c_int32),
                ("tier", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("candidates", ctypes.c_int32), ("kept", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("t_begin_ns", ctypes.c_uint64),
                ("t_end_ns", ctypes.c_uint64), ("t_explore_begin_ns", ctypes.c_uint64),
                ("t_explore_end_ns", ctypes.c_uint64)]


class KernelTimes(ctypes.Structure):
    _fields_ = [("explore_ms", ctypes.c_double), ("compact_ms", ctypes.c_double),
                ("small_ms", ctypes.c_double), ("bottom_up_ms", ctypes.c_double),
                ("explore_launches", ctypes.c_int32), ("compact_launches", ctypes.c_int32),
                ("small_launches", ctypes.c_int32), ("bottom_up_launches", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("num_sms", ctypes.c_int32), ("p_max", ctypes.c_int32),
                ("edges_per_cta", ctypes.c_int32), ("tier0_max_edges", ctypes.c_int32),
                ("kd_threads", ctypes.c_int32), ("kd_tile_edges", ctypes.c_int32),
                ("ksmall_threads", ctypes.c_int32), ("ksmall_max_frontier", ctypes.c_int32),
                ("td_chain", ctypes.c_int32), ("bu_chain", ctypes.c_int32),
                ("universal_body", ctypes.c_int32), ("prologue", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64)]


def load(build_if_missing: bool = True):
    """Load libs3bfs.so (building it in-tree first if absent/stale and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        try:
            _build.build()
        except Exception as exc:  # noqa: BLE001 -- fall through to the loud load failure
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libs3bfs.so missing and the build failed: {exc}") from exc
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libs3bfs.so not found at {LIB_PATH}: run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.s3bfs_create.argtypes = [ctypes.POINTER(vp), i32, i64, vp, vp, ctypes.POINTER(Options), vp]
    lib.s3bfs_run.argtypes = [vp, i32, vp, vp, vp]
    lib.s3bfs_clone.argtypes = [vp, ctypes.POINTER(vp), vp]
    lib.s3bfs_destroy.argtypes = [vp]
    lib.s3bfs_status_string.argtypes = [ctypes.c_int]
    lib.s3bfs_status_string.restype = ctypes.c_char_p
    lib.s3bfs_last_error.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p)]
    lib.s3bfs_get_level_stats.argtypes = [vp, ctypes.POINTER(LevelStat), i32, ctypes.POINTER(i32)]
    lib.s3bfs_get_info.argtypes = [vp, ctypes.POINTER(Info)]
    lib.s3bfs_get_kernel_times.argtypes = [vp, ctypes.POINTER(KernelTimes)]
    lib.s3bfs_debug_exclusive_scan.argtypes = [vp, vp, i32, vp]
    lib.s3bfs_debug_find_start_points.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    lib.s3bfs_debug_timeline.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    lib.s3bfs_dist_export.argtypes = [vp, ctypes.POINTER(DistPeer)]
    lib.s3bfs_dist_connect.argtypes = [vp, ctypes.POINTER(DistPeer), i32, i32]
    lib.s3bfs_dist_begin.argtypes = [vp, i32, vp, vp, vp]
    lib.s3bfs_dist_explore.argtypes = [vp, vp]
    lib.s3bfs_dist_dedup.argtypes = [vp, vp]
    lib.s3bfs_dist_advance.argtypes = [vp, vp, ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_int64)]
    lib.s3bfs_dist_advance_flag.argtypes = [vp, vp, vp]
    lib.s3bfs_dist_status.argtypes = [vp, vp, ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_int64)]
    lib.s3bfs_dist_end.argtypes = [vp, vp]
    for name in EXPORTED:
        if name != "s3bfs_status_string":
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _detail(handle) -> str:
    msg = ctypes.c_char_p()
    load().s3bfs_last_error(handle, ctypes.byref(msg))
    return (msg.value or b"").decode(errors="replace")


def _check(rc: int, where: str, handle=None) -> None:
    if rc != S3BFS_OK:
        raise S3BFSError(rc, where, _detail(handle))


def _ptr(t) -> int:
    """Device pointer of a CUDA tensor (raises for CPU tensors: no host fallback)."""
    if t is None:
        return 0
    if not t.is_cuda:
        raise ValueError("tensor must live on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return int(t.data_ptr())


def _stream(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def s3bfs_create(row_offsets, col_indices, options: Options | None = None, stream=None):
    """s3bfs_create over int32 device tensors (borrowed: keep them alive). Returns a handle."""
    import torch
    for name, t in (("row_offsets", row_offsets), ("col_indices", col_indices)):
        if t.dtype != torch.int32:
            raise ValueError(f"{name} must be int32")
    h = ctypes.c_void_p()
    n = row_offsets.numel() - 1
    nnz = col_indices.numel()
    opts = ctypes.byref(options) if options is not None else None
    col_p = _ptr(col_indices) if nnz else 0
    rc = load().s3bfs_create(ctypes.byref(h), n, nnz, _ptr(row_offsets), col_p, opts,
                             _stream(stream))
    _check(rc, "s3bfs_create")
    return h


def s3bfs_clone(handle, stream=None):
    """NEXT-2: a handle sharing `handle`'s prepared graph, with its own workspace."""
    h = ctypes.c_void_p()
    _check(load().s3bfs_clone(handle, ctypes.byref(h), _stream(stream)), "s3bfs_clone", handle)
    return h


def s3bfs_run(handle, source: int, level, parent, stream=None) -> None:
    """Enqueue Parallel-BFS(source); level/parent: int32 device tensors [n]."""
    _check(load().s3bfs_run(handle, int(source), _ptr(level), _ptr(parent), _stream(stream)),
           "s3bfs_run", handle)


def s3bfs_run_ptr(handle, source: int, level_ptr: int, parent_ptr: int, stream_ptr: int) -> None:
    """Raw-pointer form of s3bfs_run (for timed loops)."""
    _check(load().s3bfs_run(handle, int(source), level_ptr, parent_ptr, stream_ptr),
           "s3bfs_run", handle)


def s3bfs_destroy(handle) -> None:
    if handle:
        _check(load().s3bfs_destroy(handle), "s3bfs_destroy")


def s3bfs_status_string(status: int) -> str:
    return load().s3bfs_status_string(int(status)).decode()


def s3bfs_get_level_stats(handle, cap: int = 1 << 16, return_total: bool = False):
    """Per-level records of the last run as a numpy structured array.  The device keeps at
    most min(n + 1, 65536) records (and this call at most ``cap``): a deeper traversal returns
    the first records with a warning; ``return_total`` also returns the true level count."""
    buf = (LevelStat * cap)()
    num = ctypes.c_int32()
    _check(load().s3bfs_get_level_stats(handle, buf, cap, ctypes.byref(num)),
           "s3bfs_get_level_stats", handle)
    k = min(num.value, cap)
    dt = np.dtype([("level", "i4"), ("n_l", "i4"), ("e_l", "i4"), ("tier", "i4"),
                   ("grid", "i4"), ("candidates", "i4"), ("kept", "i4"), ("pad", "i4"),
                   ("t_begin_ns", "u8"), ("t_end_ns", "u8"), ("t_explore_begin_ns", "u8"),
                   ("t_explore_end_ns", "u8")])
    out = np.frombuffer(bytes(buf)[: k * ctypes.sizeof(LevelStat)], dtype=dt).copy()
    k = min(k, out.shape[0])
    if num.value > out.shape[0]:
        import warnings
        warnings.warn(f"s3bfs_get_level_stats: {num.value} levels, first {out.shape[0]} "
                      f"records kept", RuntimeWarning, stacklevel=2)
    return (out, int(num.value)) if return_total else out


def s3bfs_get_info(handle) -> dict:
    info = Info()
    _check(load().s3bfs_get_info(handle, ctypes.byref(info)), "s3bfs_get_info", handle)
    return {f: getattr(info, f) for f, _ in Info._fields_}


def s3bfs_get_kernel_times(handle) -> dict:
    kt = KernelTimes()
    _check(load().s3bfs_get_kernel_times(handle, ctypes.byref(kt)), "s3bfs_get_kernel_times",
           handle)
    return {f: getattr(kt, f) for f, _ in KernelTimes._fields_}


def s3bfs_debug_exclusive_scan(inp, out, stream=None) -> None:
    n = inp.numel()
    if out.numel() != n + 1:
        raise ValueError("out must have n+1 entries")
    _check(load().s3bfs_debug_exclusive_scan(_ptr(inp) if n else 0, _ptr(out), n,
                                             _stream(stream)), "s3bfs_debug_exclusive_scan")


def s3bfs_debug_find_start_points(excl, chunk: int, p_l: int, out_u, out_off,
                                  stream=None) -> None:
    n_l = excl.numel() - 1
    _check(load().s3bfs_debug_find_start_points(_ptr(excl), n_l, int(chunk), int(p_l),
                                                _ptr(out_u), _ptr(out_off), _stream(stream)),
           "s3bfs_debug_find_start_points")


def s3bfs_debug_timeline(handle) -> list:
    out = (ctypes.c_uint64 * 4)()
    _check(load().s3bfs_debug_timeline(handle, out), "s3bfs_debug_timeline", handle)
    return list(out)


# ---- NEXT-4: one traversal over G ranks, 1-D vertex partition (include/s3bfs.h) ----------
def s3bfs_dist_export(handle) -> DistPeer:
    out = DistPeer()
    _check(load().s3bfs_dist_export(handle, ctypes.byref(out)), "s3bfs_dist_export", handle)
    return out


def s3bfs_dist_connect(handle, peers, use_ipc: bool) -> None:
    arr = (DistPeer * len(peers))(*peers)
    _check(load().s3bfs_dist_connect(handle, arr, len(peers), 1 if use_ipc else 0),
           "s3bfs_dist_connect", handle)


def s3bfs_dist_begin(handle, source: int, level, parent, stream=None) -> None:
    _check(load().s3bfs_dist_begin(handle, int(source), _ptr(level), _ptr(parent), _stream(stream)),
           "s3bfs_dist_begin", handle)


def s3bfs_dist_explore(handle, stream=None) -> None:
    _check(load().s3bfs_dist_explore(handle, _stream(stream)), "s3bfs_dist_explore", handle)


def s3bfs_dist_dedup(handle, stream=None) -> None:
    _check(load().s3bfs_dist_dedup(handle, _stream(stream)), "s3bfs_dist_dedup", handle)


def s3bfs_dist_advance(handle, stream=None, wait: bool = True):
    """Advance the level; with wait: (done, next frontier size over all ranks) after a sync."""
    if not wait:
        _check(load().s3bfs_dist_advance(handle, _stream(stream), None, None),
               "s3bfs_dist_advance", handle)
        return None
    done, n_next = ctypes.c_int32(), ctypes.c_int64()
    _check(load().s3bfs_dist_advance(handle, _stream(stream), ctypes.byref(done),
                                     ctypes.byref(n_next)), "s3bfs_dist_advance", handle)
    return bool(done.value), int(n_next.value)


def s3bfs_dist_advance_flag(handle, flag_ptr: int, stream=None) -> None:
    """Enqueue the advance; it writes -1 (done) or the next frontier size into *flag_ptr (an
    int64 the device can write, e.g. pinned host memory)."""
    _check(load().s3bfs_dist_advance_flag(handle, _stream(stream), ctypes.c_void_p(int(flag_ptr))),
           "s3bfs_dist_advance_flag", handle)


def s3bfs_dist_status(handle, stream=None):
    """(done, next frontier size over all ranks) of the last advance; synchronises."""
    done, n_next = ctypes.c_int32(), ctypes.c_int64()
    _check(load().s3bfs_dist_status(handle, _stream(stream), ctypes.byref(done),
                                    ctypes.byref(n_next)), "s3bfs_dist_status", handle)
    return bool(done.value), int(n_next.value)


def s3bfs_dist_end(handle, stream=None) -> None:
    _check(load().s3bfs_dist_end(handle, _stream(stream)), "s3bfs_dist_end", handle)


class S3BFS:
    """Convenience owner of a handle over device CSR tensors (kept alive here)."""

    def __init__(self, row_offsets, col_indices, options: Options | None = None, stream=None):
        self.row_offsets = row_offsets
        self.col_indices = col_indices
        self.n = row_offsets.numel() - 1
        self.handle = s3bfs_create(row_offsets, col_indices, options, stream)

    def run(self, source: int, level=None, parent=None, stream=None):
        import torch
        dev = self.row_offsets.device
        if level is None:
            level = torch.empty(self.n, dtype=torch.int32, device=dev)
        if parent is None:
            parent = torch.empty(self.n, dtype=torch.int32, device=dev)
        s3bfs_run(self.handle, source, level, parent, stream)
        return level, parent

    def clone(self, stream=None) -> "S3BFS":
        """NEXT-2: another traversal context over the same prepared graph."""
        c = S3BFS.__new__(S3BFS)
        c.row_offsets, c.col_indices, c.n = self.row_offsets, self.col_indices, self.n
        c.handle = s3bfs_clone(self.handle, stream)
        return c

    def level_stats(self) -> np.ndarray:
        return s3bfs_get_level_stats(self.handle)

    def info(self) -> dict:
        return s3bfs_get_info(self.handle)

    def close(self) -> None:
        if self.handle:
            s3bfs_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
