"""B200-native S3BFS frontier-expansion path (arxiv 2209.08764), sm_100a CUDA behind a C ABI.

The package holds only the path: ``csrc/`` (kernels + C ABI, see ``include/s3bfs.h``) and the
ctypes binding ``s3bfs``.  It never imports ``oracle/`` (test infrastructure).
"""
from .s3bfs import (EXPORTED, LIB_PATH, LevelStat, Options, S3BFS, S3BFSError, load,  # noqa: F401
                    s3bfs_clone, s3bfs_create, s3bfs_debug_exclusive_scan, s3bfs_debug_find_start_points,
                    s3bfs_destroy, s3bfs_get_info, s3bfs_get_kernel_times, s3bfs_get_level_stats, s3bfs_run,
                    s3bfs_run_ptr, s3bfs_status_string)
from .dist import DistRank, traverse  # noqa: F401,E402  (NEXT-4)
