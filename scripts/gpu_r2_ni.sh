# k_small / k_cluster: per-level item-count guards (a small level pays for its own edges only)
# vs HEAD; and the TAIL tiny path vs the fa049bf build (regression check on one box)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh grid 2 gpurun_out/r2_ni_grid.log "pre|variants/libs3bfs_pre_ni.so|{}" "ni|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
ROUNDS=3 bash scripts/abx.sh tail 4 gpurun_out/r2_ni_tail.log "pre|variants/libs3bfs_pre_ni.so|{}" "ni|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_ni_er.log "pre|variants/libs3bfs_pre_ni.so|{}" "ni|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_ni_rmat20.log "pre|variants/libs3bfs_pre_ni.so|{}" "ni|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
python scripts/abx_summary.py gpurun_out/r2_ni_*.log
timeout 900 python -m pytest tests/test_dist.py -m gpu -x -q 2>&1 | tail -2
