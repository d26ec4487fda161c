# k_compact: one-round-trip prefix over all predecessor tiles vs the chained look-back
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_lb_er.log "lb0|variants/libs3bfs_lb0.so|{}" "wide|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_lb_rmat20.log "lb0|variants/libs3bfs_lb0.so|{}" "wide|$L|{}"
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_lb_rmat24.log "lb0|variants/libs3bfs_lb0.so|{}" "wide|$L|{}"
ROUNDS=2 bash scripts/abx.sh tail 4 gpurun_out/r2_lb_tail.log "lb0|variants/libs3bfs_lb0.so|{}" "wide|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_lb_*.log
