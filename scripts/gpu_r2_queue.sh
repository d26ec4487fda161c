# k_explore warp queue (claim checks + discoveries resolved 32 at a time) vs the per-group path
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_queue_rmat24.log "q0|variants/libs3bfs_q0.so|{}" "queue|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_queue_rmat20.log "q0|variants/libs3bfs_q0.so|{}" "queue|$L|{}"
ROUNDS=2 bash scripts/abx.sh er 8 gpurun_out/r2_queue_er.log "q0|variants/libs3bfs_q0.so|{}" "queue|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_queue_*.log
grep src gpurun_out/r2_queue_rmat24.log | tail -6
