# k_explore warp queue as a ring (no tail move after a flush) vs the moving queue (HEAD)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_ring_rmat24.log "head|variants/libs3bfs_head.so|{}" "ring|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_ring_rmat20.log "head|variants/libs3bfs_head.so|{}" "ring|$L|{}"
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_ring_er.log "head|variants/libs3bfs_head.so|{}" "ring|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_ring_*.log
grep -A2 "x/ring" gpurun_out/r2_ring_rmat24.log | tail -3
