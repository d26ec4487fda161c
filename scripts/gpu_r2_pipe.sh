# k_explore pipelined quad path (cp.async col stages, one batch ahead) vs the queue version
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_pipe_rmat24.log "pipe0|variants/libs3bfs_pipe0.so|{}" "pipe|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_pipe_rmat20.log "pipe0|variants/libs3bfs_pipe0.so|{}" "pipe|$L|{}"
ROUNDS=2 bash scripts/abx.sh er 8 gpurun_out/r2_pipe_er.log "pipe0|variants/libs3bfs_pipe0.so|{}" "pipe|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_pipe_*.log
grep -A3 "x/pipe " gpurun_out/r2_pipe_rmat24.log | tail -4
