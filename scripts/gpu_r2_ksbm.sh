# k_small: visited bitmap staged on chip (n <= 2^20) vs probed in L2; plus T0 = 4096 on GRID
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
B=variants/libs3bfs_ksbm0.so
ROUNDS=3 bash scripts/abx.sh grid 2 gpurun_out/r2_ksbm_grid.log "bm0|$B|{}" "bm|$L|{}" "bm-T0-4096|$L|{\"tier0_max_edges\": 4096}" "bm-T0-1024|$L|{\"tier0_max_edges\": 1024}"
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_ksbm_er.log "bm0|$B|{}" "bm|$L|{}" "bm-T0-4096|$L|{\"tier0_max_edges\": 4096}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_ksbm_rmat20.log "bm0|$B|{}" "bm|$L|{}" "bm-T0-4096|$L|{\"tier0_max_edges\": 4096}"
python scripts/abx_summary.py gpurun_out/r2_ksbm_*.log
