# k_explore<false> (no NEXT-4 code in the single-GPU kernel) vs 2b2c007 and fa049bf builds
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_tpl_rmat24.log "head2b2c|variants/libs3bfs_pre_ni.so|{}" "tpl|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_tpl_rmat20.log "head2b2c|variants/libs3bfs_pre_ni.so|{}" "tpl|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_tpl_er.log "head2b2c|variants/libs3bfs_pre_ni.so|{}" "tpl|$L|{}" "fa049bf|variants/libs3bfs_fa049bf.so|{}"
python scripts/abx_summary.py gpurun_out/r2_tpl_*.log
