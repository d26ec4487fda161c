mkdir -p gpurun_out
python scripts/dbg_small.py variants/libs3bfs_check.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -5 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=2 bash scripts/abx.sh rmat24 8 gpurun_out/r2_kc_rmat24.log "r01|variants/libs3bfs_r01.so|{}" "modes|variants/libs3bfs_modes.so|{\"hub_vertices\": 524288}" "chunk|variants/libs3bfs_chunk.so|{}" "cur|$L|{}"
ROUNDS=1 bash scripts/abx.sh rmat20 8 gpurun_out/r2_kc_rmat20.log "r01|variants/libs3bfs_r01.so|{}" "modes|variants/libs3bfs_modes.so|{\"hub_vertices\": 524288}" "cur|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_kc_*.log
python scripts/prof_run.py > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_explore|k_compact" -c 8 -f -o gpurun_out/r2_prof_chunk \
    python scripts/prof_run.py > gpurun_out/r2_ncu_full.log 2>&1
echo full_rc=$?
