# k_small CTA size: 1024 (default) vs 512 / 256 threads
mkdir -p gpurun_out
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh grid 2 gpurun_out/r2_kst_grid.log "t1024|$L|{}" "t512|variants/libs3bfs_ks512.so|{}" "t256|variants/libs3bfs_ks256.so|{}"
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_kst_er.log "t1024|$L|{}" "t512|variants/libs3bfs_ks512.so|{}" "t256|variants/libs3bfs_ks256.so|{}"
ROUNDS=2 bash scripts/abx.sh tail 4 gpurun_out/r2_kst_tail.log "t1024|$L|{}" "t512|variants/libs3bfs_ks512.so|{}" "t256|variants/libs3bfs_ks256.so|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_kst_rmat20.log "t1024|$L|{}" "t512|variants/libs3bfs_ks512.so|{}" "t256|variants/libs3bfs_ks256.so|{}"
python scripts/abx_summary.py gpurun_out/r2_kst_*.log
grep "x/" gpurun_out/r2_kst_grid.log | head -6
