# k_explore queue capacity (flush check every group: 64 entries) and the L1-preferring carve-out
mkdir -p gpurun_out
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_kq_rmat24.log "kq2|$L|{}" "kq1|variants/libs3bfs_kq1.so|{}" "maxl1|variants/libs3bfs_maxl1.so|{}" "maxl1kq1|variants/libs3bfs_maxl1kq1.so|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_kq_rmat20.log "kq2|$L|{}" "kq1|variants/libs3bfs_kq1.so|{}" "maxl1|variants/libs3bfs_maxl1.so|{}" "maxl1kq1|variants/libs3bfs_maxl1kq1.so|{}"
ROUNDS=2 bash scripts/abx.sh er 8 gpurun_out/r2_kq_er.log "kq2|$L|{}" "kq1|variants/libs3bfs_kq1.so|{}" "maxl1|variants/libs3bfs_maxl1.so|{}" "maxl1kq1|variants/libs3bfs_maxl1kq1.so|{}"
python scripts/abx_summary.py gpurun_out/r2_kq_*.log
