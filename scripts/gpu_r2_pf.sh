# k_explore L2 prefetch variants (next batch of a long row / first sector of every window row)
mkdir -p gpurun_out
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_pf_rmat24.log "base|$L|{}" "pf1|variants/libs3bfs_pf1.so|{}" "pf2|variants/libs3bfs_pf2.so|{}" "pf3|variants/libs3bfs_pf3.so|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_pf_rmat20.log "base|$L|{}" "pf1|variants/libs3bfs_pf1.so|{}" "pf2|variants/libs3bfs_pf2.so|{}" "pf3|variants/libs3bfs_pf3.so|{}"
python scripts/abx_summary.py gpurun_out/r2_pf_*.log
grep -A3 "x/pf3" gpurun_out/r2_pf_rmat24.log | tail -4
