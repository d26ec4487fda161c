# compute-sanitizer evidence (tiny suite + R-MAT 14, every tier setting) and a source-level
# ncu capture of k_explore/k_compact on R-MAT 24 (host loop, source index 0)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for t in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tests/sanitize_suite.py --quick > gpurun_out/san_$t.log 2>&1
  echo ${t}_rc=$?; tail -4 gpurun_out/san_$t.log
done
python scripts/prof_run.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_explore|k_compact" -c 5 \
    -o gpurun_out/r2_prof_src0 -f python scripts/prof_run.py > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
