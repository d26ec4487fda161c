# R28 owner-partitioned levels: parity subset, then A/B against the bitmap/tag path
set -x
mkdir -p gpurun_out
python -c "from paper_2209_08764_b200 import build as b; b.build(force=True)" > gpurun_out/px_build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "owner_partitioned or px or graph-default" > gpurun_out/px_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/px_pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "configs" > gpurun_out/px_pytest_cfg.log 2>&1; echo pytest_cfg_rc=$?
tail -5 gpurun_out/px_pytest_cfg.log
for cfg in rmat24 rmat20 er; do
  VARIANT_OUT=/dev/null VARIANT_OPTS='{"px": {}, "off": {"owner_partition": -1}}' ROUNDS=2 timeout 600 \
    python scripts/variants.py $cfg 8 cur=paper_2209_08764_b200/libs3bfs.so > gpurun_out/px_ab_$cfg.log 2>&1
  cat gpurun_out/px_ab_$cfg.log
done
