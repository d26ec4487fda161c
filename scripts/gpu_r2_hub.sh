# Round-2 experiment: k_explore visited test split (hub ids via the bitmap, others via the tag).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2_gpu_tests.log
for cfg in rmat24 rmat20; do
VARIANT_OUT=gpurun_out/r2_hub_$cfg.json ROUNDS=2 VARIANT_OPTS='{"hub-all": {"hub_vertices": -1}, "hub-2^17": {"hub_vertices": 131072}, "hub-2^19": {"hub_vertices": 524288}, "hub-2^20": {"hub_vertices": 1048576}, "hub-2^21": {"hub_vertices": 2097152}, "hub-1": {"hub_vertices": 1}}' \
  timeout 900 python scripts/variants.py $cfg 4 cur=paper_2209_08764_b200/libs3bfs.so > gpurun_out/r2_hub_$cfg.log 2>&1
echo "$cfg rc=$?"
done
