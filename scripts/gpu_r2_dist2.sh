# NEXT-4 with tag mode (owner-side visited check) + GPU suite + loopback model; PDL removed
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py -m gpu -x -q > gpurun_out/r2_dist_tests.log 2>&1; rc=$?; echo "dist tests rc=$rc"; tail -15 gpurun_out/r2_dist_tests.log
[ $rc -eq 0 ] || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
timeout 900 python scripts/dist_loopback.py rmat20 4 2 4 > gpurun_out/r2_dist_loopback_rmat20.log 2>&1; cat gpurun_out/r2_dist_loopback_rmat20.log
timeout 1500 python scripts/dist_loopback.py rmat24 4 2 4 8 > gpurun_out/r2_dist_loopback_rmat24.log 2>&1; cat gpurun_out/r2_dist_loopback_rmat24.log
