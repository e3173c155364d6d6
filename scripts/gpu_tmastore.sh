timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_ab3.py tests/test_gpu_edge_cases.py -q -x -p no:cacheprovider > gpurun_out/ts_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/ts_pytest.log
LIBS="_lib_old _lib" ARGS="--steps 5 --warmup 3 --degree 5 --degrees 4,6,7 --no-cpu-baseline --e2e-steps 1" bash scripts/gpu_ab.sh
