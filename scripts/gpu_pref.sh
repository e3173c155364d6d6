timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pref_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pref_pytest.log
LIBS="_lib_np _lib _lib_p288" ARGS="--steps 5 --warmup 3 --degree 5 --degrees 4,6,7 --no-cpu-baseline --e2e-steps 1" bash scripts/gpu_ab.sh
