timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/nts_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/nts_pytest.log | grep -E "passed|failed|Error|^E"
python -c "import __graft_entry__ as g; g.smoke()"
LIBS="_lib_old _lib" ARGS="--steps 5 --warmup 3 --degree 5 --degrees 4,6 --no-cpu-baseline --e2e-steps 1" bash scripts/gpu_ab.sh
LIBS="_lib_old _lib" ARGS="--steps 5 --warmup 3 --degree 5 --degrees '' --mass wadg --no-cpu-baseline --e2e-steps 1" bash scripts/gpu_ab.sh
