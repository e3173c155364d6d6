mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wadg.py -q -p no:cacheprovider > gpurun_out/wadg_pytest.log 2>&1; echo "pytest exit $?"; grep -E "passed|failed|Error|assert" gpurun_out/wadg_pytest.log | tail -30
