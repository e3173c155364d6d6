mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab3_pytest.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/ab3_pytest.log | grep -E "passed|failed|Error|assert|^E" | head -20
timeout 900 python bench.py > gpurun_out/bench_default_r1b.json 2> gpurun_out/bench_default_r1b.err; echo "bench $?"; cat gpurun_out/bench_default_r1b.json
