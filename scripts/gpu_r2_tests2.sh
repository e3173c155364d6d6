#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 1500 python -m pytest tests/test_gpu_mrab.py tests/test_gpu_config4.py -q --durations=10 > gpurun_out/r2_tests2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_tests2.log
