#!/bin/bash
# GPU suite (new tests first), results under gpurun_out/
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 1500 python -m pytest tests/test_gpu_shim.py tests/test_gpu_acceptance.py tests/test_gpu_partition.py -q --durations=15 > gpurun_out/r2_newtests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_newtests.log
