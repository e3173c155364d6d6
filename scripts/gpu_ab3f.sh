#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_ab3_fused.py tests/test_ab3.py tests/test_gpu_mrab.py -q > gpurun_out/ab3f_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ab3f_pytest.log
timeout 900 python scripts/integrator_rates.py > gpurun_out/ab3f_integrators.json 2> gpurun_out/ab3f_integrators.err
