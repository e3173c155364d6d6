#!/bin/bash
# round-2 GPU check: full GPU suite, a short headline bench, the reference arm
cd "$GRAFT_REPO_ROOT" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --degrees "" > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
lscpu > gpurun_out/r2_lscpu.txt
