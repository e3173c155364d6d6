#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
# memcheck / racecheck of the round-2 device paths (multi-rate AB3 update, owned-only finite scan, set_rhs)
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_mrab.py -q -x -k "single_level or levels_and_steps_match_oracle" > gpurun_out/misc1_memcheck_mrab.log 2>&1
echo "rc=$?" >> gpurun_out/misc1_memcheck_mrab.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_shim.py tests/test_gpu_partition.py -q -x > gpurun_out/misc1_memcheck_shim.log 2>&1
echo "rc=$?" >> gpurun_out/misc1_memcheck_shim.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_mrab.py -q -x -k "levels_and_steps_match_oracle" > gpurun_out/misc1_racecheck_mrab.log 2>&1
echo "rc=$?" >> gpurun_out/misc1_racecheck_mrab.log
# DMMA kernel at the low orders (PDG_WEDGE_KERNEL=d) vs the CUDA-core kernel
bash scripts/ab_bench.sh gpurun_out/misc1_lo_ab.jsonl "main env:PDG_WEDGE_KERNEL=d" "2 3" 2
