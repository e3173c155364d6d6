#!/bin/bash
# thread-per-(wedge, slice) N = 1 kernel (PDG_WEDGE_SL=1): parity, racecheck, same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
PDG_WEDGE_SL=1 timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_parity_sizes.py \
  tests/test_gpu_edge_cases.py tests/test_gpu_acceptance.py -k "1" > gpurun_out/sl_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/sl_pytest.log
PDG_WEDGE_SL=1 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python scripts/racecheck_stage.py 1 exact 20 2,2,2 > gpurun_out/sl_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/sl_racecheck.log
PDG_WEDGE_SL=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python scripts/racecheck_stage.py 1 exact 20 2,2,2 > gpurun_out/sl_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/sl_memcheck.log
bash scripts/ab_bench.sh gpurun_out/sl_ab.jsonl "main env:PDG_WEDGE_SL=1" "1" 3
bash scripts/ab_bench.sh gpurun_out/sl_hyb.jsonl "main env:PDG_WEDGE_SL=1" "1" 2 --workload hybrid
