#!/bin/bash
# WADG pre-lift mbarrier exchange (wmb) and tet slot parity (tsp): parity, racecheck, same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/wmb/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_wadg.py \
  tests/test_gpu_parity_sizes.py -k "wadg or config2_copy" > gpurun_out/mb2_pytest_wmb.log 2>&1
echo "rc=$?" >> gpurun_out/mb2_pytest_wmb.log
PDG_LIB_PATH=$V/tsp/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py \
  tests/test_gpu_parity_sizes.py tests/test_gpu_edge_cases.py > gpurun_out/mb2_pytest_tsp.log 2>&1
echo "rc=$?" >> gpurun_out/mb2_pytest_tsp.log
PDG_LIB_PATH=$V/wmb/libprismdg_b200.so timeout 900 compute-sanitizer --tool racecheck \
  --error-exitcode 9 python scripts/racecheck_stage.py 5 wadg 20 2,2,2 > gpurun_out/mb2_racecheck_wmb.log 2>&1
echo "rc=$?" >> gpurun_out/mb2_racecheck_wmb.log
bash scripts/ab_bench.sh gpurun_out/mb2_wadg.jsonl "main wmb" "5 4 6 7" 2 --mass wadg
bash scripts/ab_bench.sh gpurun_out/mb2_tet.jsonl "main tsp" "4 3 5" 2 --workload hybrid
bash scripts/ab_bench.sh gpurun_out/mb2_n6.jsonl "main noend6 mbn6" "6 5" 2
