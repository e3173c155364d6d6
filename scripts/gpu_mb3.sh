#!/bin/bash
# tet end-of-batch mbarrier (tmb) and N=5 MB + volume-first (mbvf): parity, racecheck, same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/tmb/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py \
  tests/test_gpu_parity_sizes.py tests/test_gpu_edge_cases.py > gpurun_out/mb3_pytest_tmb.log 2>&1
echo "rc=$?" >> gpurun_out/mb3_pytest_tmb.log
PDG_LIB_PATH=$V/tmb/libprismdg_b200.so timeout 900 compute-sanitizer --tool racecheck \
  --error-exitcode 9 python scripts/racecheck_hybrid.py 4 16 2 8 > gpurun_out/mb3_racecheck_tmb.log 2>&1
echo "rc=$?" >> gpurun_out/mb3_racecheck_tmb.log
PDG_LIB_PATH=$V/mbvf/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  -k "config2_copy or full_size" > gpurun_out/mb3_pytest_mbvf.log 2>&1
echo "rc=$?" >> gpurun_out/mb3_pytest_mbvf.log
bash scripts/ab_bench.sh gpurun_out/mb3_tet.jsonl "main tsp tmb" "4 3 5" 2 --workload hybrid
bash scripts/ab_bench.sh gpurun_out/mb3_n5.jsonl "main mbvf" "5" 3
PDG_LIB_PATH=$V/fud/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_parity.py -k "6 or 7" > gpurun_out/mb3_pytest_fud.log 2>&1
echo "rc=$?" >> gpurun_out/mb3_pytest_fud.log
bash scripts/ab_bench.sh gpurun_out/mb3_fud.jsonl "main fud" "6 7" 2
