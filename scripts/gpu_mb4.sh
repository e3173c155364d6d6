#!/bin/bash
# WADG flux mbarrier (wmf), exact N=6/7 V exchange by mbarrier (mb67): parity, racecheck, same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/wmf/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_wadg.py \
  tests/test_gpu_parity_sizes.py -k "wadg or config2_copy" > gpurun_out/mb4_pytest_wmf.log 2>&1
echo "rc=$?" >> gpurun_out/mb4_pytest_wmf.log
PDG_LIB_PATH=$V/mb67/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_parity.py tests/test_gpu_ab3_fused.py > gpurun_out/mb4_pytest_mb67.log 2>&1
echo "rc=$?" >> gpurun_out/mb4_pytest_mb67.log
PDG_LIB_PATH=$V/mb67/libprismdg_b200.so timeout 900 compute-sanitizer --tool racecheck \
  --error-exitcode 9 python scripts/racecheck_stage.py 7 exact 20 2,2,2 > gpurun_out/mb4_racecheck_mb67.log 2>&1
echo "rc=$?" >> gpurun_out/mb4_racecheck_mb67.log
bash scripts/ab_bench.sh gpurun_out/mb4_wadg.jsonl "main wmf" "5 6" 2 --mass wadg
bash scripts/ab_bench.sh gpurun_out/mb4_n67.jsonl "main mb67" "6 7" 2
PDG_LIB_PATH=$V/tgf/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py \
  tests/test_gpu_parity_sizes.py tests/test_gpu_edge_cases.py > gpurun_out/mb4_pytest_tgf.log 2>&1
echo "rc=$?" >> gpurun_out/mb4_pytest_tgf.log
bash scripts/ab_bench.sh gpurun_out/mb4_tet.jsonl "main tsp tgf" "4 3 6" 2 --workload hybrid
PDG_LIB_PATH=$V/smb/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_parity.py -k "1 or 2 or 3" > gpurun_out/mb4_pytest_smb.log 2>&1
echo "rc=$?" >> gpurun_out/mb4_pytest_smb.log
PDG_LIB_PATH=$V/smb/libprismdg_b200.so timeout 900 compute-sanitizer --tool racecheck \
  --error-exitcode 9 python scripts/racecheck_stage.py 2 exact 20 2,2,2 > gpurun_out/mb4_racecheck_smb.log 2>&1
echo "rc=$?" >> gpurun_out/mb4_racecheck_smb.log
bash scripts/ab_bench.sh gpurun_out/mb4_simt.jsonl "main smb" "1 2 3" 2
