#!/bin/bash
# late ticket-slot publication: exact N=5 (mls) and tet (tls): parity, same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/mls/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_ab3_fused.py -k "5 or config2_copy or full_size or bitwise" > gpurun_out/mb5_pytest_mls.log 2>&1
echo "rc=$?" >> gpurun_out/mb5_pytest_mls.log
PDG_LIB_PATH=$V/tls/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py \
  tests/test_gpu_parity_sizes.py tests/test_gpu_edge_cases.py > gpurun_out/mb5_pytest_tls.log 2>&1
echo "rc=$?" >> gpurun_out/mb5_pytest_tls.log
bash scripts/ab_bench.sh gpurun_out/mb5_n5.jsonl "main mls" "5" 3
bash scripts/ab_bench.sh gpurun_out/mb5_tet.jsonl "main tls" "4 3 5" 2 --workload hybrid
