#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/noend6b/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_ab3_fused.py -k "6 or bitwise" > gpurun_out/n6b_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/n6b_pytest.log
bash scripts/ab_bench.sh gpurun_out/n6b_ab.jsonl "main noend6b" "6" 3
