#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/fold/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_parity.py tests/test_gpu_ab3_fused.py -k "4 or 5 or 6 or 7" > gpurun_out/fold_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/fold_pytest.log
bash scripts/ab_bench.sh gpurun_out/fold_ab.jsonl "main fold" "5 6 7" 2
