#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants/split/libprismdg_b200.so
PDG_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity_sizes.py tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/split_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/split_pytest.log
if grep -q "^rc=0" gpurun_out/split_pytest.log; then
  bash scripts/ab_bench.sh gpurun_out/split_ab.jsonl "main split" "5 4" 3
fi
