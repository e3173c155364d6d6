#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants/pf/libprismdg_b200.so
PDG_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity_sizes.py -q -x -k "not full_size" > gpurun_out/pf_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pf_pytest.log
if grep -q "^rc=0" gpurun_out/pf_pytest.log; then
  bash scripts/ab_bench.sh gpurun_out/pf_ab.jsonl "main pf env:PDG_TICKET_BATCH=4,PDG_LIB_PATH=$V env:PDG_TICKET_BATCH=8,PDG_LIB_PATH=$V" "5 4 6 7" 2
fi
