#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants/pfs/libprismdg_b200.so
PDG_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity_sizes.py -q -x -k "not full_size" > gpurun_out/pfs_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pfs_pytest.log
if grep -q "^rc=0" gpurun_out/pfs_pytest.log; then
  bash scripts/ab_bench.sh gpurun_out/pfs_ab.jsonl "main pfs" "1 2 3" 3
fi
