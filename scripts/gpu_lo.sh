#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
for k in 2 3; do
  PDG_LIB_PATH=$V/lo$k/libprismdg_b200.so timeout 900 python -m pytest tests/test_gpu_parity_sizes.py tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/lo${k}_pytest.log 2>&1
  echo "rc=$?" >> gpurun_out/lo${k}_pytest.log
done
bash scripts/ab_bench.sh gpurun_out/lo_ab2.jsonl "main lo2 lo3 lo4" "1 2 3" 2
