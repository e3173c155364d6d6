#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/sp3/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_parity.py -k "1 or 2 or 3" > gpurun_out/sp3_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/sp3_pytest.log
bash scripts/ab_bench.sh gpurun_out/sp3_ab.jsonl "main sp3" "2 3" 2
bash scripts/ab_bench.sh gpurun_out/sp3_hyb.jsonl "main sp3" "2 3" 2 --workload hybrid
