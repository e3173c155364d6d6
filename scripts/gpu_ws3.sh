#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
PDG_WEDGE_WS=1 timeout 900 python -m pytest tests/test_gpu_parity_sizes.py tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/ws3_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ws3_pytest.log
if grep -q "^rc=0" gpurun_out/ws3_pytest.log; then
  bash scripts/ab_bench.sh gpurun_out/ws3_ab.jsonl "main env:PDG_WEDGE_WS=1" "5 4 6 7" 2
  PDG_WEDGE_WS=1 bash scripts/gpu_r2_prof.sh ws3 5
fi
