#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/lpl4/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_ab3_fused.py tests/test_gpu_parity.py -k "4 or 5 or config2_copy or bitwise" > gpurun_out/lpl4_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/lpl4_pytest.log
PDG_LIB_PATH=$V/lpl4/libprismdg_b200.so timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python scripts/racecheck_stage.py 4 exact 20 2,2,2 > gpurun_out/lpl4_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/lpl4_racecheck.log
bash scripts/ab_bench.sh gpurun_out/lpl4_ab.jsonl "main lpl4" "4 5" 3
