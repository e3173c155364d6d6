#!/bin/bash
# mbarrier team exchanges in the DMMA wedge kernel: parity of the variants, racecheck, same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
for v in mb1 mb2; do
  PDG_LIB_PATH=$PWD/paper_1607_03399_b200/_variants/$v/libprismdg_b200.so timeout 900 python -m pytest -q -x \
    tests/test_gpu_parity_sizes.py tests/test_gpu_ab3_fused.py tests/test_gpu_parity.py > gpurun_out/mb_pytest_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/mb_pytest_$v.log
done
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/_variants/mb2/libprismdg_b200.so timeout 900 compute-sanitizer --tool racecheck \
  --error-exitcode 9 python scripts/racecheck_stage.py 5 exact 20 2,2,2 > gpurun_out/mb_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/mb_racecheck.log
bash scripts/ab_bench.sh gpurun_out/mb_ab.jsonl "main mb1 mb2" "5 4" 3
