#!/bin/bash
# N = 6: Fu1 in the V padding column (f1v); N = 5: epilogue normals as 16-byte pairs (nv): parity + same-box A/B
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
PDG_LIB_PATH=$V/f1v/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_parity.py -k "6" > gpurun_out/mb7_pytest_f1v.log 2>&1
echo "rc=$?" >> gpurun_out/mb7_pytest_f1v.log
PDG_LIB_PATH=$V/nv/libprismdg_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_parity_sizes.py \
  tests/test_gpu_ab3_fused.py -k "5 or config2_copy or full_size or bitwise" > gpurun_out/mb7_pytest_nv.log 2>&1
echo "rc=$?" >> gpurun_out/mb7_pytest_nv.log
bash scripts/ab_bench.sh gpurun_out/mb7_f1v.jsonl "main f1v" "6" 3
bash scripts/ab_bench.sh gpurun_out/mb7_nv.jsonl "main nv" "5" 3
