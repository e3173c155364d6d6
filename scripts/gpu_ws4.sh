#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for v in wsv wsnov; do
  PDG_WEDGE_WS=1 PDG_LIB_PATH=$PWD/paper_1607_03399_b200/_variants/$v/libprismdg_b200.so timeout 900 python -m pytest tests/test_gpu_parity_sizes.py tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/ws4_pytest_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/ws4_pytest_$v.log
done
bash scripts/ab_bench.sh gpurun_out/ws4_ab.jsonl "main env:PDG_WEDGE_WS=1,PDG_LIB_PATH=$PWD/paper_1607_03399_b200/_variants/wsv/libprismdg_b200.so env:PDG_WEDGE_WS=1,PDG_LIB_PATH=$PWD/paper_1607_03399_b200/_variants/wsnov/libprismdg_b200.so" "5 4 6 7" 2
PDG_WEDGE_WS=1 PDG_LIB_PATH=$PWD/paper_1607_03399_b200/_variants/wsv/libprismdg_b200.so bash scripts/gpu_r2_prof.sh ws4 5
