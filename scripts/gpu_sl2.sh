#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
PDG_WEDGE_SL=1 timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_parity_sizes.py -k "1" > gpurun_out/sl2_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/sl2_pytest.log
bash scripts/ab_bench.sh gpurun_out/sl2_ab.jsonl "main env:PDG_WEDGE_SL=1" "1" 2
PDG_WEDGE_SL=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:wedge_sl -s 16 -c 1 \
  -o gpurun_out/sl2_n1 -f python bench.py --steps 1 --warmup 3 --degree 1 --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
