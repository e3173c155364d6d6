#!/bin/bash
# ncu --set full captures of the final stage kernels: gpu_r2_m2b.sh TAG "exact degrees" [tet] [wadg]
# (reports stay under the 64 MiB merge limit: pass a few degrees per call)
cd "$GRAFT_REPO_ROOT" || exit 1
tag=$1; degs=$2; shift 2
for n in $degs; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:wedge_ -s 16 -c 1 \
    -o gpurun_out/${tag}_full_n${n} -f python bench.py --steps 1 --warmup 3 --degree $n --degrees "" \
    --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
for x in "$@"; do
  case $x in
    tet) timeout 900 ncu --set full --import-source on --clock-control none -k regex:tet_dmma -s 8 -c 1 \
      -o gpurun_out/${tag}_tet4 -f python bench.py --steps 1 --warmup 3 --workload hybrid --degree 4 --degrees "" \
      --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1 ;;
    wadg) timeout 900 ncu --set full --import-source on --clock-control none -k regex:wedge_wadg -s 16 -c 1 \
      -o gpurun_out/${tag}_wadg5 -f python bench.py --steps 1 --warmup 3 --mass wadg --degree 5 --degrees "" \
      --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1 ;;
  esac
done
