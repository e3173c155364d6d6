#!/bin/bash
# ncu --set full captures (one non-first stage launch) of the wedge stage kernels
# for source-level analysis; usage: gpu_r2_prof.sh TAG DEGREE [DEGREE ...]
cd "$GRAFT_REPO_ROOT" || exit 1
tag=$1; shift
for n in "$@"; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:wedge_ -s 16 -c 1 \
    -o gpurun_out/${tag}_n${n} -f python bench.py --steps 1 --warmup 3 --degree $n --degrees "" \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_n${n}.log 2>&1
done
