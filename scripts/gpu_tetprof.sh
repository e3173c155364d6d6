#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tet_dmma -s 8 -c 1 \
  -o gpurun_out/tet4 -f python bench.py --steps 1 --warmup 3 --workload hybrid --degree 4 --degrees "" \
  --no-cpu-baseline --e2e-steps 1 > gpurun_out/tet4.log 2>&1
