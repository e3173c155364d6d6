#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 600 python bench.py --steps 5 --warmup 3 --degrees "" --no-cpu-baseline > gpurun_out/mo_bench_check.json 2> gpurun_out/mo_bench_check.err
bash scripts/ab_bench.sh gpurun_out/memonly_ab.jsonl "main memonly" "5 4 7 1 2 3" 1
bash scripts/ab_bench.sh gpurun_out/lo_ab.jsonl "main env:PDG_WEDGE_KERNEL=d" "2 3" 2
