#!/bin/bash
# round-2 late A/B: DMMA latency microbenchmark, 480-thread wedge CTAs, tet kernel register/ordering variants
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 120 ./scripts/micro/dmma_latency > gpurun_out/ab2_dmma_latency.txt 2>&1
bash scripts/ab_bench.sh gpurun_out/ab2_wedge.jsonl "main w480" "5 4" 2
bash scripts/ab_bench.sh gpurun_out/ab2_tet.jsonl "main tetL tetLO tetLR" "4 5 3" 2 --workload hybrid
