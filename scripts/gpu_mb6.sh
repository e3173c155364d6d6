#!/bin/bash
# low-order flux mbarrier on both workloads (main vs nosmb), late slot at N = 4 (ls45)
cd "$GRAFT_REPO_ROOT" || exit 1
bash scripts/ab_bench.sh gpurun_out/mb6_simt.jsonl "main nosmb" "1 2 3" 2
bash scripts/ab_bench.sh gpurun_out/mb6_simt_hyb.jsonl "main nosmb" "1 2 3" 2 --workload hybrid
bash scripts/ab_bench.sh gpurun_out/mb6_ls.jsonl "main ls45" "4" 3
