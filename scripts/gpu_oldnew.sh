#!/bin/bash
# same-box comparison of the build before the late round-2 synchronisation changes (old = commit 2de33cf)
# and the final build; ticket-batch re-sweep at N = 5 with the mbarrier exchanges
cd "$GRAFT_REPO_ROOT" || exit 1
bash scripts/ab_bench.sh gpurun_out/on_exact.jsonl "old main" "5 1 2 4" 2
bash scripts/ab_bench.sh gpurun_out/on_wadg.jsonl "old main" "5 7" 2 --mass wadg
bash scripts/ab_bench.sh gpurun_out/on_hybrid.jsonl "old main" "4 5" 2 --workload hybrid
bash scripts/ab_bench.sh gpurun_out/on_tb.jsonl "main env:PDG_TICKET_BATCH=1 env:PDG_TICKET_BATCH=4" "5" 2
