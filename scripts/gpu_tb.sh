#!/bin/bash
# ticket batch (elements per ticket) re-sweep on the final build
cd "$GRAFT_REPO_ROOT" || exit 1
bash scripts/ab_bench.sh gpurun_out/tb_n4.jsonl "main env:PDG_TICKET_BATCH=2 env:PDG_TICKET_BATCH=8" "4" 2
bash scripts/ab_bench.sh gpurun_out/tb_n67.jsonl "main env:PDG_TICKET_BATCH=1 env:PDG_TICKET_BATCH=4" "6 7" 2
