#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
bash scripts/ab_bench.sh gpurun_out/tbw.jsonl "main env:PDG_TICKET_BATCH=2 env:PDG_TICKET_BATCH=8" "5 7" 2 --mass wadg
