#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
V=$PWD/paper_1607_03399_b200/_variants
bash scripts/ab_bench.sh gpurun_out/knobs_tb.jsonl "main env:PDG_TICKET_BATCH=1 env:PDG_TICKET_BATCH=3 env:PDG_TICKET_BATCH=4" "5 6 7" 2
bash scripts/ab_bench.sh gpurun_out/knobs_tb4.jsonl "main env:PDG_TICKET_BATCH=2 env:PDG_TICKET_BATCH=8" "4" 2
bash scripts/ab_bench.sh gpurun_out/knobs_var.jsonl "main noend7 vf5" "5 6 7" 2
