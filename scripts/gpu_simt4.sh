#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
bash scripts/ab_bench.sh gpurun_out/simt4_ab.jsonl "main env:PDG_SIMT_MAX_N=4" "4" 2
