#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
bash scripts/ab_bench.sh gpurun_out/ws2_ab.jsonl "main env:PDG_WEDGE_WS=1" "5 4 6 7" 2
PDG_WEDGE_WS=1 bash scripts/gpu_r2_prof.sh ws 5
