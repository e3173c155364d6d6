cd "$GRAFT_REPO_ROOT"
bash scripts/ab_bench.sh gpurun_out/ab1.jsonl "base regops" "5 4 6 7" 2
bash scripts/gpu_r2_prof.sh p1 5 2
