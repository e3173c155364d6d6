# elements per ticket for the WADG DMMA kernel after the round-1 schedule changes (env PDG_TICKET_BATCH), same box
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
mkdir -p gpurun_out
for rep in 1 2; do
for B in 1 2 4; do
PDG_TICKET_BATCH=$B timeout 900 python bench.py --mass wadg --steps 5 --warmup 3 --degree 5 --degrees 4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tbw_$B.json 2>/dev/null; echo "B=$B $(summ gpurun_out/tbw_$B.json)"
done
done
