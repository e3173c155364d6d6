mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wadg.py -q -x -p no:cacheprovider > gpurun_out/wadg_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/wadg_pytest.log
PDG_WADG_TABLES=global timeout 900 python -m pytest tests/test_gpu_wadg.py -q -x -p no:cacheprovider -k "rhs_matches" > gpurun_out/wadg_pytest_g.log 2>&1; echo "pytest global exit $?"; tail -2 gpurun_out/wadg_pytest_g.log
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
for t in shared global; do
PDG_WADG_TABLES=$t timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/wadg_$t.json 2> gpurun_out/wadg_$t.err; echo "$t $(summ gpurun_out/wadg_$t.json)"
done
