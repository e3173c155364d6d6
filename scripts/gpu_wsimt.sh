timeout 900 python -m pytest tests/test_gpu_wadg.py tests/test_ab3.py -q -x -p no:cacheprovider > gpurun_out/ws_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/ws_pytest.log | grep -E "passed|failed|Error|^E"
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
for rep in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --degree 1 --degrees 2,3 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/ws.json 2>gpurun_out/ws.err; echo "simt $(summ gpurun_out/ws.json)"; tail -1 gpurun_out/ws.err
PDG_WADG_SIMT_MAX_N=0 timeout 600 python bench.py --steps 5 --warmup 3 --degree 1 --degrees 2,3 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/wd.json 2>/dev/null; echo "dmma $(summ gpurun_out/wd.json)"
done
