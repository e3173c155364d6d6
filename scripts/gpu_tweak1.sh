mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wadg.py -q -x -p no:cacheprovider > gpurun_out/tw_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/tw_pytest.log
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
for rep in 1 2; do
timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tw_$rep.json 2> gpurun_out/tw_$rep.err; echo "exact $(summ gpurun_out/tw_$rep.json)"
done
timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 3,7 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/tw_w.json 2> gpurun_out/tw_w.err; echo "wadg $(summ gpurun_out/tw_w.json)"
