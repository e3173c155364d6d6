mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wadg.py -q -x -p no:cacheprovider > gpurun_out/batch_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/batch_pytest.log
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read())
rows=[{'degree':d['config']['degree'],'value':d['value'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}ms/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
for B in 1 2 4 8 16; do
PDG_TICKET_BATCH=$B timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/batch_$B.json 2> gpurun_out/batch_$B.err
echo "B=$B"; summ gpurun_out/batch_$B.json
done
PDG_TICKET_BATCH=4 timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 3,7 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/batch_wadg4.json 2> gpurun_out/batch_wadg4.err; echo "wadg B=4"; summ gpurun_out/batch_wadg4.json
