summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
PDG_SIMT_MAX_N=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "degree" > gpurun_out/s4_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/s4_pytest.log
for rep in 1 2; do
PDG_SIMT_MAX_N=4 timeout 600 python bench.py --steps 5 --warmup 3 --degree 4 --degrees 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4.json 2>/dev/null; echo "simt4 $(summ gpurun_out/s4.json)"
PDG_WEDGE_KERNEL=dmma timeout 600 python bench.py --steps 5 --warmup 3 --degree 4 --degrees 3,2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/d4.json 2>/dev/null; echo "dmma $(summ gpurun_out/d4.json)"
done
