mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wadg.py -q -x -p no:cacheprovider > gpurun_out/wadg_pytest.log 2>&1; echo "pytest exit $?"; tail -30 gpurun_out/wadg_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/wadg_sweep.json 2> gpurun_out/wadg_sweep.err; echo "bench exit $?"; tail -3 gpurun_out/wadg_sweep.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/wadg_sweep.json").read())
rows=[{'degree':d['config']['degree'],'value':d['value'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
for r in sorted(rows,key=lambda r:r['degree']): print(r['degree'], f"{r['value']:.3e}", f"{r['wedge_kernel_avg_ms']:.3f} ms", f"{r['roofline']['achieved']:.0f} GB/s", f"{r['roofline']['frac']:.3f}")
PY
