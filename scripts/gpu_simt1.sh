mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/simt_pytest.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/simt_pytest.log | grep -E "passed|failed|Error|assert|^E" | head -20
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read())
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
timeout 900 python bench.py --steps 5 --warmup 3 --degree 1 --degrees 2,3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/simt_sweep.json 2> gpurun_out/simt_sweep.err; echo "simt $(summ gpurun_out/simt_sweep.json)"; tail -2 gpurun_out/simt_sweep.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_simt -s 16 -c 1 \
  -o gpurun_out/simt_n1_v1 python bench.py --steps 1 --warmup 3 --degree 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_simt_n1.log 2>&1; echo "ncu $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_simt -s 16 -c 1 \
  -o gpurun_out/simt_n3_v1 python bench.py --steps 1 --warmup 3 --degree 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_simt_n3.log 2>&1; echo "ncu $?"
