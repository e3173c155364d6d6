# low-order WADG kernel launch bounds fix (min 3 CTAs/SM at N=1, no spills) + WADG GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wadg.py -q -p no:cacheprovider > gpurun_out/wm_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/wm_pytest.log
timeout 1200 python bench.py --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/wm_wadg.json 2> gpurun_out/wm_wadg.err; echo "wadg $?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/wm_wadg.json'))
print('%.4g'%d['value'], round(d['roofline']['frac'],3), d['clocks'], [(r['degree'], '%.3g'%r['value'], round(r['wedge_kernel_avg_ms'],3)) for r in d.get('sweep',[])])
PY
