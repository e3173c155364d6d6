# last commit of round 1: GPU tests + smoke + default bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/last_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/last_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
timeout 1200 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; echo "bench $?"
python -c "
import json; d=json.load(open('gpurun_out/last_bench.json'))
print('%.4g'%d['value'], round(d['roofline']['frac'],3), d['clocks'], [(r['degree'], '%.3g'%r['value'], round(r['wedge_kernel_avg_ms'],3), round(r['roofline']['frac'],3)) for r in d.get('sweep',[])])"
