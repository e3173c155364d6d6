mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/v3_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/v3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
timeout 900 python bench.py > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err; echo "bench $?"; python -c "
import json; d=json.load(open('gpurun_out/v3_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['gpu_launches'], d['clocks'], [ (r['degree'], round(r['roofline']['frac'],3)) for r in d['sweep']])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/v3_ref.json 2> gpurun_out/v3_ref.err; echo "ref $?"; cat gpurun_out/v3_ref.json
