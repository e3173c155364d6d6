# final round-1 verification of the committed build: GPU tests, smoke, default bench (+sweep), WADG, hybrid N=4, reference arm
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f7_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/f7_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
timeout 1200 python bench.py > gpurun_out/f7_bench.json 2> gpurun_out/f7_bench.err; echo "bench $?"
timeout 1200 python bench.py --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/f7_wadg.json 2> gpurun_out/f7_wadg.err; echo "wadg $?"
timeout 900 python bench.py --workload hybrid --degree 4 --degrees "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/f7_hybrid_n4.json 2> gpurun_out/f7_hybrid_n4.err; echo "hybrid $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f7_ref.json 2> gpurun_out/f7_ref.err; echo "ref $?"
python - <<'PY'
import json
for f in ['f7_bench','f7_wadg','f7_hybrid_n4']:
    try: d=json.load(open(f'gpurun_out/{f}.json'))
    except Exception as e: print(f, 'fail', e); continue
    print(f, '%.4g'%d['value'], round(d['roofline']['frac'],3), d['clocks'], [(r['degree'], '%.3g'%r['value'], round(r['wedge_kernel_avg_ms'],3), round(r['roofline']['frac'],3)) for r in d.get('sweep',[])], d.get('tet_kernel_avg_ms'))
PY
