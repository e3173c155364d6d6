# WADG volume-first (_lib vs _lib_wvf0) and exact no-end-barrier up to N=7 (_lib_ne7 vs _lib); same box, alternating
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/vf2_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/vf2_pytest.log
for rep in 1 2; do
for v in _lib _lib_wvf0; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 900 python bench.py --mass wadg --steps 5 --warmup 3 --degree 5 --degrees 4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/vf2w_$v.json 2>/dev/null; echo "wadg $v $(summ gpurun_out/vf2w_$v.json)"
done
for v in _lib _lib_ne7; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 900 python bench.py --steps 5 --warmup 3 --degree 6 --degrees 7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/vf2e_$v.json 2>/dev/null; echo "exact $v $(summ gpurun_out/vf2e_$v.json)"
done
done
