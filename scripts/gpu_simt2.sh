summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
for v in _lib _lib_s128_3 _lib_s128_4 _lib_s128_5 _lib_s256_2 _lib_s64_6 _lib_s64_8; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 900 python bench.py --steps 5 --warmup 3 --degree 1 --degrees 2,3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s_$v.json 2> gpurun_out/s_$v.err; echo "$v $(summ gpurun_out/s_$v.json)"
done
