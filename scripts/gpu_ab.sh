# A/B: same box, alternating runs of two library builds
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])) + f"  clk {d['clocks']['sm_mhz']}")
PY
}
ARGS=${ARGS:-"--steps 5 --warmup 3 --degree 5 --degrees 4,6,7 --no-cpu-baseline --e2e-steps 1"}
for rep in 1 2; do for v in ${LIBS:-_lib_old _lib}; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 900 python bench.py $ARGS > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; echo "$v $(summ gpurun_out/ab_$v.json)"
done; done
