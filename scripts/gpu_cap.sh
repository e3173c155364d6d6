mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read())
except Exception as e:
  print("fail", e); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
for cap in 512 640 768 1024; do for st in 2 1; do
L=paper_1607_03399_b200/_lib_cap$cap/libprismdg_b200.so; [ $cap = 512 ] && L=paper_1607_03399_b200/_lib/libprismdg_b200.so
PDG_LIB_PATH=$PWD/$L PDG_WEDGE_STAGES=$st timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap_${cap}_$st.json 2> gpurun_out/cap_${cap}_$st.err
echo "cap=$cap st=$st $(summ gpurun_out/cap_${cap}_$st.json)"
done; done
