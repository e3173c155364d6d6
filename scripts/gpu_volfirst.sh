# volume products before the flux phase (PDG_VOL_FIRST) vs control, same box, alternating; plus GPU parity
summ() { python - "$1" <<'PY'
import json,sys
try: d=json.loads(open(sys.argv[1]).read())
except Exception as e: print("fail"); sys.exit()
rows=[{'degree':d['config']['degree'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
print(" ".join(f"N{r['degree']}:{r['wedge_kernel_avg_ms']:.3f}/{r['roofline']['frac']:.3f}" for r in sorted(rows,key=lambda r:r['degree'])))
PY
}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/vf_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/vf_pytest.log
for rep in 1 2; do
for v in _lib _lib_vf0; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/vf_$v.json 2> gpurun_out/vf_$v.err; echo "$v $(summ gpurun_out/vf_$v.json)"
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n5_vf -f python bench.py --steps 1 --warmup 3 --degree 5 --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu $?"
