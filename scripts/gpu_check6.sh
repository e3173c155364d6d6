mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu8.log
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read())
rows=[{'degree':d['config']['degree'],'value':d['value'],'roofline':d['roofline'],'wedge_kernel_avg_ms':d['wedge_kernel_avg_ms']}]+d.get('sweep',[])
for r in sorted(rows,key=lambda r:r['degree']): print(r['degree'], f"{r['value']:.3e}", f"{r['wedge_kernel_avg_ms']:.3f} ms", f"{r['roofline']['achieved']:.0f} GB/s", f"{r['roofline']['frac']:.3f}")
PY
}
for ST in 2 1; do
PDG_WEDGE_STAGES=$ST timeout 1500 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sweep_v8_st$ST.json 2> gpurun_out/sweep_v8_st$ST.err
echo "stages=$ST"; summ gpurun_out/sweep_v8_st$ST.json; tail -2 gpurun_out/sweep_v8_st$ST.err
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:wedge_dmma -s 16 -c 1 python bench.py --steps 1 --warmup 3 --degree 5 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "dram__|gpu__time|hit_rate"
