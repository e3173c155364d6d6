mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/tet_pytest.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/tet_pytest.log | grep -E "passed|failed|Error|assert|^E" | head -20
for N in 4 2 3 5; do
timeout 600 python bench.py --workload hybrid --degree $N --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/hybrid_dmma_n$N.json 2> gpurun_out/hybrid_dmma_n$N.err; echo "hybrid N=$N $?"
python - gpurun_out/hybrid_dmma_n$N.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read())
print(f"value {d['value']:.3e} wedge {d['wedge_kernel_avg_ms']:.3f} ms frac {d['roofline']['frac']:.3f} | tet {d['tet_kernel_avg_ms']:.3f} ms frac {d['tet_roofline']['frac']:.3f}")
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tet_dmma -s 16 -c 1 \
  -o gpurun_out/tet_n4_v2 python bench.py --workload hybrid --degree 4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_tet_n4_v2.log 2>&1; echo "ncu $?"
