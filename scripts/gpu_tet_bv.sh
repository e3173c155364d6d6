# tet DMMA kernel: W_a columns built while the gathers are in flight (_lib) vs control (_lib_bv0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bv_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/bv_pytest.log
for rep in 1 2; do
for v in _lib _lib_bv0; do
line="$v"
for N in 3 4 5 6; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 600 python bench.py --workload hybrid --degree $N --degrees "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bv_$v.json 2> gpurun_out/bv_$v.err
line="$line N$N:$(python -c "import json; d=json.load(open('gpurun_out/bv_$v.json')); print('%.3f/%.3f' % (d['tet_kernel_avg_ms'], d['wedge_kernel_avg_ms']))" 2>/dev/null)"
done
echo "$line"
done
done
