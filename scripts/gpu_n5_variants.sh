# exact N=5: no end barrier (_lib, adopted) vs volume-first with the end barrier (_lib_c); same box, alternating
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in _lib _lib_c; do
PDG_LIB_PATH=$PWD/paper_1607_03399_b200/$v/libprismdg_b200.so timeout 900 python bench.py --steps 5 --warmup 3 --degree 5 --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/n5v_$v.json 2>/dev/null; echo "$v N5:$(python -c "import json; print('%.3f' % json.load(open('gpurun_out/n5v_$v.json'))['wedge_kernel_avg_ms'])")"
done
done
