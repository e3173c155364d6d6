mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n5_v8 python bench.py --steps 1 --warmup 3 --degree 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_v8_n5.log 2>&1; echo "ncu1 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_wadg -s 16 -c 1 \
  -o gpurun_out/wadg_n5_v1 python bench.py --steps 1 --warmup 3 --degree 5 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_wadg_n5.log 2>&1; echo "ncu2 $?"
timeout 900 python bench.py --workload hybrid --degree 4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/hybrid_n4.json 2> gpurun_out/hybrid_n4.err; echo "hybrid $?"; cat gpurun_out/hybrid_n4.json; tail -2 gpurun_out/hybrid_n4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tet_stage -s 16 -c 1 \
  -o gpurun_out/tet_n4_v1 python bench.py --workload hybrid --degree 4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_tet_n4.log 2>&1; echo "ncu3 $?"
