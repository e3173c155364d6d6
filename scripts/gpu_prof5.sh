mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v5_n5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_v5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n5_v5 python bench.py --steps 1 --warmup 3 --degree 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_v5_n5.log 2>&1
PDG_WEDGE_STAGES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n7_v5st1 python bench.py --steps 1 --warmup 3 --degree 7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_v5_n7.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default_v5.json 2> gpurun_out/bench_default_v5.err
cat gpurun_out/bench_default_v5.json
