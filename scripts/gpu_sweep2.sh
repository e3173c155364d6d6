mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_exact.json 2> gpurun_out/final_exact.err; echo "exact $?"
for N in 1 2 3 4 5 6 7; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv -k regex:wedge_ -s 16 -c 1 python bench.py --steps 1 --warmup 3 --degree $N --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_exact_n$N.csv 2>/dev/null
done; echo traffic
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n5_v9 python bench.py --steps 1 --warmup 3 --degree 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_v9_n5.log 2>&1; echo "ncu $?"
