mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/final_exact.json 2> gpurun_out/final_exact.err; echo "exact $?"
timeout 1200 python bench.py --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_wadg.json 2> gpurun_out/final_wadg.err; echo "wadg $?"
for N in 1 2 3 4 5 6 7; do timeout 900 python bench.py --workload hybrid --degree $N --degrees "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_hybrid_n$N.json 2> gpurun_out/final_hybrid_n$N.err; done; echo hybrid
for N in 2 3 4 5 6 7; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv -k regex:tet_ -s 16 -c 1 python bench.py --workload hybrid --steps 1 --warmup 3 --degree $N --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_tet_n$N.csv 2>/dev/null
done
for N in 4; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv -k regex:wedge_ -s 16 -c 1 python bench.py --steps 1 --warmup 3 --degree $N --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_exact_n$N.csv 2>/dev/null
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv -k regex:wedge_ -s 16 -c 1 python bench.py --steps 1 --warmup 3 --degree $N --degrees "" --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_wadg_n$N.csv 2>/dev/null
done; echo traffic
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n4_v10 python bench.py --steps 1 --warmup 3 --degree 4 --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tet_dmma -s 16 -c 1 \
  -o gpurun_out/tet_n4_v4 python bench.py --workload hybrid --steps 1 --warmup 3 --degree 4 --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu $?"
