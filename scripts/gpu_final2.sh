mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/final_exact.json 2> gpurun_out/final_exact.err; echo "exact $?"
timeout 1200 python bench.py --steps 5 --warmup 3 --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_wadg.json 2> gpurun_out/final_wadg.err; echo "wadg $?"
for N in 1 2 3 4 5 6 7; do timeout 900 python bench.py --workload hybrid --degree $N --degrees "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_hybrid_n$N.json 2> gpurun_out/final_hybrid_n$N.err; done; echo hybrid
for N in 1 2 3 4 5 6 7; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv -k regex:wedge_ -s 16 -c 1 python bench.py --steps 1 --warmup 3 --degree $N --degrees "" --mass wadg --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_wadg_n$N.csv 2>/dev/null
done
for N in 2 3 4 5; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv -k regex:tet_ -s 16 -c 1 python bench.py --workload hybrid --steps 1 --warmup 3 --degree $N --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_tet_n$N.csv 2>/dev/null
done; echo traffic
