mkdir -p gpurun_out
for N in 3 5; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n${N}_v4 python bench.py --steps 1 --warmup 3 --degree $N --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_v4_n$N.log 2>&1
tail -1 gpurun_out/ncu_v4_n$N.log
done
