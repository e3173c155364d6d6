# round-1 final ncu captures of the current low-order kernel (N = 1, 2) and the ncu launch list
mkdir -p gpurun_out
for n in 1 2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_simt -s 16 -c 1 \
  -o gpurun_out/simt_n${n}_final -f python bench.py --steps 1 --warmup 3 --degree $n --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_simt_n${n}_final.log 2>&1; echo "ncu n$n $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final_n5.csv \
  python bench.py --steps 2 --warmup 3 --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_final.log 2>&1; echo "launches $?"
