mkdir -p gpurun_out
for n in 1 3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_simt -s 16 -c 1 \
  -o gpurun_out/simt_n${n}_v2 -f python bench.py --steps 1 --warmup 3 --degree $n --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_simt_n${n}_v2.log 2>&1; echo "ncu n$n $?"
done
