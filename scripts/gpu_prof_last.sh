# ncu --set full of the final exact DMMA stage kernel at N = 4 and N = 7 (round-1 last build)
mkdir -p gpurun_out
for n in 4 7; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_dmma -s 16 -c 1 \
  -o gpurun_out/wedge_n${n}_last -f python bench.py --steps 1 --warmup 3 --degree $n --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu n$n $?"
done
