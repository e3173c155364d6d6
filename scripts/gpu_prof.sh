set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tet_box" -p no:cacheprovider 2>&1 | tail -3
# launch list of one short bench (N=5), then a full capture of one wedge stage launch
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wedge_stage -s 15 -c 1 \
  -o gpurun_out/wedge_n5_v1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
timeout 1500 python bench.py --steps 5 --warmup 3 --degree 5 --degrees 1,2,3,4,6,7 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sweep_v1.json 2> gpurun_out/sweep_v1.err
cat gpurun_out/sweep_v1.json; tail -5 gpurun_out/sweep_v1.err
