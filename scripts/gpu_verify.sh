# Round-1 verification: GPU tests, smoke, default bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/verify_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/verify_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/verify_smoke.log
timeout 900 python bench.py > gpurun_out/verify_bench.json 2> gpurun_out/verify_bench.err; echo "bench exit $?"; cat gpurun_out/verify_bench.json; tail -3 gpurun_out/verify_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/verify_ref.json 2> gpurun_out/verify_ref.err; echo "ref exit $?"; cat gpurun_out/verify_ref.json
