# multi-GPU driver on one GPU: threaded DistributedLSERK parity + the partitioned bench path (1-rank NCCL group)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_partition.py -q -p no:cacheprovider > gpurun_out/dist_pytest.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/dist_pytest.log
timeout 900 python bench.py --partitioned --steps 5 --warmup 3 --degrees "" --no-cpu-baseline --e2e-steps 2 > gpurun_out/dist_bench.json 2> gpurun_out/dist_bench.err; echo "bench partitioned $?"; cat gpurun_out/dist_bench.json; tail -5 gpurun_out/dist_bench.err
timeout 900 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --partitioned --steps 5 --warmup 3 --degree 3 --degrees "" --no-cpu-baseline --e2e-steps 1 > gpurun_out/dist_bench_trun.json 2> gpurun_out/dist_bench_trun.err; echo "torchrun partitioned $?"; cat gpurun_out/dist_bench_trun.json; tail -5 gpurun_out/dist_bench_trun.err
