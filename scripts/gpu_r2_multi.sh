#!/bin/bash
# the multi-GPU bench path at one GPU on the final build: partitioned weak (config 5, 1e6 owned wedges, NCCL
# group of one, interior/boundary split launches) and strong scaling (4e6 wedges), direct and under torchrun
cd "$GRAFT_REPO_ROOT" || exit 1
tag=${1:-mg}
timeout 900 python bench.py --partitioned --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_partitioned.json 2> gpurun_out/${tag}_partitioned.err
timeout 900 python bench.py --scaling strong --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_strong.json 2> gpurun_out/${tag}_strong.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --partitioned --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_torchrun.json 2> gpurun_out/${tag}_torchrun.err
