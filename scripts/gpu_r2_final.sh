#!/bin/bash
# the driver's round-end sequence on the final build: reference arm, bench, GPU suite, smoke, launch list
cd "$GRAFT_REPO_ROOT" || exit 1
tag=${1:-f1}
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${tag}_reference.json 2> gpurun_out/${tag}_reference.err
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${tag}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_n5.csv \
  python bench.py --steps 2 --warmup 3 --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
