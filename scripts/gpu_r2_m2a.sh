#!/bin/bash
# late round-2 measurement set (small outputs): reference arm, default bench (N=5 + N=1..7 sweep), WADG and
# hybrid sweeps, GPU suite, smoke, ncu launch list
cd "$GRAFT_REPO_ROOT" || exit 1
tag=${1:-m2}
nvidia-smi -q -d CLOCK,POWER > gpurun_out/${tag}_smi.txt 2>&1
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_reference.json 2> gpurun_out/${tag}_reference.err
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 1200 python bench.py --steps 10 --warmup 3 --mass wadg --degrees 1,2,3,4,6,7 --no-cpu-baseline > gpurun_out/${tag}_wadg.json 2> gpurun_out/${tag}_wadg.err
timeout 1200 python bench.py --steps 10 --warmup 3 --workload hybrid --degree 4 --degrees 1,2,3,5,6,7 --no-cpu-baseline > gpurun_out/${tag}_hybrid.json 2> gpurun_out/${tag}_hybrid.err
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${tag}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_n5.csv \
  python bench.py --steps 2 --warmup 3 --degrees "" --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
