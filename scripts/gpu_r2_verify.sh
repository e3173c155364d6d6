#!/bin/bash
# full GPU suite + smoke + integrator rates + the strong-scaling / partitioned bench paths at one GPU
cd "$GRAFT_REPO_ROOT" || exit 1
tag=${1:-v1}
timeout 1800 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/${tag}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 python scripts/integrator_rates.py > gpurun_out/${tag}_integrators.json 2> gpurun_out/${tag}_integrators.err
timeout 1500 python bench.py --scaling strong --steps 5 --warmup 3 > gpurun_out/${tag}_strong1.json 2> gpurun_out/${tag}_strong1.err
timeout 900 python bench.py --partitioned --steps 10 --warmup 3 > gpurun_out/${tag}_partitioned1.json 2> gpurun_out/${tag}_partitioned1.err
timeout 300 python bench.py --gpus 2 --steps 2 > gpurun_out/${tag}_gpus2.out 2> gpurun_out/${tag}_gpus2.err; echo "rc=$?" >> gpurun_out/${tag}_gpus2.err
