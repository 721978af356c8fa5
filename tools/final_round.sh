#!/bin/bash
# Round-end GPU evidence in one session (each step after the previous exited 0 without a profiler):
#   bash tools/final_round.sh TAG  ->  gpurun_out/TAG_*
TAG=${1:-r02}
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.txt 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg3.json 2> gpurun_out/${TAG}_bench_cfg3.err || exit 1
timeout 600 python bench.py --config 2 > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
timeout 900 python tools/chain_time.py > gpurun_out/${TAG}_chain_split.txt 2>&1
bash tools/ncu_round.sh ${TAG}
