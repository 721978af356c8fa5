#!/bin/bash
# ncu evidence for one config on the GPU box (run after the same command passed without ncu):
#   bash tools/prof_cfg.sh CFG NTRACES TAG   ->  gpurun_out/TAG_launches.csv, TAG_{replay,cold,post}.ncu-rep
set -e
CFG=$1; NT=$2; TAG=$3
T=$(python -c "import tracegen; print(tracegen.CONFIGS[$CFG].T)")
timeout 300 python tools/run_cfg.py $CFG $NT $T 3 > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python tools/run_cfg.py $CFG $NT $T 3 > /dev/null 2>&1 || true
python tools/launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt || true
for K in replay_kernel cold_hist_kernel post_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f \
      -o gpurun_out/${TAG}_${K%%_kernel} python tools/run_cfg.py $CFG $NT $T 2 > gpurun_out/${TAG}_${K%%_kernel}.log 2>&1 || true
done
