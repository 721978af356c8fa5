#!/bin/bash
# ncu --set full of the stream-pass kernels of one config (after the same command passed without ncu):
#   bash tools/ncu_cfg.sh CFG NTRACES TAG [KERNELS...]  ->  gpurun_out/TAG_<kernel>.ncu-rep
CFG=$1; NT=$2; TAG=$3; shift 3
KS=${@:-replay_kernel cold_hist_kernel}
T=$(python -c "import tracegen; print(tracegen.CONFIGS[$CFG].T)")
timeout 300 python tools/run_cfg.py $CFG $NT $T 2 > /dev/null || exit 1
for K in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f \
      -o gpurun_out/${TAG}_${K%%_kernel} python tools/run_cfg.py $CFG $NT $T 2 > gpurun_out/${TAG}_${K%%_kernel}.log 2>&1
done
