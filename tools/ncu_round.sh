#!/bin/bash
# Round-end ncu evidence on the GPU box: launch lists of configs 2 and 3, and --set full captures of
# replay_kernel / cold_hist_kernel / post_kernel (config 3) and replay_kernel / post_kernel (config 2).
#   bash tools/ncu_round.sh TAG
TAG=${1:-r02}
for C in 3 2; do
  T=$(python -c "import tracegen; print(tracegen.CONFIGS[$C].T)")
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c${C}_launches.csv \
      python tools/run_cfg.py $C 0 $T 3 > /dev/null 2>&1
  python tools/launches.py gpurun_out/${TAG}_c${C}_launches.csv > gpurun_out/${TAG}_c${C}_launches.txt
done
bash tools/ncu_cfg.sh 3 0 ${TAG}_c3 replay_kernel cold_hist_kernel post_kernel
bash tools/ncu_cfg.sh 2 0 ${TAG}_c2 replay_kernel post_kernel
