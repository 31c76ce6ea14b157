#!/bin/bash
# ncu --set full of the warp passes (X, Y) on the bench workload (after a plain run)
mkdir -p gpurun_out
python scripts/time_groups.py > gpurun_out/tg_plain.log 2>&1 || exit 1
for k in wpass_x_kernel wpass_y_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 \
      -o gpurun_out/prof_$k -f python scripts/time_groups.py > gpurun_out/ncu_$k.log 2>&1
done
