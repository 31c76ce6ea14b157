#!/bin/bash
# session 4: ncu --set full of the register-resident passes (X, Y) on the bench workload (after a plain run)
mkdir -p gpurun_out
python scripts/time_passes_raw.py > gpurun_out/s4c_plain.log 2>&1 || exit 1
tail -3 gpurun_out/s4c_plain.log
ncu --set full --clock-control none --import-source on -k regex:wctpass_kernel -s 10 -c 2 \
      -o gpurun_out/s4c_wctpass -f python scripts/time_passes_raw.py > gpurun_out/s4c_ncu.log 2>&1
tail -2 gpurun_out/s4c_ncu.log
