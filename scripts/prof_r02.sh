#!/bin/bash
# Round-2 ncu evidence on the bench workload (config 5 per GPU, 8x8 tiles of
# 256^2), each capture after the same command ran clean without ncu:
#  * the launch list of one steady superstep (gpu__time_duration.sum);
#  * --set full of EVERY kernel of one steady superstep (raw + details CSV
#    exported on the box; the .ncu-rep stays there);
#  * --set full --import-source of the warp passes and the classifier (.ncu-rep
#    brought back for the source page); the config-1 FC derivative.
mkdir -p gpurun_out
R=${ROUND:-r02}
python scripts/profile_step.py 8 1 > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python scripts/profile_step.py 8 1 > gpurun_out/ncu_list.log 2>&1
ncu --profile-from-start off --set full --clock-control none -o /tmp/all -f \
    python scripts/profile_step.py 8 1 > gpurun_out/ncu_all.log 2>&1
ncu -i /tmp/all.ncu-rep --page raw --csv > gpurun_out/${R}_all_raw.csv 2>/dev/null
ncu -i /tmp/all.ncu-rep --page details --csv > gpurun_out/${R}_all_details.csv 2>/dev/null
for k in wpass_x_kernel wpass_y_kernel classify_f32_kernel; do
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/${R}_$k -f python scripts/profile_step.py 8 1 > gpurun_out/ncu_$k.log 2>&1
done
python scripts/prof_fc.py > gpurun_out/plain_fc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lines -s 3 -c 1 -o gpurun_out/${R}_fc_lines -f \
    python scripts/prof_fc.py > gpurun_out/ncu_fc.log 2>&1
ls -la gpurun_out
