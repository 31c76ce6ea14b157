mkdir -p gpurun_out
python scripts/prof_fc.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fc_lines -s 3 -c 1 -o gpurun_out/prof_fc python scripts/prof_fc.py > gpurun_out/ncu_fc.log 2>&1
tail -1 gpurun_out/ncu_fc.log
