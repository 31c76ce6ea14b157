mkdir -p gpurun_out
python scripts/prof_fc4.py > gpurun_out/plain_fc4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lines -s 3 -c 1 -o gpurun_out/s4q_fc4 -f python scripts/prof_fc4.py > gpurun_out/ncu_fc4.log 2>&1
tail -1 gpurun_out/ncu_fc4.log
