mkdir -p gpurun_out
FCSG_LINES_KERNEL=20 python scripts/prof_fc.py > gpurun_out/plain_fc.log 2>&1 && \
FCSG_LINES_KERNEL=20 ncu --set full --clock-control none --import-source on -k regex:lines -s 3 -c 1 -o gpurun_out/s4g_w20 -f \
    python scripts/prof_fc.py > gpurun_out/ncu_fc.log 2>&1
tail -1 gpurun_out/ncu_fc.log
