mkdir -p gpurun_out
python scripts/prof_fc_batch.py > gpurun_out/plain_fcb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lines -s 2 -c 1 -o gpurun_out/r02_fc_lines_batch -f \
    python scripts/prof_fc_batch.py > gpurun_out/ncu_fcb.log 2>&1
tail -1 gpurun_out/ncu_fcb.log
