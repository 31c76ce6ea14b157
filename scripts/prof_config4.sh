mkdir -p gpurun_out
python scripts/profile_config.py 4 1 > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv python scripts/profile_config.py 4 1 > gpurun_out/ncu4.log 2>&1
tail -1 gpurun_out/plain4.log
