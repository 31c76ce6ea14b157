mkdir -p gpurun_out
python scripts/profile_config.py 3 1 > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python scripts/profile_config.py 3 1 > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/plain3.log
