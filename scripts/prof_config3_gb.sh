mkdir -p gpurun_out
python scripts/profile_config.py 3 1 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass_kernel -s 12 -c 6 -o gpurun_out/s4v_c3 -f python scripts/profile_config.py 3 1 > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
