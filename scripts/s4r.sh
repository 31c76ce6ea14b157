mkdir -p gpurun_out
python scripts/prof_config2.py > gpurun_out/plain_c2.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:line_pass_kernel -s 3 -c 2 -o gpurun_out/s4r_c2y -f python scripts/prof_config2.py > gpurun_out/ncu_c2.log 2>&1
tail -1 gpurun_out/ncu_c2.log
