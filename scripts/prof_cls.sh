mkdir -p gpurun_out
python scripts/profile_step.py 4 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k classify_kernel -s 1 -c 1 -o gpurun_out/prof_cls2 python scripts/profile_step.py 4 1 > gpurun_out/ncu2.log 2>&1
tail -1 gpurun_out/ncu2.log
