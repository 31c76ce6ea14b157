mkdir -p gpurun_out
export FCSG_LINE_LB=4
python scripts/profile_step.py 4 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:PassBc -s 5 -c 1 -o gpurun_out/prof_passb3 python scripts/profile_step.py 4 1 > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
