# ncu --set full capture of one kernel of a steady config-5 superstep:
#   bash scripts/prof_one.sh <kernel-regex> <skip> [tiles]
mkdir -p gpurun_out
T=${3:-8}
python scripts/profile_step.py $T 1 > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$1" -s $2 -c 1 \
    -o gpurun_out/prof_one python scripts/profile_step.py $T 1 > gpurun_out/ncu_one.log 2>&1
tail -1 gpurun_out/ncu_one.log
