# ncu --set full captures of the top kernels of a steady config-5 superstep
# (8x8 tiling, the bench workload), after the same command ran clean without ncu
mkdir -p gpurun_out
python scripts/profile_step.py 8 1 > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for ks in ${KERNELS:-classify_mma_kernel:1 PassXc:6 PassYc:6}; do
  k=${ks%%:*}; s=${ks##*:}
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$k" -s $s -c 1 \
      -o gpurun_out/prof_$k python scripts/profile_step.py 8 1 > gpurun_out/ncu_$k.log 2>&1
  tail -1 gpurun_out/ncu_$k.log
done
