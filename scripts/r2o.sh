mkdir -p gpurun_out
for rep in 1 2; do
for lib in paper_2506_19370_b200/lib/ab_5170ff2.so paper_2506_19370_b200/lib/libfcsg.so; do
  echo "== $lib"; FCSG_LIB=$lib timeout 600 python scripts/time_groups.py 2>&1 | grep -E "config5|pass_|filter"
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
