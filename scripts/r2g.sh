# compute-sanitizer on the small cases (scripts/sanitize_small.py), then the
# round-2 ncu captures (scripts/prof_r02.sh)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
bash scripts/prof_r02.sh > gpurun_out/prof_r02.log 2>&1; tail -12 gpurun_out/prof_r02.log
