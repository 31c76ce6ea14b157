# full round measurement: GPU tests, smoke, bench (+ the reference arm), then ncu
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
grep -h "FAILED\|config5 100 steps\|config4 step_flow\|positivity lost\|classifier:" gpurun_out/pytest_gpu.log | head -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
bash scripts/prof_r02.sh > gpurun_out/prof_r02.log 2>&1; ls gpurun_out/*.ncu-rep
