# Final round-2 evidence on one B200, on the committed code: GPU tests, smoke,
# both bench arms, then the ncu captures of scripts/prof_r02.sh (launch list,
# --set full of every kernel of one steady superstep, source captures of the
# hot kernels, the config-1 FC derivative).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
python scripts/fc_batch_timing.py > gpurun_out/fc_batch.log 2>&1; cat gpurun_out/fc_batch.log
bash scripts/prof_r02.sh > gpurun_out/prof_r02.log 2>&1; tail -3 gpurun_out/prof_r02.log
rm -f gpurun_out/r02_all_details.csv
timeout 1500 python scripts/config_scale.py gpurun_out/config_scale.json > gpurun_out/config_scale.log 2>&1; cut -c1-200 gpurun_out/config_scale.log | tail -3
