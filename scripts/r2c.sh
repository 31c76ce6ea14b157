mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels.py tests/test_horizon.py tests/test_geometries.py -m gpu -q -x > gpurun_out/pytest_c.log 2>&1; tail -3 gpurun_out/pytest_c.log
grep -h "config5 100 steps\|config4 step_flow" gpurun_out/pytest_c.log
timeout 600 python scripts/time_groups.py > gpurun_out/tg.log 2>&1; cat gpurun_out/tg.log
