mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels.py tests/test_races.py -m gpu -q -x > gpurun_out/pytest_m.log 2>&1; tail -2 gpurun_out/pytest_m.log
timeout 600 python scripts/time_groups.py > gpurun_out/tg.log 2>&1; cat gpurun_out/tg.log
timeout 300 python scripts/fc_timing.py 2>&1 | tail -2
