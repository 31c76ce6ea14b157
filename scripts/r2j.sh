mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels.py tests/test_horizon.py tests/test_fallback_classifier.py -m gpu -q -x > gpurun_out/pytest_j.log 2>&1; tail -2 gpurun_out/pytest_j.log
grep -h "config5 100 steps" gpurun_out/pytest_j.log
timeout 600 python scripts/time_groups.py > gpurun_out/tg.log 2>&1; cat gpurun_out/tg.log
timeout 1500 python scripts/long_run_check.py 3 1000 > gpurun_out/long3.log 2>&1; tail -4 gpurun_out/long3.log
timeout 1500 python scripts/long_run_check.py 5 1200 > gpurun_out/long5.log 2>&1; tail -4 gpurun_out/long5.log
