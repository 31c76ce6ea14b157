mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels.py -m gpu -q -x -k "fc or line or deriv" > gpurun_out/pytest_e.log 2>&1; tail -2 gpurun_out/pytest_e.log
timeout 600 python scripts/time_groups.py 2 2 > gpurun_out/tg.log 2>&1; head -3 gpurun_out/tg.log
