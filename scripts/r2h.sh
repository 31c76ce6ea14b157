mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dropin.py tests/test_distributed_gpu.py tests/test_kernels.py -m gpu -q -x -rA > gpurun_out/pytest_h.log 2>&1; tail -3 gpurun_out/pytest_h.log
grep -h "classifier:" gpurun_out/pytest_h.log | head -4
timeout 600 python scripts/time_groups.py > gpurun_out/tg.log 2>&1; cat gpurun_out/tg.log
timeout 1200 python scripts/config_scale.py gpurun_out/config_scale.json > gpurun_out/config_scale.log 2>&1; tail -3 gpurun_out/config_scale.log
