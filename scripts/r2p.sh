mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py tests/test_distributed.py -q -x -rA > gpurun_out/pytest_p.log 2>&1; tail -3 gpurun_out/pytest_p.log
grep -h "Error\|error" gpurun_out/pytest_p.log | head -5
