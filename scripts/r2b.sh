mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python -m pytest tests/test_distributed_gpu.py tests/test_kernels.py -m gpu -q -x > gpurun_out/pytest_b.log 2>&1; tail -3 gpurun_out/pytest_b.log
timeout 600 python scripts/time_groups.py > gpurun_out/tg.log 2>&1; cat gpurun_out/tg.log
