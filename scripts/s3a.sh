# session 3: health check of HEAD on the B200 (full GPU suite + bench line)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3a_pytest_gpu.log 2>&1; tail -3 gpurun_out/s3a_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/s3a_bench.log 2>&1; tail -1 gpurun_out/s3a_bench.log | cut -c1-400
timeout 300 python scripts/fc_timing.py > gpurun_out/s3a_fc.log 2>&1; cat gpurun_out/s3a_fc.log
