mkdir -p gpurun_out
timeout 1700 python scripts/config2_horizon.py 512 50 100 200 > gpurun_out/config2_horizon.log 2>&1; cat gpurun_out/config2_horizon.log | tail -5
