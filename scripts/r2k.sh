mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_horizon.py -m gpu -q -x -k positivity -rA > gpurun_out/pytest_k.log 2>&1; tail -3 gpurun_out/pytest_k.log; grep -h "positivity lost" gpurun_out/pytest_k.log
timeout 1500 python scripts/config_scale.py gpurun_out/config_scale.json > gpurun_out/config_scale.log 2>&1; cut -c1-700 gpurun_out/config_scale.log | tail -4
