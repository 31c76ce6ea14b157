mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dropin.py tests/test_races.py -m gpu -q -x -rA > gpurun_out/pytest_i.log 2>&1; tail -3 gpurun_out/pytest_i.log
grep -h "classifier:" gpurun_out/pytest_i.log | head -4
timeout 1500 python scripts/config_scale.py gpurun_out/config_scale.json > gpurun_out/config_scale.log 2>&1; tail -5 gpurun_out/config_scale.log | cut -c1-600
