mkdir -p gpurun_out
for mb in 2 3 4; do echo "MINB=$mb"; FCSG_CLS32_MINB=$mb timeout 300 python scripts/time_groups.py 8 8 2>&1 | grep -E "fc_deriv|config5|viscosity"; done
timeout 600 python -m pytest tests/test_horizon.py -m gpu -q -x -k config5 2>&1 | tail -2
