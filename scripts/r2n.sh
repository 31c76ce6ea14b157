mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels.py -m gpu -q -x > gpurun_out/pytest_n.log 2>&1; tail -1 gpurun_out/pytest_n.log
for c in 5 4; do echo "max CTAs $c"; FCSG_WPASS_MAX_CTAS=$c timeout 600 python scripts/time_groups.py 2>&1 | grep -E "config5|pass_|filter|fc_deriv"; done
