# session 3: register-resident 8x35 FC line kernel: parity + config-1 timing per variant
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels.py -m gpu -q -x -k "fc_" > gpurun_out/s3b_pytest.log 2>&1; tail -2 gpurun_out/s3b_pytest.log
for v in 1 2 4; do echo "== wct WPC $v"; FCSG_WCT_WPC=$v timeout 300 python scripts/fc_timing.py 2>&1 | tail -1; done
echo "== old w280 (4-warp CTAs)"; FCSG_NO_WCT_LINES=1 timeout 300 python scripts/fc_timing.py 2>&1 | tail -1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wct_lines -c 1 -o gpurun_out/s3b_wct python scripts/fc_timing.py > gpurun_out/s3b_ncu.log 2>&1; tail -2 gpurun_out/s3b_ncu.log
