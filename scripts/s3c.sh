# session 3: 8x35 FC line kernel, table loads overlapped + PDL: parity + config-1 timing per variant
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels.py -m gpu -q -x -k "fc_" > gpurun_out/s3c_pytest.log 2>&1; tail -2 gpurun_out/s3c_pytest.log
for v in 2 4 8; do echo "== wct WPC $v"; FCSG_WCT_WPC=$v timeout 300 python scripts/fc_timing.py 2>&1 | tail -1;
  echo "== wct WPC $v no PDL"; FCSG_NO_PDL=1 FCSG_WCT_WPC=$v timeout 300 python scripts/fc_timing.py 2>&1 | tail -1; done
echo "== old w280 (4-warp CTAs)"; FCSG_NO_WCT_LINES=1 timeout 300 python scripts/fc_timing.py 2>&1 | tail -1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wct_lines -c 1 -o gpurun_out/s3c_wct python scripts/fc_timing.py > gpurun_out/s3c_ncu.log 2>&1; tail -1 gpurun_out/s3c_ncu.log
