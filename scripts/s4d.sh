mkdir -p gpurun_out
echo "== wct lines"; timeout 300 python scripts/fc_batch_timing.py 2>&1 | tail -4
echo "== w280 lines"; FCSG_NO_WCT_LINES=1 timeout 300 python scripts/fc_batch_timing.py 2>&1 | tail -4
timeout 600 python -m pytest tests/test_kernels.py -m gpu -q -x -k "register_resident" 2>&1 | tail -2
