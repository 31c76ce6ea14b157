timeout 300 python -m pytest tests/test_kernels.py -m gpu -q -x -k "fc or line or deriv" 2>&1 | tail -1
for v in 22 21 24 11 12 14; do
  echo "== variant $v"; FCSG_W280_VARIANT=$v timeout 300 python scripts/fc_timing.py 2>&1 | tail -1
done
