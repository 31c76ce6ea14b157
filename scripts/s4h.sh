# TMA-staged rows in the 8 x 35 line kernel: parity + timing against direct loads
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels.py -m gpu -q -x -k "tma_staging or variants_agree" 2>&1 | tail -3
for t in 0 1; do
  echo "== FCSG_LINES_TMA=$t"; FCSG_LINES_TMA=$t timeout 300 python scripts/fc_timing.py 2>&1 | tail -1
  FCSG_LINES_TMA=$t timeout 300 python scripts/fc_batch_timing.py 2>&1 | tail -4
done
