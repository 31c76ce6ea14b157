# 14 x 20 line kernel: parity + timing against the 8 x 35 kernel (config 1 graph-timed, and the batch sweep)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels.py -m gpu -q -x -k "fc_ or line or deriv" 2>&1 | tail -2
for k in 20 35; do
  echo "== FCSG_LINES_KERNEL=$k"; FCSG_LINES_KERNEL=$k timeout 300 python scripts/fc_timing.py 2>&1 | tail -1
  FCSG_LINES_KERNEL=$k timeout 300 python scripts/fc_batch_timing.py 2>&1 | tail -4
done
for w in 2 8; do echo "== 20, WPC $w"; FCSG_W20_WPC=$w FCSG_LINES_KERNEL=20 timeout 300 python scripts/fc_timing.py 2>&1 | tail -1; done
