mkdir -p gpurun_out
echo "== ct passes"; FCSG_WPASS_CT=1 timeout 300 python scripts/time_passes_raw.py 2>&1 | tail -3
echo "== pfa passes"; timeout 300 python scripts/time_passes_raw.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_kernels.py -m gpu -q -x -k "register_resident" 2>&1 | tail -2
FCSG_WPASS_CT=1 ncu --set full --clock-control none --import-source on -k regex:wctpass_kernel -s 10 -c 2 \
      -o gpurun_out/s4k_wctpass -f python scripts/time_passes_raw.py > gpurun_out/s4k_ncu.log 2>&1
tail -1 gpurun_out/s4k_ncu.log
