# session 4: register-resident (8 x 35) Cartesian flux passes: parity + timing against the prime-factor passes
mkdir -p gpurun_out
echo "== ct passes"; timeout 300 python scripts/time_passes_raw.py 2>&1 | tail -3
echo "== pfa passes"; FCSG_WPASS_CT=0 timeout 300 python scripts/time_passes_raw.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_kernels.py tests/test_horizon.py -m gpu -q -x > gpurun_out/s4a_pytest.log 2>&1; tail -3 gpurun_out/s4a_pytest.log
ncu --set full --clock-control none --import-source on -k regex:wctpass_kernel -s 10 -c 2 \
      -o gpurun_out/s4c_wctpass -f python scripts/time_passes_raw.py > gpurun_out/s4c_ncu.log 2>&1
tail -1 gpurun_out/s4c_ncu.log
