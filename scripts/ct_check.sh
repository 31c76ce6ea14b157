python -m pytest tests/test_kernels.py tests/test_multipatch.py -m gpu -q -x 2>&1 | tail -1
bash scripts/quick_bench.sh
