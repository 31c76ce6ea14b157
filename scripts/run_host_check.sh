python -m pytest tests/test_run_host.py -m gpu -q -x 2>&1 | tail -3
bash scripts/quick_bench.sh
