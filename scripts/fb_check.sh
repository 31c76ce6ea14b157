python -m pytest tests/test_fallback_classifier.py -m gpu -q -x 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config5_fallback_classifier'])"
