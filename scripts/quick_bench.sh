# GPU tests of the kernels + the bench line's key numbers
mkdir -p gpurun_out
python -m pytest tests/test_kernels.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k: round(v, 4) for k, v in d['kernel_groups_ms'].items()}, 'cfg2', d['config2']['ms_per_step'], 'cfg3', d['config3']['ms_per_step'], d['config3']['value'], 'cfg4', d['config4']['ms_per_step'], d['config4']['value'], 'fb', d['config5_fallback_classifier']['ms_per_step'], d['config5_fallback_classifier']['viscosity_ms'], 'e2e', d['e2e']['value'], 'fc', d['fc_derivative']['us_per_call'], 'fc4', d['fc_derivative_config1_operator']['us_per_call'])"
