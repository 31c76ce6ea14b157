# The driver's round-end sequence on one B200, timed: GPU tests, smoke, both bench arms with default flags
mkdir -p gpurun_out
t0=$(date +%s); python -m pytest tests/ -x -q -m gpu > gpurun_out/final_pytest.log 2>&1; tail -1 gpurun_out/final_pytest.log; t1=$(date +%s); echo "pytest $((t1-t0)) s"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1; t2=$(date +%s); echo "smoke $((t2-t1)) s"
python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; tail -1 gpurun_out/final_bench_ref.log | cut -c1-250; t3=$(date +%s); echo "bench ref $((t3-t2)) s"
python bench.py > gpurun_out/final_bench.log 2>&1; tail -1 gpurun_out/final_bench.log | cut -c1-250; t4=$(date +%s); echo "bench $((t4-t3)) s"
