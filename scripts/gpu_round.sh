# One measurement round on the GPU box, in two parts (gpurun brings back at
# most 64 MiB per call, and the full captures alone are ~55 MB):
#   bash scripts/gpu_round.sh bench   tests, smoke, bench (with the CPU
#                                     baseline), the reference arm, the
#                                     kernel launch list of one superstep
#   bash scripts/gpu_round.sh prof1   full ncu captures: classifier, pass X
#   bash scripts/gpu_round.sh prof2   full ncu captures: pass Y, FC derivative
mkdir -p gpurun_out
part=${1:-bench}
if [ "$part" = bench ]; then
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
python scripts/profile_step.py 8 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py 8 1 > gpurun_out/ncu1.log 2>&1
elif [ "$part" = prof1 ]; then
KERNELS="classify_mma_kernel:1 PassXc:6" bash scripts/prof_top.sh
else
KERNELS="PassYc:6" bash scripts/prof_top.sh
bash scripts/prof_fc.sh
fi
