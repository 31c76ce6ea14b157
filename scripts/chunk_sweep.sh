# stage-chunk / stream sweep of the bench (config 5, 2, 3, 4 lines)
mkdir -p gpurun_out
for cs in ${SWEEP:-2:2 2:4}; do
c=${cs%%:*}; n=${cs##*:}
FCSG_STAGE_CHUNKS=$c FCSG_STAGE_STREAMS=$n python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c$n.log 2>&1
echo "chunks $c streams $n"; tail -1 gpurun_out/bench_$c$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['gpu_launches'], 'cfg2', d['config2']['ms_per_step'], 'cfg3', d['config3']['ms_per_step'], 'cfg4', d['config4']['ms_per_step'])"
done
