TAG=${1:-r01f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_70b_$TAG.json 2> gpurun_out/bench_70b_$TAG.err; echo "bench 70b rc=$?"
for c in 7b 13b 70b_dp 13b_layer; do
timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?"
done
for c in 70b 7b 13b 70b_dp 13b_layer; do
python -c "import json;d=json.load(open('gpurun_out/bench_${c}_$TAG.json'));print('$c',round(d['value']),round(d['ms_per_step'],1),round(d['pct_peak']['of_burst'],4),d['clocks']['sm_mhz'],round(d['e2e']['value']) if d.get('e2e') else None, d['status'])"
done
timeout 1500 bash scripts/gpu_ncu.sh $TAG; echo "ncu rc=$?"
