TAG=${1:-r01f}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_adamf_$TAG.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu_adamf_$TAG.log
for c in 70b 7b 13b 70b_dp; do
for f in "" "--no-fused-adam"; do
timeout 900 python bench.py --config $c $f --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_af_${c}${f}_$TAG.json 2> gpurun_out/bench_af_${c}${f}_$TAG.err; echo "bench $c '$f' rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_af_${c}${f}_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],2),round(d['pct_peak']['of_burst'],4),d['clocks']['sm_mhz'],round(d['e2e']['value']), {k:round(v['ms_per_launch']*v['launches_per_step'],2) for k,v in d['kernels'].items() if 'adam' in k or 'dw' in k})"
done; done
