TAG=${1:-r01h}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_70b_$TAG.json 2> gpurun_out/bench_70b_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_70b_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],1),round(d['pct_peak']['of_burst'],4),d['clocks']['sm_mhz'],round(d['e2e']['value']),d['status'],{k:(round(v['ms_per_launch'],3),round(v.get('gbs',0))) for k,v in d['kernels'].items() if 'transpose' in k or 'a7' in k or 'a10' in k})"
