TAG=${1:-r01h}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vp_fused.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pytest_bw2_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_bw2_$TAG.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_bw2_$TAG.json 2> gpurun_out/bench_bw2_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_bw2_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],1),d['clocks']['sm_mhz'],{k:(round(v['ms_per_launch'],3),round(v.get('gbs',0))) for k,v in d['kernels'].items() if 'gbs' in v})"
