TAG=${1:-r01g}
timeout 600 python -m pytest tests/test_gpu_adam_fused.py -x -q -p no:cacheprovider > gpurun_out/pytest_adamf3_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_adamf3_$TAG.log
for c in 7b 13b 70b 7b 13b; do
for f in "--fused-adam" ""; do
timeout 900 python bench.py --config $c $f --no-cpu-baseline --no-e2e --steps 6 --warmup 3 > gpurun_out/bench_af3_${c}${f}_$TAG.json 2> gpurun_out/bench_af3_${c}${f}_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_af3_${c}${f}_$TAG.json'));print('$c','$f',round(d['value']),round(d['ms_per_step'],3),d['clocks']['sm_mhz'],{k:round(v['ms_per_launch']*v['launches_per_step'],2) for k,v in d['kernels'].items() if 'adam' in k or 'dw' in k})"
done; done
