TAG=${1:-r01h}
timeout 900 python -m pytest tests/test_gpu_adam_fused.py tests/test_gpu_layer.py tests/test_gpu_dp_fused.py tests/test_gpu_vp_fused.py -x -q -p no:cacheprovider > gpurun_out/pytest_laf_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_laf_$TAG.log
for f in "" "--fused-adam"; do
timeout 900 python bench.py --config 13b_layer $f --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_laf${f}_$TAG.json 2> gpurun_out/bench_laf${f}_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_laf${f}_$TAG.json'));print('13b_layer','$f',round(d['value']),round(d['ms_per_step'],2),d['clocks']['sm_mhz'],d['status'])"
done
