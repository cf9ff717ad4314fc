TAG=${1:-r01f}
timeout 600 python -m pytest tests/test_gpu_adam_fused.py tests/test_gpu_init_optim.py -x -q -p no:cacheprovider > gpurun_out/pytest_ovl_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_ovl_$TAG.log
for c in 70b 7b 13b 70b_dp 13b_layer; do
timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_ovl_${c}_$TAG.json 2> gpurun_out/bench_ovl_${c}_$TAG.err; echo "bench $c rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_ovl_${c}_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],2),round(d['pct_peak']['of_burst'],4),d['clocks']['sm_mhz'],round(d['e2e']['value']),d['status'])"
done
