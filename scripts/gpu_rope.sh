TAG=${1:-r01f}
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_backbone.py tests/test_gpu_attention.py tests/test_gpu_vp.py tests/test_gpu_vp_fused.py tests/test_gpu_dp_fused.py tests/test_gpu_pp.py -x -q -p no:cacheprovider > gpurun_out/pytest_rope_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_rope_$TAG.log
timeout 900 python bench.py --config 13b_layer --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_rope_13b_layer_$TAG.json 2> gpurun_out/bench_rope_13b_layer_$TAG.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_rope_13b_layer_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],2),round(d['pct_peak']['of_burst'],4),d['clocks']['sm_mhz'],round(d['e2e']['value']),{k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k.startswith('L2') or k.startswith('L8')})"
timeout 900 python bench.py --backbone-layers 20 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_rope_bb_$TAG.json 2> gpurun_out/bench_rope_bb_$TAG.err; echo "bench bb rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_rope_bb_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],2),d.get('pct_peak'),{k:round(v['ms_per_launch'],3) for k,v in d.get('kernels',{}).items() if 'proj' in k})"
