for v in "" "EE_GEMM_HINT_B=1" "EE_GEMM_HINT_A=2" "EE_GEMM_HINT_B=1 EE_GEMM_HINT_A=2" ""; do
env $v timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/bench_hint.json 2> gpurun_out/bench_hint.err
python -c "import json;d=json.load(open('gpurun_out/bench_hint.json'));print('$v' or 'default',round(d['value']),round(d['ms_per_step'],1),d['clocks']['sm_mhz'])"
done
timeout 600 python -m pytest tests/test_gpu_vp_fused.py tests/test_gpu_dp_fused.py -q -k "ipc" -p no:cacheprovider 2>&1 | tail -2
