TAG=${1:-r01g}
timeout 600 python -m pytest tests/test_gpu_init_optim.py tests/test_gpu_adam_fused.py -x -q -p no:cacheprovider > gpurun_out/pytest_sh_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sh_$TAG.log
for c in 7b 70b; do
timeout 900 python bench.py --config $c --no-cpu-baseline --steps 6 --warmup 3 > gpurun_out/bench_sh_${c}_$TAG.json 2> gpurun_out/bench_sh_${c}_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_sh_${c}_$TAG.json'));print('$c',round(d['value']),round(d['ms_per_step'],3),round(d['e2e']['value']),round(d['e2e']['ms_per_step'],3))"
done
