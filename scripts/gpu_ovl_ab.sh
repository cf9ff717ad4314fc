TAG=${1:-r01f}
for c in 7b 70b 7b 70b; do
for f in "" "--no-overlap"; do
timeout 900 python bench.py --config $c $f --no-cpu-baseline --no-e2e --steps 8 --warmup 3 > gpurun_out/bench_ovlab_${c}${f}_$TAG.json 2> gpurun_out/bench_ovlab_${c}${f}_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_ovlab_${c}${f}_$TAG.json'));print('$c','$f',round(d['value']),round(d['ms_per_step'],3),d['clocks']['sm_mhz'])"
done; done
