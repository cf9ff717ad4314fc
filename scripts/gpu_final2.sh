TAG=${1:-r01h}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_70b_$TAG.json 2> gpurun_out/bench_70b_$TAG.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_70b_$TAG.json'));print(round(d['value']),round(d['ms_per_step'],1),round(d['pct_peak']['of_burst'],4),d['clocks'],round(d['e2e']['value']),d['status'],d['roofline']['kernel'],round(d['roofline']['frac'],3),d['gpu_launches'])"
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref_$TAG.json
