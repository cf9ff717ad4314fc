# a7 from the stored P~ (elementwise) vs the recompute GEMM: full GPU tests + benches.
TAG=${1:-r01f}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_dsp_$TAG.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_dsp_$TAG.log
for c in 70b 7b 13b; do
for r in 0 1; do
EE_DS_RECOMPUTE=$r timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_dsp_${c}_r${r}_$TAG.json 2> gpurun_out/bench_dsp_${c}_r${r}_$TAG.err; echo "bench $c recompute=$r rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_dsp_${c}_r${r}_$TAG.json'));print(d['value'],d['ms_per_step'],d['pct_peak']['of_burst'],d['clocks']['sm_mhz'],{k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k.startswith('a5') or k.startswith('a7')}, d['loss_last_step'])"
done; done
