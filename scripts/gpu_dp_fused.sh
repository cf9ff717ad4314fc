# Fused DP (ZeRO-1) + fused VP: GPU tests, N=1 A/B (fused path at world 1 vs plain), 2 ranks on one GPU.
TAG=${1:-r01f}
timeout 900 python -m pytest tests/test_gpu_dp_fused.py tests/test_gpu_vp_fused.py -x -q > gpurun_out/pytest_dpfused_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_dpfused_$TAG.log
for f in "" "--force-dp-fused"; do
timeout 900 python bench.py --config 70b_dp $f --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_dp1${f}_$TAG.json 2> gpurun_out/bench_dp1${f}_$TAG.err; echo "bench dp1 '$f' rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_dp1${f}_$TAG.json'));print(d['value'],d['ms_per_step'],d['pct_peak']['of_burst'], {k:(v['ms_per_launch'],v['launches_per_step']) for k,v in d['kernels'].items() if 'adam' in k})"
tail -3 gpurun_out/bench_dp1${f}_$TAG.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config 13b --tokens 4096 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_dp2shared_$TAG.json 2> gpurun_out/bench_dp2shared_$TAG.err; echo "bench dp2 shared rc=$?"
tail -c 400 gpurun_out/bench_dp2shared_$TAG.json; grep -v OMP gpurun_out/bench_dp2shared_$TAG.err | tail -5
