# Fused VP collectives: parity tests, P=1 bench (fused vs nccl path), 2 ranks on one GPU (IPC).
TAG=${1:-r01f}
timeout 900 python -m pytest tests/test_gpu_vp_fused.py tests/test_gpu_vp.py -x -q > gpurun_out/pytest_vpfused_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_vpfused_$TAG.log
for c in fused nccl; do
timeout 600 python bench.py --parallel vp --vp-comm $c --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_vp1_${c}_$TAG.json 2> gpurun_out/bench_vp1_${c}_$TAG.err; echo "bench vp1 $c rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_vp1_${c}_$TAG.json'));print(d['value'],d['ms_per_step'],d['pct_peak']['of_burst'])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --parallel vp --config 13b --tokens 8192 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/bench_vp2shared_$TAG.json 2> gpurun_out/bench_vp2shared_$TAG.err; echo "bench vp2 shared rc=$?"
tail -c 600 gpurun_out/bench_vp2shared_$TAG.json; tail -5 gpurun_out/bench_vp2shared_$TAG.err
