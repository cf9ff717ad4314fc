# Full GPU suite + benches of every config after the dS / fused-collective changes.
TAG=${1:-r01f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_$TAG.log
grep -E "^(64|256)\.0 " gpurun_out/pytest_gpu_$TAG.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_70b_$TAG.json 2> gpurun_out/bench_70b_$TAG.err; echo "bench 70b rc=$?"
for c in 7b 13b 70b_dp 13b_layer; do
timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?"
done
for c in 70b 7b 13b 70b_dp 13b_layer; do
python -c "import json;d=json.load(open('gpurun_out/bench_${c}_$TAG.json'));print('$c',round(d['value']),round(d['ms_per_step'],1),round(d['pct_peak']['of_burst'],4),d['clocks']['sm_mhz'],d['e2e']['value'] if d.get('e2e') else None)"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --config tiny_layer --tokens 1024 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_dp2layer_$TAG.json 2> gpurun_out/bench_dp2layer_$TAG.err; echo "bench dp2 layer shared rc=$?"
tail -c 300 gpurun_out/bench_dp2layer_$TAG.json
