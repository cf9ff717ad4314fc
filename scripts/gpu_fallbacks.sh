TAG=${1:-r01j}
for f in "--dp-comm nccl" "--parallel vp --vp-comm nccl" "--config 70b_dp --tokens 4096 --dp-comm nccl"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config 13b --tokens 4096 $f --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_fb.json 2> gpurun_out/bench_fb.err; echo "'$f' rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_fb.json'));print(round(d['value']),round(d['ms_per_step'],1),d['status'],d['config']['workload'][:40],d['config'].get('dp_comm') or d['config'].get('vp_comm'),d['loss_last_step'])"
grep -v OMP gpurun_out/bench_fb.err | grep -v "^\*" | tail -2
done
