# world-2 DP and VP paths of bench.py on ONE GPU (gloo over CUDA tensors; test mode)
for par in dp vp; do
echo "== $par"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --config 13b --tokens 4096 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --parallel $par 2>&1 | grep -v "^W\|warn" | tail -3 | cut -c1-600
done
