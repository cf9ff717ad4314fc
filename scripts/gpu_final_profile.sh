TAG=${1:-r01d}
bash scripts/gpu_ncu.sh $TAG > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -c 3000 gpurun_out/bench_$TAG.json
