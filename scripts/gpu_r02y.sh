#!/bin/bash
# r02y consolidation on one box (current code: decode kernels + PDL): GPU tier
# + smoke, the default bench line, the reference arm, the config sweep, two
# ranks sharing the GPU through --gpus 2, the decode bench.
TAG=${1:-r02y}
mkdir -p gpurun_out
bash scripts/gpu_suite.sh $TAG
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
bash scripts/gpu_configs_r02.sh ${TAG}s > gpurun_out/${TAG}_configs.txt 2>&1
timeout 900 python bench.py --gpus 2 --config 13b --steps 3 --no-cpu-baseline > gpurun_out/${TAG}_13b_2ranks_one_gpu.json 2> gpurun_out/${TAG}_2ranks.err
timeout 300 python scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer_70b.jsonl 2>> gpurun_out/${TAG}_infer.err
timeout 300 python scripts/bench_infer.py 7b > gpurun_out/${TAG}_infer_7b.jsonl 2>> gpurun_out/${TAG}_infer.err
cat gpurun_out/${TAG}_configs.txt
tail -c 300 gpurun_out/${TAG}_bench.json
