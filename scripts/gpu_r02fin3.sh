#!/bin/bash
# Final-code check after the last kernel edits: GPU tier + smoke, default bench line, decode bench.
TAG=${1:-r02fin3}
mkdir -p gpurun_out
bash scripts/gpu_suite.sh $TAG
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer_70b.jsonl 2>> gpurun_out/${TAG}_infer.err
timeout 900 python bench.py --config 13b_layer --dp-comm plain --no-cpu-baseline > gpurun_out/${TAG}_13b_layer.json 2>> gpurun_out/${TAG}_bench.err
tail -c 300 gpurun_out/${TAG}_bench.json
for p in 1 2 4 8; do timeout 300 python scripts/dp_emulate.py --config 70b_dp --ranks $p --strong; done > gpurun_out/${TAG}_dp_emulate_strong.jsonl 2>> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --gpus 2 --config 13b --steps 3 --no-cpu-baseline > gpurun_out/${TAG}_13b_2ranks_one_gpu.json 2>> gpurun_out/${TAG}_bench.err
