#!/bin/bash
# r02 consolidation on one box: GPU tier + smoke, the default bench line, the
# reference arm (driver-style invocations), the 13b_layer line.
TAG=${1:-r02z}
mkdir -p gpurun_out
bash scripts/gpu_suite.sh $TAG
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
timeout 900 python bench.py --config 13b_layer --dp-comm plain --no-cpu-baseline > gpurun_out/${TAG}_bench_13b_layer.json 2> gpurun_out/${TAG}_bench_13b_layer.err
tail -c 400 gpurun_out/${TAG}_bench.json
