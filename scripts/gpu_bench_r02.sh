#!/bin/bash
# r02 bench checks: default line (C4, N=1), 2 ranks on one GPU from --gpus 2, plain-path A/B.
TAG=${1:-r02b}
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20) > gpurun_out/${TAG}_host.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --gpus 2 --config 13b --steps 3 --no-e2e > gpurun_out/${TAG}_bench_2rank.json 2> gpurun_out/${TAG}_bench_2rank.err
echo "rc=$?" >> gpurun_out/${TAG}_bench_2rank.err
timeout 600 python bench.py --dp-comm plain --no-ds-ablation --no-cpu-baseline > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err
echo "rc=$?" >> gpurun_out/${TAG}_bench_plain.err
tail -c 600 gpurun_out/${TAG}_bench.json
