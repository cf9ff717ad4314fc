#!/bin/bash
# Final-code consolidation on one box (driver-style invocations): GPU tier +
# smoke, default bench line, reference arm, config sweep, --gpus 2 on one GPU,
# decode bench, ncu launch list + --set full of one exit's GEMMs.
TAG=${1:-r02fin}
mkdir -p gpurun_out
bash scripts/gpu_suite.sh $TAG
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
bash scripts/gpu_configs_r02.sh ${TAG}s > gpurun_out/${TAG}_configs.txt 2>&1
timeout 900 python bench.py --gpus 2 --config 13b --steps 3 --no-cpu-baseline > gpurun_out/${TAG}_13b_2ranks_one_gpu.json 2> gpurun_out/${TAG}_2ranks.err
timeout 300 python scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer_70b.jsonl 2>> gpurun_out/${TAG}_infer.err
timeout 300 python scripts/bench_infer.py 7b > gpurun_out/${TAG}_infer_7b.jsonl 2>> gpurun_out/${TAG}_infer.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm -s 0 -c 9 \
    -o gpurun_out/prof_gemm_$TAG python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
cat gpurun_out/${TAG}_configs.txt
tail -c 300 gpurun_out/${TAG}_bench.json
