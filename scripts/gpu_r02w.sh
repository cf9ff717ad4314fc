#!/bin/bash
# r02w: current HEAD (gain identity A28) -- GPU tier + smoke, default bench
# line, ncu launch list and --set full of one exit's GEMMs.
TAG=${1:-r02w}
mkdir -p gpurun_out
bash scripts/gpu_suite.sh $TAG
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 300 gpurun_out/${TAG}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm -s 0 -c 9 \
    -o gpurun_out/prof_gemm_$TAG python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
ls -la gpurun_out/ | tail -6
timeout 600 python scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer.jsonl 2> gpurun_out/${TAG}_infer.err
EE_INFER_M=1 EE_INFER_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file gpurun_out/launches_infer_$TAG.csv python scripts/bench_infer.py 70b > gpurun_out/ncu_infer_$TAG.log 2>&1
