#!/bin/bash
# Final-code ncu evidence for the default bench step: launch list + one exit's GEMMs (--set full).
TAG=${1:-r02f}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm -s 0 -c 10 \
    -o gpurun_out/prof_gemm_$TAG python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
ls -la gpurun_out/ | tail -4
