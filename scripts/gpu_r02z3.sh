#!/bin/bash
# r02z3: ncu --set full of our GEMM and cuBLAS on the a2 shape (second launch of each).
TAG=${1:-r02z3}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:"gemm|nvjet|xmma|cutlass|sm100" -s 2 -c 2 -o gpurun_out/prof_gemm_vs_cublas_$TAG \
    python scripts/gemm_vs_cublas_one.py > gpurun_out/ncu_gemm_vs_cublas_$TAG.log 2>&1
tail -3 gpurun_out/ncu_gemm_vs_cublas_$TAG.log
