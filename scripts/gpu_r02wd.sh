#!/bin/bash
# r02wd: 256 x 512 pair tiles (EE_GEMM_WIDE=2, any K) vs 256 x 256 on the plain
# fp32-output GEMM, beside cuBLAS (power-capped, ~3 s per measurement).
TAG=${1:-r02wd}
mkdir -p gpurun_out
for w in 0 2; do
  EE_GEMM_WIDE=$w timeout 600 python scripts/cublas_ab.py > gpurun_out/${TAG}_cublas_w$w.jsonl 2>> gpurun_out/${TAG}.err
  EE_GEMM_WIDE=$w timeout 600 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum \
    --clock-control none -k regex:"gemm|nvjet" --csv --log-file gpurun_out/${TAG}_ncu_w$w.csv python scripts/gemm_vs_cublas_one.py > /dev/null 2>&1
done
