#!/bin/bash
# r02z2: our tcgen05 GEMM vs cuBLAS on the step's shapes; compute-sanitizer on
# the decode kernels; ncu --set full of one decode call's skinny kernels.
TAG=${1:-r02z2}
mkdir -p gpurun_out
timeout 900 python scripts/cublas_ab.py > gpurun_out/${TAG}_cublas_ab.jsonl 2> gpurun_out/${TAG}_cublas_ab.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_decode.py > gpurun_out/${TAG}_sanitize_decode_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitize_decode_$tool.log
done
EE_INFER_M=1 EE_INFER_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:skinny -s 6 -c 3 \
    -o gpurun_out/prof_decode_$TAG python scripts/bench_infer.py 70b > gpurun_out/ncu_decode_$TAG.log 2>&1
tail -2 gpurun_out/${TAG}_sanitize_decode_*.log
cat gpurun_out/${TAG}_cublas_ab.jsonl
