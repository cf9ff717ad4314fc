#!/bin/bash
# r02x: TMA-fed stream-K decode kernels (skinny.cu) + PDL -- parity, A/B vs the
# previous build (ablib/base.so), ncu launch list of the new decode call.
TAG=${1:-r02x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_infer.py -q -rA -x > gpurun_out/${TAG}_pytest_infer.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_infer.log
tail -3 gpurun_out/${TAG}_pytest_infer.log
for rep in 1 2; do
  timeout 300 python scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer_new_$rep.jsonl 2>> gpurun_out/${TAG}_infer.err
  EE_PDL=0 timeout 300 python scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer_nopdl_$rep.jsonl 2>> gpurun_out/${TAG}_infer.err
  timeout 300 python scripts/ab_lib.py ablib/base.so scripts/bench_infer.py 70b > gpurun_out/${TAG}_infer_base_$rep.jsonl 2>> gpurun_out/${TAG}_infer.err
done
timeout 300 python scripts/bench_infer.py 7b > gpurun_out/${TAG}_infer_7b_new.jsonl 2>> gpurun_out/${TAG}_infer.err
timeout 300 python scripts/ab_lib.py ablib/base.so scripts/bench_infer.py 7b > gpurun_out/${TAG}_infer_7b_base.jsonl 2>> gpurun_out/${TAG}_infer.err
EE_INFER_M=1 EE_INFER_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file gpurun_out/launches_infer_$TAG.csv python scripts/bench_infer.py 70b > gpurun_out/ncu_infer_$TAG.log 2>&1
head -100 gpurun_out/${TAG}_infer_*.jsonl
