#!/bin/bash
# r02xb: exits batched per decode launch (up to 4) -- parity, A/B vs the
# unbatched build (ablib/prev.so), ncu launch list.
TAG=${1:-r02xb}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_infer.py -q -rA -x > gpurun_out/${TAG}_pytest_infer.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_infer.log
tail -3 gpurun_out/${TAG}_pytest_infer.log
for rep in 1 2; do
  for c in 70b 7b 13b; do
    timeout 300 python scripts/bench_infer.py $c > gpurun_out/${TAG}_infer_${c}_new_$rep.jsonl 2>> gpurun_out/${TAG}_infer.err
    timeout 300 python scripts/ab_lib.py ablib/prev.so scripts/bench_infer.py $c > gpurun_out/${TAG}_infer_${c}_prev_$rep.jsonl 2>> gpurun_out/${TAG}_infer.err
  done
done
EE_INFER_M=1 EE_INFER_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file gpurun_out/launches_infer_$TAG.csv python scripts/bench_infer.py 70b > gpurun_out/ncu_infer_$TAG.log 2>&1
for f in gpurun_out/${TAG}_infer_*_1.jsonl; do echo $f; head -3 $f | cut -c1-110; done
