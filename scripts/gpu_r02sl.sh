#!/bin/bash
# r02sl: GEMM epilogue accumulator wait -- try_wait suspend hint (EE_GEMM_SLEEP=1,
# the old default) vs poll + nanosleep(N ns); interleaved C4 bench A/B, cuBLAS
# comparison, ncu instruction counts on the a2 shape.
TAG=${1:-r02sl}
mkdir -p gpurun_out
for rep in 1 2; do
  for sl in 1 1000 300; do
    EE_GEMM_SLEEP=$sl timeout 600 python bench.py --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c4_sl${sl}_$rep.json 2>> gpurun_out/${TAG}_bench.err
  done
done
for sl in 1 1000; do
  EE_GEMM_SLEEP=$sl timeout 600 python scripts/cublas_ab.py > gpurun_out/${TAG}_cublas_sl${sl}.jsonl 2>> gpurun_out/${TAG}_cublas.err
  EE_GEMM_SLEEP=$sl timeout 600 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum --clock-control none \
    -k regex:"gemm|nvjet" --csv --log-file gpurun_out/${TAG}_ncu_inst_sl${sl}.csv python scripts/gemm_vs_cublas_one.py > /dev/null 2>&1
done
for f in gpurun_out/${TAG}_c4_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"; done
