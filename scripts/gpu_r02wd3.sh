#!/bin/bash
# ${TAG}: 256 x 512 pair tiles for the long-K GEMMs (EE_GEMM_WIDE=1) in the step: interleaved C4 / C2 A/B.
TAG=${1:-r02wd3}
mkdir -p gpurun_out
for rep in 1 2; do
  for w in 0 3; do
    EE_GEMM_WIDE=$w timeout 600 python bench.py --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c4_w${w}_$rep.json 2>> gpurun_out/${TAG}.err
    EE_GEMM_WIDE=$w timeout 600 python bench.py --config 13b --dp-comm plain --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c2_w${w}_$rep.json 2>> gpurun_out/${TAG}.err
  done
done
for f in gpurun_out/${TAG}_c*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
k=d['kernels']; print('$f', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], ' '.join(f'{n}:{v[\"tflops_exec\"]:.0f}' for n,v in k.items() if v.get('tflops_exec')))"; done
