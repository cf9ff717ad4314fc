#!/bin/bash
# r02sw: SwiGLU-backward epilogue with both halves' loads issued first: parity, interleaved C2 / 13B-Layer / C4 A/B vs ablib/prev3.so.
TAG=${1:-r02sw}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_largen.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for lib in new prev; do
    if [ $lib = new ]; then L=paper_2402_00518_b200/libee_b200.so; else L=ablib/prev3.so; fi
    timeout 600 python scripts/ab_lib.py $L bench.py --config 13b --dp-comm plain --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c2_${lib}_$rep.json 2>> gpurun_out/${TAG}.err
    timeout 600 python scripts/ab_lib.py $L bench.py --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c4_${lib}_$rep.json 2>> gpurun_out/${TAG}.err
  done
done
for f in gpurun_out/${TAG}_c*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
k=d['kernels']; print('$f', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], 'dm', round(k['a11_dm_swiglu_bwd']['tflops_exec']))"; done
