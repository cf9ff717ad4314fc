#!/bin/bash
# r02v: gain identity (MLP exits without the du GEMM) -- GPU tier, then an
# interleaved A/B against the previous build (ablib/base.so) on C4 and C2.
TAG=${1:-r02v}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for rep in 1 2; do
  for lib in new base; do
    if [ $lib = new ]; then L=paper_2402_00518_b200/libee_b200.so; else L=ablib/base.so; fi
    timeout 600 python scripts/ab_lib.py $L bench.py --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c4_${lib}_${rep}.json 2>>gpurun_out/${TAG}_bench.err
    timeout 600 python scripts/ab_lib.py $L bench.py --config 13b --dp-comm plain --no-cpu-baseline --no-ds-ablation --no-e2e > gpurun_out/${TAG}_c2_${lib}_${rep}.json 2>>gpurun_out/${TAG}_bench.err
  done
done
for f in gpurun_out/${TAG}_c*_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('clocks',{}).get('sm_mhz'))")"; done
