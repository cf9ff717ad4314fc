#!/bin/bash
# r02ax: attention backward timing experiments (variants with the dK/dV softmax
# and / or the dV/dK MMAs compiled out; results garbage, timing only).
TAG=${1:-r02ax}
mkdir -p gpurun_out
for rep in 1 2; do
  for v in prev2 expt_nosm expt_nodvdk expt_both; do
    EE_LIB_AB=ablib/$v.so timeout 300 python scripts/attn_bwd_ab.py > gpurun_out/${TAG}_${v}_$rep.jsonl 2>&1
  done
done
for f in gpurun_out/${TAG}_*.jsonl; do echo "$f $(head -1 $f)"; done
