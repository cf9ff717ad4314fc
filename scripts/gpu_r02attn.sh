#!/bin/bash
# r02attn: ncu --set full (source-level) of the attention backward kernels at the 13B Layer shape.
TAG=${1:-r02attn}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_(dkdv|dq)" -s 2 -c 2 \
    -o gpurun_out/prof_attn_bwd_$TAG python scripts/attn_bwd_one.py > gpurun_out/ncu_attn_bwd_$TAG.log 2>&1
tail -3 gpurun_out/ncu_attn_bwd_$TAG.log
