#!/bin/bash
# r02ab: attention backward softmax with packed f32x2 ops + hoisted causal mask vs the previous build.
TAG=${1:-r02ab}
mkdir -p gpurun_out
EE_LIB_AB=${PREV:-ablib/prev.so} timeout 300 python scripts/attn_dump.py /tmp/attn_prev.pt > gpurun_out/${TAG}_dump.log 2>&1
timeout 300 python scripts/attn_dump.py /tmp/attn_new.pt >> gpurun_out/${TAG}_dump.log 2>&1
python scripts/attn_cmp.py /tmp/attn_prev.pt /tmp/attn_new.pt > gpurun_out/${TAG}_bitwise.txt 2>&1
for rep in 1 2; do
  EE_LIB_AB=${PREV:-ablib/prev.so} timeout 300 python scripts/attn_bwd_ab.py > gpurun_out/${TAG}_prev_$rep.jsonl 2>&1
  timeout 300 python scripts/attn_bwd_ab.py > gpurun_out/${TAG}_new_$rep.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_layer.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
cat gpurun_out/${TAG}_bitwise.txt; tail -2 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_prev_*.jsonl gpurun_out/${TAG}_new_*.jsonl
