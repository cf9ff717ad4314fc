#!/bin/bash
# r02dp8: the a12 gain-identity epilogue at small K (DP over 8 ranks: 8192 tokens
# per rank): strong-scaling rank emulation P = 1/2/4/8 + the parity tests that
# cover a12 (single GPU, large N, fused DP, comm).
TAG=${1:-r02dp8}
mkdir -p gpurun_out
for p in 1 2 4 8; do timeout 300 python scripts/dp_emulate.py --config 70b_dp --ranks $p --strong; done > gpurun_out/${TAG}_dp_emulate_strong.jsonl 2> gpurun_out/${TAG}.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_largen.py tests/test_gpu_fullsize.py tests/test_gpu_dp_fused.py tests/test_gpu_comm.py tests/test_gpu_adam_fused.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
python -c "
import json
for l in open('gpurun_out/${TAG}_dp_emulate_strong.jsonl'):
    d=json.loads(l); print(d['ranks'], round(d['ms_per_step_rank0'],1), d['kernels_ms_per_step'].get('a12_dw_gateup'))"
