timeout 300 python -m pytest tests/test_gpu_gemm.py -q -k large_k 2>&1 | grep -E "assert|Error|passed|failed" | head -5
EE_GEMM_CTA=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -q -k large_k 2>&1 | tail -1
for cta in 1 2 1 2; do
EE_GEMM_CTA=$cta timeout 900 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('CTA=$cta', round(d['ms_per_step'],1), round(d['value']), d['clocks']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
