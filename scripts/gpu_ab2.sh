timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for cta in 1 2; do
EE_GEMM_CTA=$cta timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('CTA=$cta', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
