for g in 4 8 4 8; do
EE_GEMM_GROUP_LONGK=$g timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('LONGK=$g', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
