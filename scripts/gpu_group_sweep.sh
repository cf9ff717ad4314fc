for g in 16 4 8 32 64 16; do
EE_GEMM_GROUP=$g timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('GROUP=$g', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'], {n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
