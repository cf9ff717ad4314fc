timeout 900 python bench.py --config 7b --steps 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print(round(d['ms_per_step'],2), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); [print(n, v) for n,v in k.items()]"
