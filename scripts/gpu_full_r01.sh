timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for ws in 2 1 2 1; do
EE_GEMM_WAVESYNC=$ws timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('WAVESYNC=$ws', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
bash scripts/gpu_ncu.sh r01b
