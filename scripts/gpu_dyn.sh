EE_GEMM_CTA=2 timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
EE_GEMM_CTA=2 python scripts/trace_gemm.py
M="--metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control base -k regex:gemm -s 0 -c 3"
for cta in 1 2; do
echo "CTA=$cta"
EE_GEMM_CTA=$cta ncu $M python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "dram__bytes|duration|hit_rate" | awk '{printf "%s %s  ", $1, $3} END {print ""}'
done
for cta in 1 2 1 2; do
EE_GEMM_CTA=$cta timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('CTA=$cta', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
