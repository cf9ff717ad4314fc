M="--metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control base -k regex:gemm -s 0 -c 10"
for g in 1 2 4; do
echo "LONGK GROUP=$g"
EE_GEMM_GROUP_LONGK=$g ncu $M python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "dram__bytes_read|duration" | awk '{printf "%s ", $3} END {print ""}'
done
for g in 4 2 1 4 2; do
EE_GEMM_GROUP_LONGK=$g timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('LONGK=$g', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz'])"
done
