timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print(round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
ncu --metrics lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum --clock-control base -k regex:gemm -s 0 -c 10 python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "lts__t_sectors|duration" | awk '{printf "%s ", $3} END {print ""}'
