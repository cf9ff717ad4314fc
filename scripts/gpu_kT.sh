timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print(round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); print({n: round(v['ms_per_launch'],2) for n,v in list(k.items())[:16]})"
done
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control base -k regex:gemm -s 0 -c 10 python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "gemm2|tensor|dram|duration" | awk '{printf "%s %s\n", $1, $3}' | paste - - - - 
