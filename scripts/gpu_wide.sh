timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_vp.py -x -q 2>&1 | tail -2
for w in 1 0 1 0; do
EE_GEMM_WIDE=$w timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('WIDE=$w', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz']); print({n: round(v['ms_per_launch'],1) for n,v in list(k.items())[:10]})"
done
EE_GEMM_WIDE=1 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control base -k regex:gemm -s 0 -c 10 python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "dram__bytes_read|duration|tensor" | awk '{printf "%s ", $3} END {print ""}'
