timeout 900 python -m pytest tests/test_gpu_init_optim.py tests/test_gpu_infer.py -x -q 2>&1 | tail -2
for c in 7b 13b 70b_dp; do
timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print('$c', round(d['ms_per_step'],1), round(d['value']), round(d['pct_peak']['of_burst'],3), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value']), d['config']['update_schedule'], d['loss_last_step'])"
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
