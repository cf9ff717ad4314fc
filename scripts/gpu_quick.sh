# quick correctness + bench cycle (one GPU)
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_init_optim.py -x -q 2>&1 | tail -5
timeout 900 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print(json.dumps(d)); [print(n, round(v['ms_per_launch'],2), round(v.get('tflops_exec',0))) for n,v in k.items()]"
